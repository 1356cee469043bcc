// adamas_b200.cu — C ABI implementation (include/adamas_b200.h).
// Host side owns the device cache arrays and launches the sm_100a kernels in
// ops.cuh / fused_decode.cuh on the caller's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <fstream>
#include <list>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/adamas_b200.h"
#include "fused_decode.cuh"
#include "ops.cuh"
#include "harness_select.cuh"

using namespace adamas_dev;

struct adamas_cache {
  int n_kv = 0, head_dim = 0, bits = 0, dtype = 0, device = 0;
  int64_t capacity = 0, seq_len = 0;
  // Tokens >= dirty_from were written by the most recent kernel that wrote
  // this cache; a PDL-launched decode step streams only tokens below it before
  // its grid-dependency wait.
  int64_t dirty_from = 0;
  void* K = nullptr;
  void* V = nullptr;
  uint4* codes = nullptr;  // [n_kv][2 planes][capacity] x 16 B
  int* status = nullptr;  // device sticky status word
  // multi-cluster units: [unit][4] barrier words (zeroed once), lazily sized
  // histogram / partial scratch
  int* xsync = nullptr;
  uint32_t* xhist = nullptr;
  float* xpart = nullptr;
  size_t x_unit_heads = 0;  // (unit, cluster, head) slots the scratch holds
  // decode scratch (lazily grown)
  int32_t* scores = nullptr;
  size_t scores_elems = 0;
  uint16_t* qref = nullptr;
  int32_t* idx = nullptr;
  size_t idx_elems = 0;
};

namespace {

thread_local std::string g_last_error;
unsigned long long* g_trace = nullptr;  // adamas_debug_trace

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define ADAMAS_CUDA(call)                                                                   \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail(ADAMAS_ERR_RUNTIME, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

int launch_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ADAMAS_ERR_RUNTIME, std::string(what) + ": " + cudaGetErrorString(e));
  return ADAMAS_OK;
}

size_t elem_size(int dtype) { return dtype == ADAMAS_BF16 ? 2 : 4; }

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

int sm_count() {
  static std::mutex mu;
  static int n[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  std::lock_guard<std::mutex> lock(mu);
  if (n[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

int check_cache(const adamas_cache* c) {
  if (c == nullptr) return fail(ADAMAS_ERR_CONFIG, "null cache handle");
  return ADAMAS_OK;
}

int grow(int32_t** p, size_t* have, size_t need) {
  if (*have >= need) return ADAMAS_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  ADAMAS_CUDA(cudaMalloc(p, need * sizeof(int32_t)));
  *have = need;
  return ADAMAS_OK;
}

template <typename T>
int launch_append(adamas_cache* c, const void* keys, const void* values, const uint16_t* codes_ref,
                  int64_t n_tokens, cudaStream_t s) {
  const int64_t n_vec = n_tokens * c->n_kv;
  const int64_t warp_blocks = (n_tokens + kAppendNV - 1) / kAppendNV * c->n_kv;  // (token block, kv-head) per warp
  const int64_t blocks_needed = (warp_blocks + kAppendWarps - 1) / kAppendWarps;
  const int grid = (int)std::min<int64_t>(blocks_needed, (int64_t)sm_count() * 4);  // a resident grid, loops
  if (codes_ref)
    append_kernel<T, true><<<grid, kAppendWarps * 32, 0, s>>>(
        (const T*)keys, (const T*)values, codes_ref, n_vec, c->n_kv, c->seq_len, c->capacity, (T*)c->K,
        (T*)c->V, c->codes, c->status);
  else if (n_vec < 4 * kAppend8Warps)  // a few vectors: the 2-per-warp kernel, no idle groups
    append_kernel<T, false><<<grid, kAppendWarps * 32, 0, s>>>(
        (const T*)keys, (const T*)values, nullptr, n_vec, c->n_kv, c->seq_len, c->capacity, (T*)c->K,
        (T*)c->V, c->codes, c->status);
  else {  // bulk: four vectors per warp through the 8-lane encoder
    const int64_t blocks8 = (n_vec + 4 * kAppend8Warps - 1) / (4 * kAppend8Warps);
    const int grid8 = (int)std::min<int64_t>(blocks8, (int64_t)sm_count() * 8);
    append8_kernel<T><<<grid8, kAppend8Warps * 32, 0, s>>>((const T*)keys, (const T*)values, n_vec, c->n_kv,
                                                           c->seq_len, c->capacity, (T*)c->K, (T*)c->V, c->codes,
                                                           c->status);
  }
  return launch_check("append_kernel");
}

int do_append(adamas_cache* c, const void* keys, const void* values, const uint16_t* codes_ref,
              int64_t n_tokens, void* stream) {
  if (int rc = check_cache(c)) return rc;
  if (n_tokens < 0) return fail(ADAMAS_ERR_CONFIG, "append: negative token count");
  if (n_tokens == 0) return ADAMAS_OK;
  if (!keys || !values) return fail(ADAMAS_ERR_CONFIG, "append: null key/value pointer");
  if (c->seq_len + n_tokens > c->capacity)
    return fail(ADAMAS_ERR_CONFIG, "append: cache capacity exceeded");
  const int rc = c->dtype == ADAMAS_BF16
                     ? launch_append<__nv_bfloat16>(c, keys, values, codes_ref, n_tokens, as_stream(stream))
                     : launch_append<float>(c, keys, values, codes_ref, n_tokens, as_stream(stream));
  if (rc == ADAMAS_OK) {
    c->dirty_from = c->seq_len;
    c->seq_len += n_tokens;
  }
  return rc;
}

int check_heads(const adamas_cache* c, int n_q) {
  if (n_q < 1 || n_q % c->n_kv != 0)
    return fail(ADAMAS_ERR_CONFIG, "n_q_heads must be a positive multiple of n_kv_heads");
  return ADAMAS_OK;
}


int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// Launch-plan knobs. Read from the environment ONCE (first use); tests and
// tools override them explicitly through adamas_set_tuning. Nothing on the
// launch path reads the environment.
struct Tuning {
  int qsplit = 0, cluster = 0, P = 1, stages = 0, smem_kb = 0;
  int exact_encode = 0, dbg = 0, no_pdl = 0, composed = 0, require_fused = 0;
  unsigned generation = 0;  // bumped on every change: invalidates cached plans
};
std::mutex g_tuning_mu;
Tuning& tuning_ref() {
  static Tuning t = [] {
    Tuning x;
    x.qsplit = env_int("ADAMAS_QSPLIT", 0);
    x.cluster = env_int("ADAMAS_CLUSTER", 0);
    x.P = std::max(1, env_int("ADAMAS_P", 1));
    x.stages = env_int("ADAMAS_STAGES", 0);
    x.smem_kb = env_int("ADAMAS_SMEM_KB", 0);
    x.exact_encode = env_int("ADAMAS_EXACT_ENCODE", 0);
    x.dbg = env_int("ADAMAS_DBG", 0);
    x.no_pdl = env_int("ADAMAS_NO_PDL", 0);
    x.composed = env_int("ADAMAS_NO_FUSED", 0);
    x.require_fused = env_int("ADAMAS_REQUIRE_FUSED", 0);
    return x;
  }();
  return t;
}
Tuning tuning() {
  std::lock_guard<std::mutex> lock(g_tuning_mu);
  return tuning_ref();
}

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

// Per-device, per-kernel launch facts: the dynamic shared memory a kernel has
// been configured for, and how many clusters of a (C, smem) shape co-reside.
struct KernelFacts {
  size_t smem_configured = 0;
  std::vector<std::pair<std::pair<int, size_t>, int>> max_clusters;  // ((C, smem) -> clusters)
};
std::mutex g_facts_mu;
KernelFacts& kernel_facts(const void* kern, int dev) {
  static std::list<std::pair<std::pair<const void*, int>, KernelFacts>> facts;  // stable references
  for (auto& f : facts)
    if (f.first.first == kern && f.first.second == dev) return f.second;
  facts.push_back({{kern, dev}, KernelFacts{}});
  return facts.back().second;
}

// Global scratch of multi-cluster units (not during graph capture: the first
// eager launch of a shape sizes it).
int ensure_unit_scratch(adamas_cache* c, size_t slots) {
  if (c->x_unit_heads >= slots) return ADAMAS_OK;
  cudaFree(c->xhist);
  cudaFree(c->xpart);
  c->xhist = nullptr;
  c->xpart = nullptr;
  c->x_unit_heads = 0;
  ADAMAS_CUDA(cudaMalloc(&c->xhist, slots * kHistBins * sizeof(uint32_t)));
  ADAMAS_CUDA(cudaMalloc(&c->xpart, slots * kPartStride * sizeof(float)));
  c->x_unit_heads = slots;
  return ADAMAS_OK;
}

// ----------------------------------------------------------------- fused launcher
template <typename T, int G, int SW, int MODE, int CT = 0, bool COLL = false>
int launch_fused_t(FusedParams prm, int C, size_t smem, cudaStream_t s) {
  auto kern = fused_decode_kernel<T, G, SW, MODE, CT, COLL>;
  const int dev = current_device();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(prm.n_seqs * prm.n_kv * prm.qsplit * prm.P * C));
  cfg.blockDim = dim3(kFusedThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[3];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int max_clusters = 0;  // clusters of this (C, smem) shape co-resident on this device
  {
    std::lock_guard<std::mutex> lock(g_facts_mu);
    KernelFacts& kf = kernel_facts((const void*)kern, dev);
    if (kf.smem_configured < smem) {
      ADAMAS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      ADAMAS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      // all of the unified L1/shared array as shared memory: two CTAs per SM need it
      ADAMAS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      kf.smem_configured = smem;
    }
    if (prm.pdl || prm.P > 1) {
      for (auto& e : kf.max_clusters)
        if (e.first.first == C && e.first.second == smem) max_clusters = e.second;
      if (max_clusters == 0) {
        if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters <= 0)
          max_clusters = -1;
        kf.max_clusters.push_back({{C, smem}, max_clusters});
      }
    }
  }
  const int64_t clusters = (int64_t)prm.n_seqs * prm.n_kv * prm.qsplit * prm.P;
  // PDL only when every cluster is co-resident (one wave): dependents then
  // occupy only SMs this grid does not need.
  if (prm.pdl && clusters > max_clusters) prm.pdl = 0;
  // spin barriers between the clusters of a unit: every cluster must be resident at once
  if (prm.P > 1 && clusters > max_clusters) return kFusedUnsupported;
  if (prm.pdl) {
    attr[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
    ++cfg.numAttrs;
  }
  ADAMAS_CUDA(cudaLaunchKernelEx(&cfg, kern, prm));
  return ADAMAS_OK;
}

// Instance choice: FULL only where the launch needs the two-hop exchange,
// multi-cluster units or candidates mode; the compaction form SW from the
// rank length (spans cover it with 2 or 4 mask words, else 32-token groups).
template <typename T, int G>
int launch_fused_g(const FusedParams& prm, int C, size_t smem, cudaStream_t s, bool full, int sw, bool coll) {
  if (full) return sw == 2 ? launch_fused_t<T, G, 2, 1>(prm, C, smem, s) : launch_fused_t<T, G, 0, 1>(prm, C, smem, s);
  if (prm.cand) {  // lean candidates (sw 2, C 4, G <= 2: the one-hop shapes of sequence sharding)
    if constexpr (G <= 2)
      return coll ? launch_fused_t<T, G, 2, 2, 4, true>(prm, C, smem, s) : launch_fused_t<T, G, 2, 2, 4>(prm, C, smem, s);
    else return kFusedUnsupported;
  }
  if (sw == 2) {
    if (C == 4) return coll ? launch_fused_t<T, G, 2, 0, 4, true>(prm, C, smem, s) : launch_fused_t<T, G, 2, 0, 4>(prm, C, smem, s);
    return launch_fused_t<T, G, 2, 0>(prm, C, smem, s);
  }
  if (sw == 4) return C == 1 ? launch_fused_t<T, G, 4, 0, 1, true>(prm, C, smem, s) : launch_fused_t<T, G, 4, 0, 0, true>(prm, C, smem, s);
  return launch_fused_t<T, G, 0, 0>(prm, C, smem, s);
}

template <typename T>
int launch_fused_dtype(const FusedParams& prm, int G, int C, size_t smem, cudaStream_t s) {
  const int64_t nt = kConsumers / G;
  const int sw = prm.chunk <= nt * 64 ? 2 : prm.chunk <= nt * 128 ? 4 : 0;
  const bool coll = prm.chunk > nt * 16;  // spans of 32+ tokens per thread: collected-order masks
  // candidates mode has a lean instance for the common one-hop shape (sw 2, C 4; sequence sharding)
  const bool full = prm.P > 1 || C * G > 8 || (prm.cand != nullptr && !(sw == 2 && C == 4 && G <= 2));
  switch (G) {
    case 1: return launch_fused_g<T, 1>(prm, C, smem, s, full, sw, coll);
    case 2: return launch_fused_g<T, 2>(prm, C, smem, s, full, sw, coll);
    case 4: return launch_fused_g<T, 4>(prm, C, smem, s, full, sw, coll);
    case 8:  // test shapes only: one instance per mode, 32-token groups
      return full || prm.cand ? launch_fused_t<T, 8, 0, 1>(prm, C, smem, s) : launch_fused_t<T, 8, 0, 0>(prm, C, smem, s);
  }
  return kFusedUnsupported;
}

// A launch plan: how one decode step of a shape maps onto clusters.
struct FusedPlan {
  int ok = 0;  // 0: the shape does not fit the single-launch kernel
  int qsplit = 1, G = 1, C = 1, P = 1, chunk = 0, stages = 0;
  size_t smem = 0;
};

// Clusters of C CTAs with `smem` bytes of dynamic shared memory each that
// co-reside on this device (cudaOccupancyMaxActiveClusters of a fused-kernel
// instance: one 544-thread CTA per SM, so the shared-memory size decides).
// Measured on B200 at ~200 KB: 33 clusters of 4, 15 of 8, 7 of 16 (not 148 / C:
// clusters must fit inside a GPC).
int max_active_clusters(int C, size_t smem) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, std::pair<int, size_t>>, int>> memo;  // ((dev, (C, smem)) -> n)
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : memo)
    if (e.first.first == dev && e.first.second.first == C && e.first.second.second == smem) return e.second;
  auto kern = fused_decode_kernel<__nv_bfloat16, 1, 0, 1, 0>;
  {  // configure it for the largest size once (launches of this instance never lower it)
    std::lock_guard<std::mutex> flock(g_facts_mu);
    KernelFacts& kf = kernel_facts((const void*)kern, dev);
    const size_t max_smem = 220 * 1024;
    if (kf.smem_configured < max_smem) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_smem);
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      kf.smem_configured = max_smem;
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)C);
  cfg.blockDim = dim3(kFusedThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = sm_count() / C;  // unknown: assume a full machine
  }
  memo.push_back({{dev, {C, smem}}, n});
  return n;
}

// C CTAs per (sequence, kv-head, q-split part) unit and the per-rank chunk
// for a fixed q-split. P > 1 (opt-in) exchanges histograms and partials
// through global memory with a self-resetting barrier; it is exact but
// measured slower than splitting the q-heads (qsplit), so the automatic
// choice grows C only.
FusedPlan plan_for_split_c(int n_seqs, int n_kv, int n_q, int64_t s_max, int64_t budget, int qsplit, int C,
                           const Tuning& tu);

// The automatic cluster size: the largest C (up to 16) whose grid still fits
// the machine, grown when the rank's chunk does not fit shared memory, then
// shrunk while the clusters would not all co-reside (a grid of more clusters
// than fit runs in two waves: measured 16 x 8-CTA clusters 16.1 us vs 16 x 4
// at 9.2 us per layer for 16 heads of 32K).
FusedPlan plan_for_split(int n_seqs, int n_kv, int n_q, int64_t s_max, int64_t budget, int qsplit, const Tuning& tu) {
  FusedPlan pl = plan_for_split_c(n_seqs, n_kv, n_q, s_max, budget, qsplit, tu.cluster, tu);
  if (!pl.ok || tu.cluster > 0) return pl;
  const int64_t clusters = (int64_t)n_seqs * n_kv * qsplit * pl.P;
  if (clusters * pl.C > sm_count() || clusters <= max_active_clusters(pl.C, pl.smem)) return pl;
  for (int C = pl.C / 2; C >= 1; C /= 2) {
    const FusedPlan q = plan_for_split_c(n_seqs, n_kv, n_q, s_max, budget, qsplit, C, tu);
    if (q.ok && q.C == C && clusters <= max_active_clusters(C, q.smem)) return q;
  }
  return pl;
}

FusedPlan plan_for_split_c(int n_seqs, int n_kv, int n_q, int64_t s_max, int64_t budget, int qsplit, int C_req,
                           const Tuning& tu) {
  FusedPlan pl;
  const int G = n_q / (n_kv * qsplit);
  if (n_q % (n_kv * qsplit) || (G != 1 && G != 2 && G != 4 && G != 8)) return pl;
  if (n_seqs > kMaxSeqs || budget > (1 << 20)) return pl;
  const int units = n_seqs * n_kv * qsplit;
  int C = C_req;
  if (C <= 0) {
    C = 1;
    while (C < 16 && units * C * 2 <= sm_count()) C *= 2;
    // Prefer the one-hop exchange (C x G <= 8, the lean instance) while the
    // rank stays short: measured 4 heads x 32K, C 16 (two hops) 8.20 us vs
    // C 8 7.21 (profiles/r02z2_proxy_h4_c*.json).
    while (C > 1 && C * G > 8 && (s_max + (int64_t)(C / 2) - 1) / (C / 2) <= 8192) C /= 2;
  }
  const int P = std::max(1, tu.P);
  for (;;) {
    int64_t chunk = (s_max + (int64_t)C * P - 1) / ((int64_t)C * P);
    chunk = (chunk + 255) / 256 * 256;
    const int selcap = (int)std::min<int64_t>(budget, chunk);
    // one CTA per SM when the grid fits the machine, else two (always two
    // with the 8-warp build, so consecutive launches co-reside)
    size_t smem_cap = kCtasPerSm == 1 && (size_t)units * C * P <= (size_t)sm_count() ? 220 * 1024 : 108 * 1024;
    if (tu.smem_kb > 0) smem_cap = (size_t)tu.smem_kb * 1024;  // experiments
    const FusedSmem base(G, C, (int)chunk, selcap, 0, P);
    const int want = (int)std::min<int64_t>(kMaxStages, std::max<int64_t>(2, (chunk + kStageTok - 1) / kStageTok));
    int stages = tu.stages;
    if (stages <= 0) {
      stages = want;
      while (stages > 2 && base.total + (size_t)stages * kStageTok * 32 > smem_cap) --stages;
    }
    const FusedSmem L(G, C, (int)chunk, selcap, stages, P);
    const bool fits = chunk <= 65280  // u16 histogram exchange: per-rank counts must stay < 2^16
                      && (L.total <= smem_cap || (stages == 2 && L.total <= (kCtasPerSm == 1 ? 220 : 108) * 1024));
    if (fits) {
      pl.ok = 1;
      pl.qsplit = qsplit;
      pl.G = G;
      pl.C = C;
      pl.P = P;
      pl.chunk = (int)chunk;
      pl.stages = stages;
      pl.smem = L.total;
      return pl;
    }
    if (C >= 16) return pl;  // out of options
    C *= 2;
  }
}

// The automatic q-split (each q-split part re-reads the kv-head's codes for
// its share of the q-heads): among the plans whose clusters all co-reside in
// one wave, the one with the most CTAs (the most SMs streaming), then the
// smallest split; if no plan fits one wave, the one with the smallest cluster
// (measured: 16 x 32K Llama batch, qsplit 1 x C 2 101 us vs qsplit 2 x C 1 87 us
// per layer-step), then the smallest split.
FusedPlan plan_fused(int n_seqs, int n_kv, int n_q, int64_t s_max, int64_t budget, int qsplit, const Tuning& tu) {
  if (qsplit > 0) return plan_for_split(n_seqs, n_kv, n_q, s_max, budget, qsplit, tu);
  if (tu.qsplit > 0) return plan_for_split(n_seqs, n_kv, n_q, s_max, budget, tu.qsplit, tu);
  const int G_all = n_q / n_kv;
  FusedPlan best;
  int64_t best_key[3] = {0, 0, 0};
  for (int qs = 1; qs <= G_all; qs *= 2) {
    if (G_all % qs) break;
    const FusedPlan pl = plan_for_split(n_seqs, n_kv, n_q, s_max, budget, qs, tu);
    if (!pl.ok) continue;
    const int64_t clusters = (int64_t)n_seqs * n_kv * qs * pl.P;
    const bool one_wave = clusters * pl.C <= sm_count() && clusters <= max_active_clusters(pl.C, pl.smem);
    const int64_t key[3] = {one_wave ? 0 : 1, one_wave ? -clusters * pl.C : pl.C, qs};
    if (!best.ok || std::lexicographical_compare(key, key + 3, best_key, best_key + 3)) {
      best = pl;
      std::copy(key, key + 3, best_key);
    }
  }
  return best;
}

// Plans are pure functions of the shape and the tuning: the last few are
// cached (a decode loop repeats the same shape for every layer).
FusedPlan plan_cached(int n_seqs, int n_kv, int n_q, int64_t s_max, int64_t budget, int qsplit, const Tuning& tu) {
  struct Entry {
    int dev, n_seqs, n_kv, n_q, qsplit;
    int64_t s_max, budget;
    unsigned gen;
    FusedPlan plan;
  };
  static std::mutex mu;
  static Entry ring[16];
  static int used = 0, next = 0;
  const int dev = current_device();
  {
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < used; ++i) {
      const Entry& e = ring[i];
      if (e.dev == dev && e.n_seqs == n_seqs && e.n_kv == n_kv && e.n_q == n_q && e.qsplit == qsplit &&
          e.s_max == s_max && e.budget == budget && e.gen == tu.generation)
        return e.plan;
    }
  }
  const FusedPlan pl = plan_fused(n_seqs, n_kv, n_q, s_max, budget, qsplit, tu);
  std::lock_guard<std::mutex> lock(mu);
  ring[next] = Entry{dev, n_seqs, n_kv, n_q, qsplit, s_max, budget, tu.generation, pl};
  next = (next + 1) % 16;
  used = std::min(used + 1, 16);
  return pl;
}

// Plans and launches one fused decode step. Returns kFusedUnsupported when
// the shape does not fit the single-launch kernel (the caller composes
// operators instead).
int fused_decode_launch(adamas_cache* const* caches, int n_seqs, int n_kv, int n_q, int dtype, const void* q,
                        const void* k_new, const void* v_new, int64_t budget, float* out, int32_t* idx,
                        cudaStream_t s, int append = 1, uint32_t* cand = nullptr, int64_t cand_base = 0,
                        int qsplit = 0, const PeerPush* peers = nullptr) {
  const Tuning tu = tuning();
  int64_t s_max = 0;
  for (int i = 0; i < n_seqs; ++i) s_max = std::max(s_max, caches[i]->seq_len + append);
  if (s_max < 1) s_max = 1;
  const FusedPlan pl = plan_cached(n_seqs, n_kv, n_q, s_max, budget, qsplit, tu);
  if (!pl.ok) return kFusedUnsupported;
  FusedParams prm{};
  prm.n_seqs = n_seqs;
  prm.n_kv = n_kv;
  prm.C = pl.C;
  prm.chunk = pl.chunk;
  prm.budget = (int)budget;
  prm.stages = pl.stages;
  prm.exact_encode = tu.exact_encode;
  prm.dbg = tu.dbg;
  prm.pdl = tu.no_pdl ? 0 : 1;
  prm.append = append;
  prm.qsplit = pl.qsplit;
  prm.P = pl.P;
  if (pl.P > 1)
    for (int i = 0; i < n_seqs; ++i)
      if (int rc = ensure_unit_scratch(caches[i], (size_t)n_kv * pl.qsplit * pl.P * pl.G)) return rc;
  prm.cand = cand;
  prm.cand_base = cand_base;
  prm.peers = peers ? *peers : PeerPush{};
  prm.q = q;
  prm.k_new = k_new;
  prm.v_new = v_new;
  prm.out = out;
  prm.idx = idx;
  prm.trace = g_trace;
  for (int i = 0; i < n_seqs; ++i) {
    prm.seq[i].codes = caches[i]->codes;
    prm.seq[i].K = caches[i]->K;
    prm.seq[i].V = caches[i]->V;
    prm.seq[i].status = caches[i]->status;
    prm.seq[i].cap = caches[i]->capacity;
    prm.seq[i].s_old = caches[i]->seq_len;
    prm.seq[i].clean = std::min(caches[i]->dirty_from, caches[i]->seq_len);
    prm.seq[i].xhist = caches[i]->xhist;
    prm.seq[i].xpart = caches[i]->xpart;
    prm.seq[i].xsync = caches[i]->xsync;
  }
  return dtype == ADAMAS_BF16 ? launch_fused_dtype<__nv_bfloat16>(prm, pl.G, pl.C, pl.smem, s)
                              : launch_fused_dtype<float>(prm, pl.G, pl.C, pl.smem, s);
}

}  // namespace

namespace {
constexpr char kAdkvMagic[4] = {'A', 'D', 'K', 'V'};
constexpr uint32_t kAdkvVersion = 1;

float bf16_bits_to_float(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
uint16_t float_to_bf16_bits(float f) {  // round to nearest even (as the device conversion)
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return (uint16_t)((u >> 16) | 0x40);  // NaN
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
template <typename Tp>
void put(std::ofstream& os, Tp v) { os.write(reinterpret_cast<const char*>(&v), sizeof(Tp)); }
template <typename Tp>
bool get(std::ifstream& is, Tp& v) { return (bool)is.read(reinterpret_cast<char*>(&v), sizeof(Tp)); }
}  // namespace

// ------------------------------------------------------------------ f3 harness selection
// Device code store of build_cache for n_inst independent key matrices.
struct adamas_hsel {
  int head_dim = 0, bits = 0, hadamard = 1;
  int64_t n_inst = 0, seq_len = 0;
  uint32_t* planes = nullptr;  // [n_inst * seq_len][2][W] (bits 1, 2)
  uint8_t* bytes = nullptr;    // [n_inst * seq_len][D] (bits 3)
  size_t code_cap = 0;         // bytes allocated for the codes
  void* qcodes = nullptr;      // encoded queries
  size_t q_cap = 0;
  uint32_t* scores = nullptr;
  size_t scores_cap = 0;
  int* status = nullptr;       // device status word (kHselZero | kHselNonFinite)
};

// Peer-memory exchange of the sequence-sharded decode: one mailbox
// per rank in its own HBM, mapped into every rank through CUDA IPC.
//   keys      [world][n_q][budget] u32   slot r written by rank r (phase 1)
//   partials  [world][n_q][132] f32      slot r written by rank r (phase 2)
//   key_flag  [32] u32, part_flag [32] u32   epoch published by rank r
//   arrive    [2] u32 (own launches' CTA arrival counters; padded lines)
struct adamas_mailbox {
  int rank = 0, world = 1, n_q = 0;
  int64_t budget = 0;
  size_t keys_off = 0, part_off = 0, kflag_off = 0, pflag_off = 0, arrive_off = 0, bytes = 0;
  char* base = nullptr;                 // own mailbox (cudaMalloc: IPC-exportable)
  char* peer[kMaxPeers] = {};           // every rank's mailbox as mapped here (peer[rank] = base)
  bool ipc_opened[kMaxPeers] = {};
  int* status = nullptr;
};

// PageSummaries (baselines.cpp:34-54) of n_inst key matrices, device resident.
struct adamas_pages {
  int64_t page_size = 0, n_inst = 0, seq_len = 0;
  int head_dim = 0;
  double* mins = nullptr;  // [n_inst][pages][head_dim]; maxs follows in the same allocation
  double* maxs = nullptr;
  size_t cap = 0;
};

namespace {

bool pow2_dim(int d) { return d >= 2 && d <= kHselMaxDim && (d & (d - 1)) == 0; }

size_t hsel_code_bytes(int D, int bits) {
  return bits == 3 ? (size_t)D : (size_t)2 * hsel_words(D) * sizeof(uint32_t);
}

int hsel_encode(int D, int bits, int hadamard, const double* x, int64_t n_vec, void* codes, int* status,
                cudaStream_t s) {
  if (n_vec == 0) return ADAMAS_OK;
  const int grid = (int)std::min<int64_t>((n_vec + kHselWarps - 1) / kHselWarps, (int64_t)sm_count() * 16);
  uint32_t* pl = bits == 3 ? nullptr : static_cast<uint32_t*>(codes);
  uint8_t* by = bits == 3 ? static_cast<uint8_t*>(codes) : nullptr;
#define HSEL_ENC(E_)                                                                                      \
  do {                                                                                                     \
    if (bits == 1) hsel_encode_kernel<E_, 1><<<grid, kHselWarps * 32, 0, s>>>(x, n_vec, D, hadamard, pl, by, status); \
    else if (bits == 2) hsel_encode_kernel<E_, 2><<<grid, kHselWarps * 32, 0, s>>>(x, n_vec, D, hadamard, pl, by, status); \
    else hsel_encode_kernel<E_, 3><<<grid, kHselWarps * 32, 0, s>>>(x, n_vec, D, hadamard, pl, by, status); \
  } while (0)
  switch (D >= 32 ? D / 32 : 1) {
    case 1: HSEL_ENC(1); break;
    case 2: HSEL_ENC(2); break;
    case 4: HSEL_ENC(4); break;
    case 8: HSEL_ENC(8); break;
    case 16: HSEL_ENC(16); break;
    case 32: HSEL_ENC(32); break;
    default: return fail(ADAMAS_ERR_CONFIG, "hsel: unsupported head_dim");
  }
#undef HSEL_ENC
  return launch_check("hsel_encode_kernel");
}

// Reads and clears the status word; the reference throws ConfigError from
// compute_thresholds for the first bad vector (quantizer.cpp:46-47).
int hsel_status_check(int* status, cudaStream_t s) {
  int h = 0;
  ADAMAS_CUDA(cudaMemcpyAsync(&h, status, sizeof(int), cudaMemcpyDeviceToHost, s));
  ADAMAS_CUDA(cudaStreamSynchronize(s));
  if (h == 0) return ADAMAS_OK;
  ADAMAS_CUDA(cudaMemsetAsync(status, 0, sizeof(int), s));
  if (h & kHselNonFinite) return fail(ADAMAS_ERR_CONFIG, "non-finite input to compute_thresholds");
  return fail(ADAMAS_ERR_CONFIG, "degenerate scale: input vector is all zeros");
}

// Scratch of the harness entry points: stream-ordered allocations from a
// library-owned pool that keeps freed memory (the default pool returns it to
// the driver at every synchronisation, and re-mapping 100 MB buffers costs
// milliseconds per call).
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, s);
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      cudaMemPool_t pool;
      if (cudaError_t e = cudaMemPoolCreate(&pool, &props)) return e;
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      pools[dev] = pool;
    }
  }
  return cudaMallocFromPoolAsync(p, std::max<size_t>(bytes, 8), pools[dev], s);
}

// Grow a pool-backed buffer (freed stream-ordered into the retained pool, so
// handles can be created and destroyed per sweep without driver unmaps).
int pool_grow(void** p, size_t* have, size_t need, cudaStream_t s) {
  if (*have >= need) return ADAMAS_OK;
  if (*p) cudaFreeAsync(*p, s);
  *p = nullptr;
  *have = 0;
  ADAMAS_CUDA(scratch_alloc(p, need, s));
  *have = need;
  return ADAMAS_OK;
}

// dynamic shared memory of seq_select_attend_kernel: the q-head's keys
size_t sel_smem(int n_ranks, int64_t budget) {
  // up to kSelMaxKeys keys (32 KB) on top of ~29 KB static; a function
  // attribute is per device
  static std::mutex mu;
  static bool done[64] = {};
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(mu);
  if (dev >= 0 && dev < 64 && !done[dev]) {
    cudaFuncSetAttribute(seq_select_attend_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSelMaxKeys * 4);
    cudaFuncSetAttribute(seq_select_attend_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSelMaxKeys * 4);
    done[dev] = true;
  }
  return (size_t)n_ranks * budget * sizeof(uint32_t);
}

// Launch with programmatic stream serialization (PDL) unless ADAMAS_NO_PDL:
// the kernel's griddepcontrol.wait orders it after its predecessor, while its
// launch and prologue overlap the predecessor's tail.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = tuning().no_pdl ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

int check_rows(int64_t n_rows, int64_t rows_per_inst, int64_t n_inst) {
  if (n_rows < 0 || rows_per_inst < 1) return fail(ADAMAS_ERR_CONFIG, "rows: bad row count / rows_per_inst");
  if (n_rows > 0 && (n_rows - 1) / rows_per_inst >= n_inst)
    return fail(ADAMAS_ERR_CONFIG, "rows: more query rows than instances * rows_per_inst");
  return ADAMAS_OK;
}

int topk_launch(int mode, const void* scores, int64_t n_rows, int64_t n, int64_t k, int64_t* idx, cudaStream_t s) {
  if (n_rows == 0) return ADAMAS_OK;
  if (n_rows > 0x7fffffff) return fail(ADAMAS_ERR_CONFIG, "topk: too many rows");
  if (mode == 0)
    hsel_topk_kernel<0><<<(unsigned)n_rows, kHselTopkThreads, 0, s>>>(scores, n, k, idx);
  else
    hsel_topk_kernel<1><<<(unsigned)n_rows, kHselTopkThreads, 0, s>>>(scores, n, k, idx);
  return launch_check("hsel_topk_kernel");
}

int dot_scores(const double* q, const double* keys, int64_t n_rows, int64_t rows_per_inst, int64_t S, int D,
               double* out, cudaStream_t s) {
  if (n_rows == 0 || S == 0) return ADAMAS_OK;
  if (n_rows > 65535) return fail(ADAMAS_ERR_CONFIG, "dot: at most 65535 query rows per call");
  const dim3 grid((unsigned)((S + kHselDotTok - 1) / kHselDotTok), (unsigned)n_rows);
  hsel_dot_kernel<<<grid, kHselDotTok, 0, s>>>(q, keys, S, D, rows_per_inst, out);
  return launch_check("hsel_dot_kernel");
}

}  // namespace

extern "C" {

void adamas_debug_trace(unsigned long long* device_buffer) { g_trace = device_buffer; }

int adamas_set_tuning(const int* values, int n) {
  if (n < 0 || (n > 0 && !values)) return fail(ADAMAS_ERR_CONFIG, "set_tuning: bad arguments");
  std::lock_guard<std::mutex> lock(g_tuning_mu);
  Tuning& t = tuning_ref();
  int* fields[] = {&t.qsplit, &t.cluster, &t.P, &t.stages, &t.smem_kb, &t.exact_encode, &t.dbg,
                   &t.no_pdl, &t.composed, &t.require_fused};
  constexpr int kFields = (int)(sizeof(fields) / sizeof(fields[0]));
  if (n > kFields) return fail(ADAMAS_ERR_CONFIG, "set_tuning: too many values");
  for (int i = 0; i < n; ++i) *fields[i] = values[i];
  if (t.P < 1) t.P = 1;
  ++t.generation;
  return ADAMAS_OK;
}

int adamas_get_tuning(int* values, int n) {
  if (n < 0 || (n > 0 && !values)) return fail(ADAMAS_ERR_CONFIG, "get_tuning: bad arguments");
  const Tuning t = tuning();
  const int v[] = {t.qsplit, t.cluster, t.P, t.stages, t.smem_kb, t.exact_encode, t.dbg, t.no_pdl, t.composed,
                   t.require_fused};
  for (int i = 0; i < n && i < (int)(sizeof(v) / sizeof(v[0])); ++i) values[i] = v[i];
  return ADAMAS_OK;
}

const char* adamas_version(void) { return "adamas-b200 0.1 (sm_100a)"; }

const char* adamas_last_error(void) { return g_last_error.c_str(); }

int adamas_cache_create(adamas_cache** out, int n_kv_heads, int head_dim, int bits, int64_t capacity,
                        int kv_dtype) {
  if (out == nullptr) return fail(ADAMAS_ERR_CONFIG, "null output handle");
  *out = nullptr;
  // KvCache ctor checks (kv_cache.cpp:33-34) plus the kernels' specialization.
  if (head_dim == 0) return fail(ADAMAS_ERR_CONFIG, "KvCache: head_dim must be positive");
  if (bits < 1 || bits > 3) return fail(ADAMAS_ERR_CONFIG, "KvCache: bits must be 1, 2, or 3");
  if (head_dim != kHeadDim) return fail(ADAMAS_ERR_CONFIG, "adamas-b200 kernels specialize head_dim = 128");
  if (bits != 2) return fail(ADAMAS_ERR_CONFIG, "adamas-b200 kernels specialize 2-bit codes");
  if (n_kv_heads < 1) return fail(ADAMAS_ERR_CONFIG, "n_kv_heads must be positive");
  if (capacity < 1 || capacity > (int64_t(1) << 31) - 1)
    return fail(ADAMAS_ERR_CONFIG, "capacity must be in [1, 2^31)");
  if (kv_dtype != ADAMAS_F32 && kv_dtype != ADAMAS_BF16) return fail(ADAMAS_ERR_CONFIG, "unknown kv dtype");
  auto* c = new adamas_cache;
  c->n_kv = n_kv_heads;
  c->head_dim = head_dim;
  c->bits = bits;
  c->dtype = kv_dtype;
  c->capacity = capacity;
  cudaGetDevice(&c->device);
  const size_t rows = (size_t)n_kv_heads * (size_t)capacity;
  const size_t kv_bytes = rows * head_dim * elem_size(kv_dtype);
  cudaError_t e = cudaMalloc(&c->K, kv_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&c->V, kv_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&c->codes, rows * 2 * sizeof(uint4));
  if (e == cudaSuccess) e = cudaMalloc(&c->status, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(c->status, 0, sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&c->xsync, (size_t)n_kv_heads * kMaxG * 4 * sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(c->xsync, 0, (size_t)n_kv_heads * kMaxG * 4 * sizeof(int));
  if (e != cudaSuccess) {
    adamas_cache_destroy(c);
    return fail(ADAMAS_ERR_RUNTIME, std::string("cache allocation: ") + cudaGetErrorString(e));
  }
  *out = c;
  return ADAMAS_OK;
}

int adamas_cache_destroy(adamas_cache* c) {
  if (c == nullptr) return ADAMAS_OK;
  cudaFree(c->K);
  cudaFree(c->V);
  cudaFree(c->codes);
  cudaFree(c->status);
  cudaFree(c->xsync);
  cudaFree(c->xhist);
  cudaFree(c->xpart);
  cudaFree(c->scores);
  cudaFree(c->qref);
  cudaFree(c->idx);
  delete c;
  return ADAMAS_OK;
}

int adamas_cache_seq_len(const adamas_cache* c, int64_t* out) {
  if (int rc = check_cache(c)) return rc;
  if (!out) return fail(ADAMAS_ERR_CONFIG, "null output");
  *out = c->seq_len;
  return ADAMAS_OK;
}

int adamas_cache_truncate(adamas_cache* c, int64_t seq_len) {
  if (int rc = check_cache(c)) return rc;
  if (seq_len < 0 || seq_len > c->seq_len) return fail(ADAMAS_ERR_CONFIG, "truncate: out of range");
  c->seq_len = seq_len;
  return ADAMAS_OK;
}

int adamas_cache_buffers(const adamas_cache* c, void** keys, void** values, void** codes) {
  if (int rc = check_cache(c)) return rc;
  if (keys) *keys = c->K;
  if (values) *values = c->V;
  if (codes) *codes = c->codes;
  return ADAMAS_OK;
}

int adamas_cache_status(adamas_cache* c, void* stream, int* status) {
  if (int rc = check_cache(c)) return rc;
  int h = 0;
  ADAMAS_CUDA(cudaMemcpyAsync(&h, c->status, sizeof(int), cudaMemcpyDeviceToHost, as_stream(stream)));
  ADAMAS_CUDA(cudaMemsetAsync(c->status, 0, sizeof(int), as_stream(stream)));
  ADAMAS_CUDA(cudaStreamSynchronize(as_stream(stream)));
  if (status) *status = h;
  return ADAMAS_OK;
}

int adamas_cache_append(adamas_cache* c, const void* keys, const void* values, int64_t n_tokens,
                        void* stream) {
  return do_append(c, keys, values, nullptr, n_tokens, stream);
}

int adamas_cache_append_coded(adamas_cache* c, const void* keys, const void* values,
                              const uint16_t* codes_ref, int64_t n_tokens, void* stream) {
  if (!codes_ref) return fail(ADAMAS_ERR_CONFIG, "append_coded: null codes");
  return do_append(c, keys, values, codes_ref, n_tokens, stream);
}

int adamas_cache_codes_ref(const adamas_cache* c, int64_t start, int64_t n, uint16_t* out_ref,
                           void* stream) {
  if (int rc = check_cache(c)) return rc;
  if (start < 0 || n < 0 || start + n > c->seq_len) return fail(ADAMAS_ERR_CONFIG, "codes_ref: range");
  if (n == 0) return ADAMAS_OK;
  const int64_t vecs = n * c->n_kv;
  const int grid = (int)((vecs + 7) / 8);
  codes_to_ref_kernel<<<grid, 256, 0, as_stream(stream)>>>(c->codes, c->n_kv, c->capacity, start, n, out_ref);
  return launch_check("codes_to_ref_kernel");
}

int adamas_encode_query(const adamas_cache* c, const void* q, int n_q, uint16_t* out_ref, void* stream) {
  if (int rc = check_cache(c)) return rc;
  if (n_q < 1 || !q || !out_ref) return fail(ADAMAS_ERR_CONFIG, "encode_query: bad arguments");
  const int grid = (n_q + kAppendWarps - 1) / kAppendWarps;
  if (c->dtype == ADAMAS_BF16)
    encode_query_kernel<__nv_bfloat16><<<grid, kAppendWarps * 32, 0, as_stream(stream)>>>(
        (const __nv_bfloat16*)q, n_q, out_ref, c->status);
  else
    encode_query_kernel<float><<<grid, kAppendWarps * 32, 0, as_stream(stream)>>>((const float*)q, n_q, out_ref,
                                                                                  c->status);
  return launch_check("encode_query_kernel");
}

int adamas_score(const adamas_cache* c, const uint16_t* q_ref, int n_q, int32_t* scores, void* stream) {
  if (int rc = check_cache(c)) return rc;
  if (int rc = check_heads(c, n_q)) return rc;
  if (!q_ref || !scores) return fail(ADAMAS_ERR_CONFIG, "score: null pointer");
  if (c->seq_len == 0) return ADAMAS_OK;  // estimator: empty cache -> empty scores
  const int64_t per_block = (int64_t)kScoreThreads * kScoreTokensPerThread;
  dim3 grid((unsigned)((c->seq_len + per_block - 1) / per_block), (unsigned)n_q);
  score_kernel<kMetricManhattan><<<grid, kScoreThreads, 0, as_stream(stream)>>>(c->codes, c->capacity, c->seq_len,
                                                                              n_q / c->n_kv, q_ref, scores);
  return launch_check("score_kernel");
}

int adamas_score_metric(const adamas_cache* c, const uint16_t* q_ref, int n_q, int metric, int32_t* scores,
                        void* stream) {
  if (metric == ADAMAS_METRIC_MANHATTAN) return adamas_score(c, q_ref, n_q, scores, stream);
  if (int rc = check_cache(c)) return rc;
  if (int rc = check_heads(c, n_q)) return rc;
  if (!q_ref || !scores) return fail(ADAMAS_ERR_CONFIG, "score_metric: null pointer");
  if (metric != ADAMAS_METRIC_EUCLIDEAN_SQ && metric != ADAMAS_METRIC_HAMMING_1BIT)
    return fail(ADAMAS_ERR_CONFIG, "score_metric: unknown metric");
  if (c->seq_len == 0) return ADAMAS_OK;
  const int64_t per_block = (int64_t)kScoreThreads * kScoreTokensPerThread;
  dim3 grid((unsigned)((c->seq_len + per_block - 1) / per_block), (unsigned)n_q);
  if (metric == ADAMAS_METRIC_EUCLIDEAN_SQ)
    score_kernel<kMetricEuclideanSq><<<grid, kScoreThreads, 0, as_stream(stream)>>>(
        c->codes, c->capacity, c->seq_len, n_q / c->n_kv, q_ref, scores);
  else
    score_kernel<kMetricHamming1><<<grid, kScoreThreads, 0, as_stream(stream)>>>(
        c->codes, c->capacity, c->seq_len, n_q / c->n_kv, q_ref, scores);
  return launch_check("score_kernel");
}

int adamas_topk(const int32_t* scores, int n_rows, int64_t n, int64_t k, int32_t* idx, void* stream) {
  if (n_rows < 1 || n < 0 || k < 0) return fail(ADAMAS_ERR_CONFIG, "topk: bad sizes");
  if (k == 0) return ADAMAS_OK;
  if (!idx || (n > 0 && !scores)) return fail(ADAMAS_ERR_CONFIG, "topk: null pointer");
  if (n > (int64_t(1) << 31) - 1 || k > (int64_t(1) << 31) - 1) return fail(ADAMAS_ERR_CONFIG, "topk: n or k too large");
  topk_kernel<<<n_rows, kTopkThreads, 0, as_stream(stream)>>>(scores, n, k, idx);
  return launch_check("topk_kernel");
}

int adamas_sparse_attention(const adamas_cache* c, const void* q, int n_q, const int32_t* idx, int64_t k,
                            float* out, float* lse, void* stream) {
  if (int rc = check_cache(c)) return rc;
  if (int rc = check_heads(c, n_q)) return rc;
  if (k < 1) return fail(ADAMAS_ERR_CONFIG, "sparse_attention: empty selection");
  if (!q || !idx || !out) return fail(ADAMAS_ERR_CONFIG, "sparse_attention: null pointer");
  const int group = n_q / c->n_kv;
  if (c->dtype == ADAMAS_BF16)
    attend_kernel<__nv_bfloat16><<<n_q, kAttnWarps * 32, 0, as_stream(stream)>>>(
        (const __nv_bfloat16*)c->K, (const __nv_bfloat16*)c->V, c->capacity, c->seq_len, group,
        (const __nv_bfloat16*)q, idx, k, out, lse, c->status);
  else
    attend_kernel<float><<<n_q, kAttnWarps * 32, 0, as_stream(stream)>>>(
        (const float*)c->K, (const float*)c->V, c->capacity, c->seq_len, group, (const float*)q, idx, k, out, lse,
        c->status);
  return launch_check("attend_kernel");
}

int adamas_decode_step_batched(adamas_cache* const* caches, int n_seqs, const void* q, int n_q,
                               const void* k_new, const void* v_new, int64_t budget, float* out, int32_t* idx,
                               void* stream) {  if (!caches || n_seqs < 1) return fail(ADAMAS_ERR_CONFIG, "decode: no caches");
  adamas_cache* c0 = caches[0];
  if (int rc = check_cache(c0)) return rc;
  if (int rc = check_heads(c0, n_q)) return rc;
  if (budget < 1) return fail(ADAMAS_ERR_CONFIG, "decode: budget must be >= 1 (empty selection)");
  if (!q || !k_new || !v_new || !out) return fail(ADAMAS_ERR_CONFIG, "decode: null pointer");
  for (int i = 0; i < n_seqs; ++i) {
    adamas_cache* c = caches[i];
    if (int rc = check_cache(c)) return rc;
    if (c->n_kv != c0->n_kv || c->dtype != c0->dtype)
      return fail(ADAMAS_ERR_CONFIG, "decode: batched caches differ in shape");
    if (c->seq_len + 1 > c->capacity) return fail(ADAMAS_ERR_CONFIG, "decode: cache capacity exceeded");
  }
  const size_t es = elem_size(c0->dtype);
  const size_t q_stride = (size_t)n_q * kHeadDim * es, kv_stride = (size_t)c0->n_kv * kHeadDim * es;
  const Tuning tu = tuning();
  int rc = tu.composed
               ? kFusedUnsupported
               : fused_decode_launch(caches, n_seqs, c0->n_kv, n_q, c0->dtype, q, k_new, v_new, budget, out, idx,
                                     as_stream(stream));
  if (rc == kFusedUnsupported && tu.require_fused)
    return fail(ADAMAS_ERR_CONFIG, "decode: shape not supported by the fused kernel (ADAMAS_REQUIRE_FUSED)");
  if (rc == kFusedUnsupported) {
    // Operator composition (same semantics, several launches).
    for (int i = 0; i < n_seqs; ++i) {
      adamas_cache* c = caches[i];
      const char* qi = (const char*)q + i * q_stride;
      const char* ki = (const char*)k_new + i * kv_stride;
      const char* vi = (const char*)v_new + i * kv_stride;
      float* oi = out + (size_t)i * n_q * kHeadDim;
      if ((rc = do_append(c, ki, vi, nullptr, 1, stream))) return rc;
      if ((rc = grow(&c->scores, &c->scores_elems, (size_t)n_q * c->seq_len))) return rc;
      if (!c->qref) ADAMAS_CUDA(cudaMalloc(&c->qref, 4096 * 16 * sizeof(uint16_t)));
      if (n_q > 4096) return fail(ADAMAS_ERR_CONFIG, "decode: too many heads");
      int32_t* id = idx ? idx + (size_t)i * n_q * budget : nullptr;
      if (!id) {
        if ((rc = grow(&c->idx, &c->idx_elems, (size_t)n_q * budget))) return rc;
        id = c->idx;
      }
      if ((rc = adamas_encode_query(c, qi, n_q, c->qref, stream))) return rc;
      if ((rc = adamas_score(c, c->qref, n_q, c->scores, stream))) return rc;
      if ((rc = adamas_topk(c->scores, n_q, c->seq_len, budget, id, stream))) return rc;
      if ((rc = adamas_sparse_attention(c, qi, n_q, id, budget, oi, nullptr, stream))) return rc;
    }
    return ADAMAS_OK;
  }
  if (rc != ADAMAS_OK) return rc;
  for (int i = 0; i < n_seqs; ++i) {
    caches[i]->dirty_from = caches[i]->seq_len;
    caches[i]->seq_len += 1;
  }
  return ADAMAS_OK;
}

int adamas_decode_step(adamas_cache* c, const void* q, int n_q, const void* k_new, const void* v_new,
                       int64_t budget, float* out, int32_t* idx, void* stream) {
  adamas_cache* arr[1] = {c};
  return adamas_decode_step_batched(arr, 1, q, n_q, k_new, v_new, budget, out, idx, stream);
}

int adamas_seq_local_candidates(adamas_cache* c, const void* q, int n_q, const void* k_new, const void* v_new,
                                int append, int64_t base_index, int64_t budget, uint32_t* cand_keys, void* stream) {
  if (int rc = check_cache(c)) return rc;
  if (int rc = check_heads(c, n_q)) return rc;
  if (budget < 1) return fail(ADAMAS_ERR_CONFIG, "seq_local_candidates: budget must be >= 1");
  if (!q || !cand_keys || (append && (!k_new || !v_new))) return fail(ADAMAS_ERR_CONFIG, "seq_local_candidates: null pointer");
  if (base_index < 0 || base_index + c->seq_len + (append ? 1 : 0) > (int64_t(1) << 23))
    return fail(ADAMAS_ERR_CONFIG, "seq_local_candidates: global token index must stay below 2^23");
  if (append && c->seq_len + 1 > c->capacity) return fail(ADAMAS_ERR_CONFIG, "seq_local_candidates: cache capacity exceeded");
  if (c->seq_len + (append ? 1 : 0) == 0) {  // empty shard: no candidates
    ADAMAS_CUDA(cudaMemsetAsync(cand_keys, 0xff, (size_t)n_q * budget * sizeof(uint32_t), as_stream(stream)));
    return ADAMAS_OK;
  }
  adamas_cache* arr[1] = {c};
  const int rc = fused_decode_launch(arr, 1, c->n_kv, n_q, c->dtype, q, k_new, v_new, budget, nullptr, nullptr,
                                     as_stream(stream), append ? 1 : 0, cand_keys, base_index);
  if (rc == kFusedUnsupported) return fail(ADAMAS_ERR_CONFIG, "seq_local_candidates: shape not supported by the fused kernel");
  if (rc != ADAMAS_OK) return rc;
  if (append) {
    c->dirty_from = c->seq_len;
    c->seq_len += 1;
  }
  return ADAMAS_OK;
}

namespace {
// seq_select_attend_kernel launch for the gathered-keys path; with `out` the
// same launch merges this rank's partial with the others' already in
// `partials` (slot `my_slot` is this rank's).
int launch_select_attend(const adamas_cache* c, const void* q, int n_q, const uint32_t* gathered, int n_ranks,
                         int64_t budget, int64_t total_len, int64_t rank_base, float* partial, int32_t* global_idx,
                         const float* merge_parts, float* out, cudaStream_t st) {
  const int k_eff = (int)std::min<int64_t>(budget, total_len);
  const int group = n_q / c->n_kv;
  if (c->dtype == ADAMAS_BF16)
    ADAMAS_CUDA(launch_pdl(seq_select_attend_kernel<__nv_bfloat16>, dim3(n_q), dim3(kSelThreads),
                           sel_smem(n_ranks, budget), st, (const __nv_bfloat16*)c->K, (const __nv_bfloat16*)c->V,
                           c->capacity, group, (const __nv_bfloat16*)q, gathered, n_ranks, n_q, budget, k_eff,
                           rank_base, c->seq_len, partial, global_idx, PeerPush{}, (const uint32_t*)nullptr, c->status,
                           merge_parts, (const uint32_t*)nullptr, out));
  else
    ADAMAS_CUDA(launch_pdl(seq_select_attend_kernel<float>, dim3(n_q), dim3(kSelThreads), sel_smem(n_ranks, budget),
                           st, (const float*)c->K, (const float*)c->V, c->capacity, group, (const float*)q, gathered,
                           n_ranks, n_q, budget, k_eff, rank_base, c->seq_len, partial, global_idx, PeerPush{},
                           (const uint32_t*)nullptr, c->status, merge_parts, (const uint32_t*)nullptr, out));
  return launch_check("seq_select_attend_kernel");
}

int check_select_attend(const adamas_cache* c, const void* q, int n_q, const uint32_t* gathered, int n_ranks,
                        int64_t budget, int64_t total_len, const float* partial) {
  if (int rc = check_cache(c)) return rc;
  if (int rc = check_heads(c, n_q)) return rc;
  if (n_ranks < 1 || budget < 1 || total_len < 1) return fail(ADAMAS_ERR_CONFIG, "seq_select_attend: bad sizes");
  if ((int64_t)n_ranks * budget > kSelMaxKeys || budget > kSelMaxSurv)
    return fail(ADAMAS_ERR_CONFIG, "seq_select_attend: n_ranks * budget exceeds 8192 (or budget > 2048)");
  if (!q || !gathered || !partial) return fail(ADAMAS_ERR_CONFIG, "seq_select_attend: null pointer");
  return ADAMAS_OK;
}
}  // namespace

int adamas_seq_select_attend(const adamas_cache* c, const void* q, int n_q, const uint32_t* gathered, int n_ranks,
                             int64_t budget, int64_t total_len, int64_t rank_base, float* partial, int32_t* global_idx,
                             void* stream) {
  if (int rc = check_select_attend(c, q, n_q, gathered, n_ranks, budget, total_len, partial)) return rc;
  return launch_select_attend(c, q, n_q, gathered, n_ranks, budget, total_len, rank_base, partial, global_idx,
                              nullptr, nullptr, as_stream(stream));
}

int adamas_seq_select_attend_merge(const adamas_cache* c, const void* q, int n_q, const uint32_t* gathered,
                                   int n_ranks, int64_t budget, int64_t total_len, int64_t rank_base, float* partials,
                                   int my_slot, float* out, int32_t* global_idx, void* stream) {
  if (int rc = check_select_attend(c, q, n_q, gathered, n_ranks, budget, total_len, partials)) return rc;
  if (my_slot < 0 || my_slot >= n_ranks || !out) return fail(ADAMAS_ERR_CONFIG, "seq_select_attend_merge: bad slot / out");
  return launch_select_attend(c, q, n_q, gathered, n_ranks, budget, total_len, rank_base,
                              partials + (int64_t)my_slot * n_q * kPartialStride, global_idx, partials, out,
                              as_stream(stream));
}

int adamas_lse_merge(const float* partials, int n_ranks, int n_q, float* out, void* stream) {
  if (n_ranks < 1 || n_q < 1) return fail(ADAMAS_ERR_CONFIG, "lse_merge: bad sizes");
  if (!partials || !out) return fail(ADAMAS_ERR_CONFIG, "lse_merge: null pointer");
  ADAMAS_CUDA(launch_pdl(lse_merge_kernel, dim3(n_q), dim3(32), 0, as_stream(stream), partials, n_ranks, n_q, out,
                         (const uint32_t*)nullptr, (const uint32_t*)nullptr, (int*)nullptr));
  return launch_check("lse_merge_kernel");
}

// ---------------------------------------------------------------- ADKV snapshots
// The reference's KvCache snapshot (kv_cache.cpp:111-165, README "KV
// snapshots"): magic "ADKV", u32 version (1), u32 seq_len, u32 head_dim,
// u8 bits, f32 keys [seq][d], f32 values [seq][d], u16 code words [seq][d/8].
// One file per kv-head (the reference cache is one head).

int adamas_cache_save_adkv(const adamas_cache* c, int kv_head, const char* path, void* stream) {
  if (int rc = check_cache(c)) return rc;
  if (kv_head < 0 || kv_head >= c->n_kv) return fail(ADAMAS_ERR_CONFIG, "save_adkv: kv_head out of range");
  if (!path) return fail(ADAMAS_ERR_CONFIG, "save_adkv: null path");
  const int64_t n = c->seq_len;
  const size_t es = elem_size(c->dtype);
  std::vector<uint8_t> kraw((size_t)n * kHeadDim * es), vraw(kraw.size());
  std::vector<uint16_t> words((size_t)c->n_kv * n * 16);
  uint16_t* dwords = nullptr;
  cudaStream_t st = as_stream(stream);
  if (n > 0) {
    const char* kb = static_cast<const char*>(c->K) + (size_t)kv_head * c->capacity * kHeadDim * es;
    const char* vb = static_cast<const char*>(c->V) + (size_t)kv_head * c->capacity * kHeadDim * es;
    ADAMAS_CUDA(cudaMemcpyAsync(kraw.data(), kb, kraw.size(), cudaMemcpyDeviceToHost, st));
    ADAMAS_CUDA(cudaMemcpyAsync(vraw.data(), vb, vraw.size(), cudaMemcpyDeviceToHost, st));
    ADAMAS_CUDA(cudaMalloc(&dwords, words.size() * sizeof(uint16_t)));
    int rc = adamas_cache_codes_ref(c, 0, n, dwords, stream);
    if (rc == ADAMAS_OK) {
      cudaError_t e = cudaMemcpyAsync(words.data(), dwords, words.size() * sizeof(uint16_t), cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) rc = fail(ADAMAS_ERR_RUNTIME, std::string("save_adkv: ") + cudaGetErrorString(e));
    }
    cudaFree(dwords);
    if (rc != ADAMAS_OK) return rc;
  }
  std::ofstream os(path, std::ios::binary);
  if (!os) return fail(ADAMAS_ERR_RUNTIME, std::string("save_adkv: cannot open ") + path);
  os.write(kAdkvMagic, 4);
  put(os, kAdkvVersion);
  put(os, (uint32_t)n);
  put(os, (uint32_t)kHeadDim);
  put(os, (uint8_t)2);
  for (const auto* raw : {&kraw, &vraw})
    for (int64_t i = 0; i < n * kHeadDim; ++i) {
      float f;
      if (c->dtype == ADAMAS_BF16) f = bf16_bits_to_float(reinterpret_cast<const uint16_t*>(raw->data())[i]);
      else f = reinterpret_cast<const float*>(raw->data())[i];
      put(os, f);
    }
  const uint16_t* hw = words.data() + (size_t)kv_head * n * 16;
  os.write(reinterpret_cast<const char*>(hw), (size_t)n * 16 * sizeof(uint16_t));
  if (!os) return fail(ADAMAS_ERR_RUNTIME, std::string("save_adkv: write failed for ") + path);
  return ADAMAS_OK;
}

int adamas_cache_load_adkv(adamas_cache* c, const char* const* paths, int n_paths, void* stream) {
  if (int rc = check_cache(c)) return rc;
  if (!paths || n_paths != c->n_kv) return fail(ADAMAS_ERR_CONFIG, "load_adkv: one snapshot per kv-head");
  int64_t n = -1;
  std::vector<std::vector<float>> K(n_paths), V(n_paths);
  std::vector<std::vector<uint16_t>> W(n_paths);
  for (int h = 0; h < n_paths; ++h) {
    std::ifstream is(paths[h], std::ios::binary);
    if (!is) return fail(ADAMAS_ERR_RUNTIME, std::string("load_adkv: cannot open ") + paths[h]);
    char magic[4];
    if (!is.read(magic, 4) || std::memcmp(magic, kAdkvMagic, 4) != 0)
      return fail(ADAMAS_ERR_RUNTIME, "load_adkv: bad magic");
    uint32_t version = 0, seq = 0, d = 0;
    uint8_t bits = 0;
    if (!get(is, version) || version != kAdkvVersion) return fail(ADAMAS_ERR_RUNTIME, "load_adkv: unknown version");
    if (!get(is, seq) || !get(is, d) || !get(is, bits)) return fail(ADAMAS_ERR_RUNTIME, "load_adkv: truncated header");
    if (bits != 1 && bits != 2) return fail(ADAMAS_ERR_RUNTIME, "load_adkv: unsupported code width");
    if (d != kHeadDim || bits != 2)
      return fail(ADAMAS_ERR_CONFIG, "load_adkv: adamas-b200 caches hold head_dim = 128, 2-bit codes");
    if (n >= 0 && (int64_t)seq != n) return fail(ADAMAS_ERR_CONFIG, "load_adkv: snapshots differ in length");
    n = seq;
    K[h].resize((size_t)n * kHeadDim);
    V[h].resize((size_t)n * kHeadDim);
    W[h].resize((size_t)n * 16);
    if (!is.read(reinterpret_cast<char*>(K[h].data()), K[h].size() * 4) ||
        !is.read(reinterpret_cast<char*>(V[h].data()), V[h].size() * 4) ||
        !is.read(reinterpret_cast<char*>(W[h].data()), W[h].size() * 2))
      return fail(ADAMAS_ERR_RUNTIME, "load_adkv: truncated payload");
  }
  if (n <= 0) return ADAMAS_OK;
  if (c->seq_len + n > c->capacity) return fail(ADAMAS_ERR_CONFIG, "load_adkv: cache capacity exceeded");
  const size_t es = elem_size(c->dtype);
  // token-major [n][n_kv][128] (the append layout); codes verbatim (no re-encode)
  std::vector<uint8_t> hk((size_t)n * n_paths * kHeadDim * es), hv(hk.size());
  std::vector<uint16_t> hw((size_t)n * n_paths * 16);
  for (int64_t t = 0; t < n; ++t)
    for (int h = 0; h < n_paths; ++h) {
      const size_t dst = ((size_t)t * n_paths + h) * kHeadDim, src = (size_t)t * kHeadDim;
      for (int e = 0; e < kHeadDim; ++e) {
        if (c->dtype == ADAMAS_BF16) {
          reinterpret_cast<uint16_t*>(hk.data())[dst + e] = float_to_bf16_bits(K[h][src + e]);
          reinterpret_cast<uint16_t*>(hv.data())[dst + e] = float_to_bf16_bits(V[h][src + e]);
        } else {
          reinterpret_cast<float*>(hk.data())[dst + e] = K[h][src + e];
          reinterpret_cast<float*>(hv.data())[dst + e] = V[h][src + e];
        }
      }
      std::memcpy(&hw[((size_t)t * n_paths + h) * 16], &W[h][(size_t)t * 16], 32);
    }
  void *dk = nullptr, *dv = nullptr, *dw = nullptr;
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaMalloc(&dk, hk.size());
  if (e == cudaSuccess) e = cudaMalloc(&dv, hv.size());
  if (e == cudaSuccess) e = cudaMalloc(&dw, hw.size() * 2);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dk, hk.data(), hk.size(), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dv, hv.data(), hv.size(), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dw, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice, st);
  int rc = e == cudaSuccess ? do_append(c, dk, dv, static_cast<const uint16_t*>(dw), n, stream)
                            : fail(ADAMAS_ERR_RUNTIME, std::string("load_adkv: ") + cudaGetErrorString(e));
  if (rc == ADAMAS_OK && (e = cudaStreamSynchronize(st)) != cudaSuccess)
    rc = fail(ADAMAS_ERR_RUNTIME, std::string("load_adkv: ") + cudaGetErrorString(e));
  cudaFree(dk);
  cudaFree(dv);
  cudaFree(dw);
  return rc;
}

void adamas_codes_ref_to_planes(const uint16_t* ref, int64_t n, uint32_t* planes) {
  for (int64_t v = 0; v < n; ++v) {
    const uint8_t* b = reinterpret_cast<const uint8_t*>(ref + v * 16);
    uint32_t* p = planes + v * 8;
    for (int w = 0; w < 8; ++w) p[w] = 0;
    for (int e = 0; e < kHeadDim; ++e) {
      const uint32_t code = (b[e / 4] >> (2 * (e % 4))) & 3u;
      p[e % 4] |= (code & 1u) << (e / 4);
      p[4 + e % 4] |= ((code ^ (code >> 1)) & 1u) << (e / 4);  // x plane: lo ^ hi
    }
  }
}

void adamas_codes_planes_to_ref(const uint32_t* planes, int64_t n, uint16_t* ref) {
  for (int64_t v = 0; v < n; ++v) {
    const uint32_t* p = planes + v * 8;
    uint8_t* b = reinterpret_cast<uint8_t*>(ref + v * 16);
    for (int i = 0; i < 32; ++i) b[i] = 0;
    for (int e = 0; e < kHeadDim; ++e) {
      const uint32_t lo = (p[e % 4] >> (e / 4)) & 1u, x = (p[4 + e % 4] >> (e / 4)) & 1u;
      const uint32_t code = lo | ((lo ^ x) << 1);
      b[e / 4] |= (uint8_t)(code << (2 * (e % 4)));
    }
  }
}

// ------------------------------------------------------------------ f3 harness selection
int adamas_hsel_create(adamas_hsel** out, int head_dim, int bits, int with_hadamard) {
  if (!out) return fail(ADAMAS_ERR_CONFIG, "hsel_create: null out");
  *out = nullptr;
  if (!pow2_dim(head_dim))
    return fail(ADAMAS_ERR_CONFIG, "hsel: head_dim must be a power of two in [2, 1024], got " +
                                       std::to_string(head_dim));
  if (bits < 1 || bits > 3)
    return fail(ADAMAS_ERR_CONFIG, "bucketization width must be 1, 2, or 3 bits, got " + std::to_string(bits));
  auto* h = new adamas_hsel();
  h->head_dim = head_dim;
  h->bits = bits;
  h->hadamard = with_hadamard ? 1 : 0;
  if (scratch_alloc(reinterpret_cast<void**>(&h->status), sizeof(int), 0) != cudaSuccess ||
      cudaMemsetAsync(h->status, 0, sizeof(int), 0) != cudaSuccess || cudaStreamSynchronize(0) != cudaSuccess) {
    delete h;
    return fail(ADAMAS_ERR_RUNTIME, "hsel_create: cudaMalloc failed");
  }
  *out = h;
  return ADAMAS_OK;
}

int adamas_hsel_destroy(adamas_hsel* h) {
  if (!h) return ADAMAS_OK;
  // pool-backed buffers go back to the retained pool (no driver unmap) once
  // every stream's queued work on them is done
  cudaDeviceSynchronize();
  for (void* b : {(void*)h->planes, (void*)h->bytes, h->qcodes, (void*)h->scores, (void*)h->status})
    if (b) cudaFreeAsync(b, 0);
  delete h;
  return ADAMAS_OK;
}

int adamas_hsel_build(adamas_hsel* h, const double* keys, int64_t n_inst, int64_t seq_len, void* stream) {
  if (!h) return fail(ADAMAS_ERR_CONFIG, "null hsel handle");
  if (n_inst < 0 || seq_len < 0) return fail(ADAMAS_ERR_CONFIG, "hsel_build: negative size");
  if (n_inst * seq_len > 0 && !keys) return fail(ADAMAS_ERR_CONFIG, "hsel_build: null keys");
  cudaStream_t s = as_stream(stream);
  const int64_t n_vec = n_inst * seq_len;
  const size_t need = std::max<size_t>(1, (size_t)n_vec * hsel_code_bytes(h->head_dim, h->bits));
  void** buf = h->bits == 3 ? reinterpret_cast<void**>(&h->bytes) : reinterpret_cast<void**>(&h->planes);
  if (int rc = pool_grow(buf, &h->code_cap, need, s)) return rc;
  h->n_inst = n_inst;
  h->seq_len = seq_len;
  if (int rc = hsel_encode(h->head_dim, h->bits, h->hadamard, keys, n_vec, *buf, h->status, s)) return rc;
  return hsel_status_check(h->status, s);
}

int adamas_hsel_codes_ref(const adamas_hsel* h, int64_t first, int64_t n, void* out, void* stream) {
  if (!h) return fail(ADAMAS_ERR_CONFIG, "null hsel handle");
  if (first < 0 || n < 0 || first + n > h->n_inst * h->seq_len)
    return fail(ADAMAS_ERR_CONFIG, "hsel_codes_ref: range out of bounds");
  if (n == 0) return ADAMAS_OK;
  const int W = hsel_words(h->head_dim);
  const int grid = (int)std::min<int64_t>((n * h->head_dim + 255) / 256, (int64_t)sm_count() * 8);
  hsel_codes_ref_kernel<<<grid, 256, 0, as_stream(stream)>>>(
      h->planes ? h->planes + first * 2 * W : nullptr, h->bytes ? h->bytes + first * h->head_dim : nullptr, n,
      h->head_dim, h->bits, out);
  return launch_check("hsel_codes_ref_kernel");
}

int adamas_hsel_select(adamas_hsel* h, const double* queries, int64_t n_rows, int64_t rows_per_inst, int metric,
                       int64_t budget, int64_t* idx, void* stream) {
  if (!h) return fail(ADAMAS_ERR_CONFIG, "null hsel handle");
  if (metric != ADAMAS_METRIC_MANHATTAN && metric != ADAMAS_METRIC_EUCLIDEAN_SQ)
    return fail(ADAMAS_ERR_CONFIG, "hsel_select: metric must be manhattan or euclidean_sq");
  if (budget < 0) return fail(ADAMAS_ERR_CONFIG, "hsel_select: negative budget");
  if (int rc = check_rows(n_rows, rows_per_inst, h->n_inst)) return rc;
  if (n_rows == 0) return ADAMAS_OK;
  if (!queries || (budget > 0 && !idx)) return fail(ADAMAS_ERR_CONFIG, "hsel_select: null pointer");
  // grid.y limit: chunks of whole instances
  const int64_t step = std::max<int64_t>(1, 32768 / rows_per_inst) * rows_per_inst;
  if (std::min(step, n_rows) > 65535) return fail(ADAMAS_ERR_CONFIG, "hsel_select: more than 65535 rows per instance");
  if (step < n_rows) {
    for (int64_t r0 = 0; r0 < n_rows; r0 += step) {
      adamas_hsel sub = *h;  // same codes, shifted instance window; own scratch below
      const int64_t inst0 = r0 / rows_per_inst;
      sub.n_inst = h->n_inst - inst0;
      const size_t cb = hsel_code_bytes(h->head_dim, h->bits) / (h->bits == 3 ? 1 : sizeof(uint32_t));
      if (h->planes) sub.planes = h->planes + (size_t)inst0 * h->seq_len * cb;
      if (h->bytes) sub.bytes = h->bytes + (size_t)inst0 * h->seq_len * cb;
      const int rc = adamas_hsel_select(&sub, queries + r0 * h->head_dim, std::min(step, n_rows - r0), rows_per_inst,
                                        metric, budget, idx + r0 * budget, stream);
      h->qcodes = sub.qcodes; h->q_cap = sub.q_cap; h->scores = sub.scores; h->scores_cap = sub.scores_cap;
      if (rc) return rc;
    }
    return ADAMAS_OK;
  }
  cudaStream_t s = as_stream(stream);
  const int D = h->head_dim;
  if (int rc = pool_grow(&h->qcodes, &h->q_cap, (size_t)n_rows * hsel_code_bytes(D, h->bits), s)) return rc;
  if (int rc = hsel_encode(D, h->bits, h->hadamard, queries, n_rows, h->qcodes, h->status, s)) return rc;
  if (int rc = hsel_status_check(h->status, s)) return rc;
  const int64_t S = h->seq_len;
  if (budget == 0) return ADAMAS_OK;
  if (S == 0) {
    ADAMAS_CUDA(cudaMemsetAsync(idx, 0xff, (size_t)n_rows * budget * sizeof(int64_t), s));
    return ADAMAS_OK;
  }
  void* sc = h->scores;
  if (int rc = pool_grow(&sc, &h->scores_cap, (size_t)n_rows * S * sizeof(uint32_t), s)) return rc;
  h->scores = static_cast<uint32_t*>(sc);
  const dim3 grid((unsigned)((S + kHselScoreThreads - 1) / kHselScoreThreads), (unsigned)n_rows);
  const uint32_t* qp = h->bits == 3 ? nullptr : static_cast<const uint32_t*>(h->qcodes);
  const uint8_t* qb = h->bits == 3 ? static_cast<const uint8_t*>(h->qcodes) : nullptr;
#define HSEL_SCORE(B_, M_) \
  hsel_score_kernel<B_, M_><<<grid, kHselScoreThreads, 0, s>>>(h->planes, h->bytes, qp, qb, S, D, rows_per_inst, h->scores)
  const bool l1 = metric == ADAMAS_METRIC_MANHATTAN;
  if (h->bits == 1) HSEL_SCORE(1, kMetricManhattan);
  else if (h->bits == 2) { if (l1) HSEL_SCORE(2, kMetricManhattan); else HSEL_SCORE(2, kMetricEuclideanSq); }
  else { if (l1) HSEL_SCORE(3, kMetricManhattan); else HSEL_SCORE(3, kMetricEuclideanSq); }
#undef HSEL_SCORE
  if (int rc = launch_check("hsel_score_kernel")) return rc;
  return topk_launch(0, h->scores, n_rows, S, budget, idx, s);
}

int adamas_dot_topk(const double* queries, const double* keys, int64_t n_rows, int64_t rows_per_inst, int64_t n_inst,
                    int64_t seq_len, int head_dim, int64_t k, int64_t* idx, double* scores, void* stream) {
  if (head_dim < 1 || head_dim > kHselMaxDim) return fail(ADAMAS_ERR_CONFIG, "dot_topk: head_dim out of range");
  if (k < 0 || seq_len < 0) return fail(ADAMAS_ERR_CONFIG, "dot_topk: negative size");
  if (int rc = check_rows(n_rows, rows_per_inst, n_inst)) return rc;
  if (n_rows == 0) return ADAMAS_OK;
  cudaStream_t s = as_stream(stream);
  double* sc = scores;
  if (!sc) ADAMAS_CUDA(scratch_alloc(reinterpret_cast<void**>(&sc), (size_t)n_rows * seq_len * 8, s));
  int rc = dot_scores(queries, keys, n_rows, rows_per_inst, seq_len, head_dim, sc, s);
  if (!rc && k > 0) rc = topk_launch(1, sc, n_rows, seq_len, k, idx, s);
  if (!scores) cudaFreeAsync(sc, s);
  return rc;
}

int adamas_topk_f64(const double* scores, int64_t n_rows, int64_t n, int64_t k, int64_t* idx, void* stream) {
  if (n_rows < 0 || n < 0 || k < 0) return fail(ADAMAS_ERR_CONFIG, "topk_f64: negative size");
  if (n_rows == 0 || k == 0) return ADAMAS_OK;
  if (!scores || !idx) return fail(ADAMAS_ERR_CONFIG, "topk_f64: null pointer");
  return topk_launch(1, scores, n_rows, n, k, idx, as_stream(stream));
}

int adamas_pages_create(adamas_pages** out, int64_t page_size, int head_dim) {
  if (!out) return fail(ADAMAS_ERR_CONFIG, "pages_create: null out");
  *out = nullptr;
  if (page_size < 1) return fail(ADAMAS_ERR_CONFIG, "PageSummaries: page_size must be positive");
  if (head_dim < 1 || head_dim > kHselMaxDim) return fail(ADAMAS_ERR_CONFIG, "PageSummaries: head_dim out of range");
  auto* p = new adamas_pages();
  p->page_size = page_size;
  p->head_dim = head_dim;
  *out = p;
  return ADAMAS_OK;
}

int adamas_pages_destroy(adamas_pages* p) {
  if (!p) return ADAMAS_OK;
  cudaDeviceSynchronize();
  if (p->mins) cudaFreeAsync(p->mins, 0);
  delete p;
  return ADAMAS_OK;
}

int adamas_pages_build(adamas_pages* p, const double* keys, int64_t n_inst, int64_t seq_len, void* stream) {
  if (!p) return fail(ADAMAS_ERR_CONFIG, "null pages handle");
  if (n_inst < 0 || seq_len < 0) return fail(ADAMAS_ERR_CONFIG, "pages_build: negative size");
  const int64_t P = (seq_len + p->page_size - 1) / p->page_size;
  const size_t half = (size_t)n_inst * P * p->head_dim;
  void* buf = p->mins;
  if (int rc = pool_grow(&buf, &p->cap, std::max<size_t>(16, 2 * half * sizeof(double)), as_stream(stream))) return rc;
  p->mins = static_cast<double*>(buf);
  p->maxs = p->mins + half;
  p->n_inst = n_inst;
  p->seq_len = seq_len;
  if (half == 0) return ADAMAS_OK;
  if (!keys) return fail(ADAMAS_ERR_CONFIG, "pages_build: null keys");
  const int g = (int)std::min<int64_t>(((int64_t)half + 255) / 256, (int64_t)sm_count() * 16);
  hsel_page_summary_kernel<<<g, 256, 0, as_stream(stream)>>>(keys, n_inst, seq_len, p->head_dim, p->page_size,
                                                              p->mins, p->maxs);
  return launch_check("hsel_page_summary_kernel");
}

int adamas_pages_select(adamas_pages* p, const double* queries, int64_t n_rows, int64_t rows_per_inst, int64_t budget,
                        int64_t* idx, int64_t* counts, void* stream) {
  if (!p) return fail(ADAMAS_ERR_CONFIG, "null pages handle");
  if (budget < 0) return fail(ADAMAS_ERR_CONFIG, "page_select: negative budget");
  if (int rc = check_rows(n_rows, rows_per_inst, p->n_inst)) return rc;
  if (n_rows == 0 || budget == 0) return ADAMAS_OK;
  if (n_rows > 65535) return fail(ADAMAS_ERR_CONFIG, "page_select: at most 65535 query rows per call");
  if (!queries || !idx || !counts) return fail(ADAMAS_ERR_CONFIG, "page_select: null pointer");
  cudaStream_t s = as_stream(stream);
  const int64_t S = p->seq_len, ps_ = p->page_size;
  if (budget >= S) {  // baselines.cpp:74-78: everything
    hsel_topk_kernel<0><<<(unsigned)n_rows, kHselTopkThreads, 0, s>>>(nullptr, S, budget, idx);
    if (int rc = launch_check("hsel_topk_kernel")) return rc;
    hsel_fill_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, s>>>(counts, n_rows, S);
    return launch_check("hsel_fill_kernel");
  }
  if (budget % ps_ != 0) return fail(ADAMAS_ERR_CONFIG, "page_select: budget must be a multiple of the page size");
  const int64_t P = (S + ps_ - 1) / ps_, kp = budget / ps_;
  double* sc = nullptr;
  int64_t* pages = nullptr;
  ADAMAS_CUDA(scratch_alloc(reinterpret_cast<void**>(&sc), (size_t)n_rows * P * 8, s));
  ADAMAS_CUDA(scratch_alloc(reinterpret_cast<void**>(&pages), (size_t)n_rows * kp * 8, s));
  const dim3 grid((unsigned)((P + kHselPageTile - 1) / kHselPageTile), (unsigned)n_rows);
  hsel_page_score_kernel<<<grid, kHselPageTile, 0, s>>>(queries, p->mins, p->maxs, rows_per_inst, P, p->head_dim, sc);
  int rc = launch_check("hsel_page_score_kernel");
  if (!rc) rc = topk_launch(1, sc, n_rows, P, kp, pages, s);
  if (!rc) {
    hsel_page_expand_kernel<<<(unsigned)n_rows, 256, 0, s>>>(pages, kp, S, ps_, budget, idx, counts);
    rc = launch_check("hsel_page_expand_kernel");
  }
  cudaFreeAsync(sc, s);
  cudaFreeAsync(pages, s);
  return rc;
}

int adamas_page_select(const double* queries, const double* keys, int64_t n_rows, int64_t rows_per_inst,
                       int64_t n_inst, int64_t seq_len, int head_dim, int64_t page_size, int64_t budget, int64_t* idx,
                       int64_t* counts, void* stream) {
  adamas_pages* p = nullptr;
  if (int rc = adamas_pages_create(&p, page_size, head_dim)) return rc;
  int rc = adamas_pages_build(p, keys, n_inst, seq_len, stream);
  if (!rc) rc = adamas_pages_select(p, queries, n_rows, rows_per_inst, budget, idx, counts, stream);
  if (!rc) rc = cudaStreamSynchronize(as_stream(stream)) == cudaSuccess ? ADAMAS_OK : fail(ADAMAS_ERR_RUNTIME, "page_select: sync");
  adamas_pages_destroy(p);
  return rc;
}

int adamas_attention_f64(const double* queries, const double* keys, const double* values, int64_t n_rows,
                         int64_t rows_per_inst, int64_t n_inst, int64_t seq_len, int head_dim, const int64_t* idx,
                         int64_t idx_stride, const int64_t* counts, double* out, void* stream) {
  if (head_dim < 1 || head_dim > kHselMaxDim) return fail(ADAMAS_ERR_CONFIG, "attention_f64: head_dim out of range");
  if (int rc = check_rows(n_rows, rows_per_inst, n_inst)) return rc;
  if (n_rows == 0) return ADAMAS_OK;
  if (seq_len < 1 || (idx && idx_stride < 1)) return fail(ADAMAS_ERR_CONFIG, "full_attention: no keys to attend over");
  if (n_rows > 0x7fffffff) return fail(ADAMAS_ERR_CONFIG, "attention_f64: too many rows");
  cudaStream_t s = as_stream(stream);
  const int64_t n_max = idx ? idx_stride : seq_len;
  double* lg = nullptr;
  ADAMAS_CUDA(scratch_alloc(reinterpret_cast<void**>(&lg), (size_t)n_rows * n_max * 8, s));
  hsel_attention_kernel<<<(unsigned)n_rows, kHselAttnThreads, 0, s>>>(queries, keys, values, seq_len, head_dim,
                                                                       rows_per_inst, idx, idx_stride, counts, lg,
                                                                       n_max, out);
  const int rc = launch_check("hsel_attention_kernel");
  cudaFreeAsync(lg, s);
  return rc;
}

// ---------------------------------------------------------------- peer-memory sequence sharding
namespace {
PeerPush key_push(const adamas_mailbox* m) {
  PeerPush pp{};
  pp.n = m->world;
  for (int r = 0; r < m->world; ++r) {
    pp.keys[r] = reinterpret_cast<uint32_t*>(m->peer[r] + m->keys_off) + (size_t)m->rank * m->n_q * m->budget;
    pp.flag[r] = reinterpret_cast<uint32_t*>(m->peer[r] + m->kflag_off) + m->rank;
  }
  pp.arrive = reinterpret_cast<unsigned int*>(m->base + m->arrive_off);
  pp.epoch = reinterpret_cast<uint32_t*>(m->base + m->arrive_off) + 64;
  pp.bump = 1;
  return pp;
}
PeerPush part_push(const adamas_mailbox* m) {
  PeerPush pp{};
  pp.n = m->world;
  for (int r = 0; r < m->world; ++r) {
    pp.part[r] = reinterpret_cast<float*>(m->peer[r] + m->part_off) + (size_t)m->rank * m->n_q * kPartialStride;
    pp.flag[r] = reinterpret_cast<uint32_t*>(m->peer[r] + m->pflag_off) + m->rank;
  }
  pp.arrive = reinterpret_cast<unsigned int*>(m->base + m->arrive_off) + 32;
  pp.epoch = reinterpret_cast<uint32_t*>(m->base + m->arrive_off) + 64;
  pp.bump = 0;
  return pp;
}
int check_mailbox(const adamas_mailbox* m) {
  if (!m) return fail(ADAMAS_ERR_CONFIG, "null mailbox");
  for (int r = 0; r < m->world; ++r)
    if (!m->peer[r]) return fail(ADAMAS_ERR_CONFIG, "mailbox: not connected to every rank");
  return ADAMAS_OK;
}
}  // namespace

int adamas_mailbox_create(adamas_mailbox** out, int rank, int world, int n_q_heads, int64_t budget) {
  if (!out) return fail(ADAMAS_ERR_CONFIG, "mailbox_create: null out");
  *out = nullptr;
  if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world)
    return fail(ADAMAS_ERR_CONFIG, "mailbox_create: world must be 1..8 and 0 <= rank < world");
  if (n_q_heads < 1 || budget < 1 || (int64_t)world * budget > kSelMaxKeys || budget > kSelMaxSurv)
    return fail(ADAMAS_ERR_CONFIG, "mailbox_create: world * budget must be <= 8192 (budget <= 2048)");
  auto* m = new adamas_mailbox();
  m->rank = rank;
  m->world = world;
  m->n_q = n_q_heads;
  m->budget = budget;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  m->keys_off = 0;
  m->part_off = al((size_t)world * n_q_heads * budget * 4);
  m->kflag_off = m->part_off + al((size_t)world * n_q_heads * kPartialStride * 4);
  m->pflag_off = m->kflag_off + 256;
  m->arrive_off = m->pflag_off + 256;
  m->bytes = m->arrive_off + 512;  // arrive[0] keys, arrive[32] partials, [64] step epoch
  if (cudaMalloc(&m->base, m->bytes) != cudaSuccess || cudaMemset(m->base, 0, m->bytes) != cudaSuccess ||
      cudaMalloc(&m->status, sizeof(int)) != cudaSuccess || cudaMemset(m->status, 0, sizeof(int)) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(m->base);
    cudaFree(m->status);
    delete m;
    return fail(ADAMAS_ERR_RUNTIME, "mailbox_create: device allocation failed");
  }
  m->peer[rank] = m->base;
  *out = m;
  return ADAMAS_OK;
}

int adamas_mailbox_ipc_handle(const adamas_mailbox* m, void* handle) {
  if (!m || !handle) return fail(ADAMAS_ERR_CONFIG, "mailbox_ipc_handle: null pointer");
  cudaIpcMemHandle_t h;
  ADAMAS_CUDA(cudaIpcGetMemHandle(&h, m->base));
  std::memcpy(handle, &h, sizeof(h));
  return ADAMAS_OK;
}

int adamas_mailbox_connect(adamas_mailbox* m, const void* handles) {
  if (!m || !handles) return fail(ADAMAS_ERR_CONFIG, "mailbox_connect: null pointer");
  for (int r = 0; r < m->world; ++r) {
    if (r == m->rank || m->peer[r]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + (size_t)r * ADAMAS_IPC_HANDLE_BYTES, sizeof(h));
    void* ptr = nullptr;
    ADAMAS_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    m->peer[r] = static_cast<char*>(ptr);
    m->ipc_opened[r] = true;
  }
  return ADAMAS_OK;
}

int adamas_mailbox_connect_local(adamas_mailbox* const* boxes, int world) {
  if (!boxes || world < 1 || world > kMaxPeers) return fail(ADAMAS_ERR_CONFIG, "mailbox_connect_local: bad arguments");
  for (int i = 0; i < world; ++i) {
    if (!boxes[i] || boxes[i]->world != world || boxes[i]->rank != i)
      return fail(ADAMAS_ERR_CONFIG, "mailbox_connect_local: boxes must be ranks 0..world-1 of one world");
  }
  for (int i = 0; i < world; ++i)
    for (int r = 0; r < world; ++r) boxes[i]->peer[r] = boxes[r]->base;
  return ADAMAS_OK;
}

int adamas_mailbox_status(adamas_mailbox* m, int* status) {
  if (!m || !status) return fail(ADAMAS_ERR_CONFIG, "mailbox_status: null pointer");
  ADAMAS_CUDA(cudaMemcpy(status, m->status, sizeof(int), cudaMemcpyDeviceToHost));
  return ADAMAS_OK;
}

int adamas_mailbox_destroy(adamas_mailbox* m) {
  if (!m) return ADAMAS_OK;
  cudaDeviceSynchronize();
  for (int r = 0; r < m->world; ++r)
    if (m->ipc_opened[r]) cudaIpcCloseMemHandle(m->peer[r]);
  cudaFree(m->base);
  cudaFree(m->status);
  delete m;
  return ADAMAS_OK;
}

int adamas_seq_p2p_local(adamas_cache* c, adamas_mailbox* m, const void* q, int n_q, const void* k_new,
                         const void* v_new, int append, int64_t base_index, void* stream) {
  if (int rc = check_cache(c)) return rc;
  if (int rc = check_mailbox(m)) return rc;
  if (int rc = check_heads(c, n_q)) return rc;
  if (n_q != m->n_q) return fail(ADAMAS_ERR_CONFIG, "seq_p2p_local: n_q differs from the mailbox's");
  if (!q || (append && (!k_new || !v_new))) return fail(ADAMAS_ERR_CONFIG, "seq_p2p_local: null pointer");
  if (base_index < 0 || base_index + c->seq_len + (append ? 1 : 0) > (int64_t(1) << 23))
    return fail(ADAMAS_ERR_CONFIG, "seq_p2p_local: global token index must stay below 2^23");
  if (append && c->seq_len + 1 > c->capacity) return fail(ADAMAS_ERR_CONFIG, "seq_p2p_local: cache capacity exceeded");
  cudaStream_t s = as_stream(stream);
  const PeerPush pp = key_push(m);  // the launch's last CTA advances the device-side step epoch
  if (c->seq_len + (append ? 1 : 0) == 0) {  // empty shard: no candidates, still publish
    peer_empty_keys_kernel<<<1, 256, 0, s>>>(pp, (int64_t)n_q * m->budget);
    return launch_check("peer_empty_keys_kernel");
  }
  adamas_cache* arr[1] = {c};
  const int rc = fused_decode_launch(arr, 1, c->n_kv, n_q, c->dtype, q, k_new, v_new, m->budget, nullptr, nullptr, s,
                                     append ? 1 : 0, pp.keys[m->rank], base_index, 0, &pp);
  if (rc == kFusedUnsupported) return fail(ADAMAS_ERR_CONFIG, "seq_p2p_local: shape not supported by the fused kernel");
  if (rc != ADAMAS_OK) return rc;
  if (append) {
    c->dirty_from = c->seq_len;
    c->seq_len += 1;
  }
  return ADAMAS_OK;
}

namespace {
int p2p_select_attend(const adamas_cache* c, adamas_mailbox* m, const void* q, int n_q, int64_t total_len,
                      int64_t rank_base, int32_t* global_idx, float* merge_out, void* stream) {
  if (int rc = check_cache(c)) return rc;
  if (int rc = check_mailbox(m)) return rc;
  if (int rc = check_heads(c, n_q)) return rc;
  if (n_q != m->n_q || total_len < 1 || !q) return fail(ADAMAS_ERR_CONFIG, "seq_p2p_select_attend: bad arguments");
  const int k_eff = (int)std::min<int64_t>(m->budget, total_len);
  const int group = n_q / c->n_kv;
  const PeerPush pp = part_push(m);
  const uint32_t* keys = reinterpret_cast<const uint32_t*>(m->base + m->keys_off);
  const uint32_t* kflags = reinterpret_cast<const uint32_t*>(m->base + m->kflag_off);
  const PeerPush& pk = pp;
  // merge_out: the merge runs in the same launch (one CTA per q-head, all resident)
  const float* parts = reinterpret_cast<const float*>(m->base + m->part_off);
  const uint32_t* pflags = reinterpret_cast<const uint32_t*>(m->base + m->pflag_off);
  const size_t dyn = sel_smem(m->world, m->budget);
  const float* mp = merge_out ? parts : nullptr;
  const uint32_t* mf = merge_out ? pflags : nullptr;
  if (c->dtype == ADAMAS_BF16)
    ADAMAS_CUDA(launch_pdl(seq_select_attend_kernel<__nv_bfloat16>, dim3(n_q), dim3(kSelThreads), dyn,
                           as_stream(stream), (const __nv_bfloat16*)c->K, (const __nv_bfloat16*)c->V, c->capacity,
                           group, (const __nv_bfloat16*)q, keys, m->world, n_q, m->budget, k_eff, rank_base,
                           c->seq_len, (float*)nullptr, global_idx, pk, kflags, m->status, mp, mf, merge_out));
  else
    ADAMAS_CUDA(launch_pdl(seq_select_attend_kernel<float>, dim3(n_q), dim3(kSelThreads), dyn, as_stream(stream),
                           (const float*)c->K, (const float*)c->V, c->capacity, group, (const float*)q, keys, m->world,
                           n_q, m->budget, k_eff, rank_base, c->seq_len, (float*)nullptr, global_idx, pk, kflags,
                           m->status, mp, mf, merge_out));
  return launch_check("seq_select_attend_kernel");
}

}  // namespace

int adamas_seq_p2p_select_attend(const adamas_cache* c, adamas_mailbox* m, const void* q, int n_q, int64_t total_len,
                                 int64_t rank_base, int32_t* global_idx, void* stream) {
  return p2p_select_attend(c, m, q, n_q, total_len, rank_base, global_idx, nullptr, stream);
}

int adamas_seq_p2p_merge(adamas_mailbox* m, float* out, void* stream) {
  if (int rc = check_mailbox(m)) return rc;
  if (!out) return fail(ADAMAS_ERR_CONFIG, "seq_p2p_merge: null out");
  const float* parts = reinterpret_cast<const float*>(m->base + m->part_off);
  const uint32_t* pflags = reinterpret_cast<const uint32_t*>(m->base + m->pflag_off);
  const uint32_t* epoch = reinterpret_cast<const uint32_t*>(m->base + m->arrive_off) + 64;
  ADAMAS_CUDA(launch_pdl(lse_merge_kernel, dim3(m->n_q), dim3(32), 0, as_stream(stream), parts, m->world, m->n_q, out,
                         pflags, epoch, m->status));
  return launch_check("lse_merge_kernel");
}

int adamas_seq_step_p2p(adamas_cache* c, adamas_mailbox* m, const void* q, int n_q, const void* k_new,
                        const void* v_new, int append, int64_t base_index, int64_t total_len, float* out,
                        int32_t* global_idx, void* stream) {
  if (!out) return fail(ADAMAS_ERR_CONFIG, "seq_step_p2p: null out");
  if (int rc = adamas_seq_p2p_local(c, m, q, n_q, k_new, v_new, append, base_index, stream)) return rc;
  // merge in the same launch only when every select CTA is resident at once
  // (its CTAs wait for each other's partials): occupancy, not just the SM count
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, int>, int>> resident;  // ((device, dtype) -> CTAs per SM)
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    const int dev = current_device();
    for (auto& e : resident)
      if (e.first.first == dev && e.first.second == c->dtype) per_sm = e.second;
    if (per_sm == 0) {
      const size_t dyn = sel_smem(m->world, m->budget);
      cudaError_t e = c->dtype == ADAMAS_BF16
                          ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, seq_select_attend_kernel<__nv_bfloat16>,
                                                                         kSelThreads, dyn)
                          : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, seq_select_attend_kernel<float>,
                                                                         kSelThreads, dyn);
      if (e != cudaSuccess || per_sm < 0) per_sm = 0;
      resident.push_back({{dev, c->dtype}, per_sm});
    }
  }
  if ((int64_t)n_q <= (int64_t)per_sm * sm_count())
    return p2p_select_attend(c, m, q, n_q, total_len, base_index, global_idx, out, stream);
  if (int rc = adamas_seq_p2p_select_attend(c, m, q, n_q, total_len, base_index, global_idx, stream)) return rc;
  return adamas_seq_p2p_merge(m, out, stream);
}

}  // extern "C"

