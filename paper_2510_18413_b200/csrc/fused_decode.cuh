// fused_decode.cuh — one Adamas decode step of one layer in ONE launch.
//
// Work unit = (sequence, kv-head) with its G = n_q / n_kv query heads. A
// thread-block cluster of C CTAs owns a unit; CTA rank r owns the contiguous
// token range [r * chunk, min(S, (r + 1) * chunk)) where S includes the token
// appended by this very step (Alg. 1: update before estimate).
//
//   prologue  one lane starts the bulk-copy (TMA engine) stream of the rank's
//             lo/hi code planes into a deep shared-memory ring; warps 0..G-1
//             encode the G query heads (fp64 FWHT + RMS thresholds, bit-exact)
//             meanwhile; the rank owning position S-1 encodes the new key and
//             appends (k, v, code) to the cache (kv_cache.cpp:62-71)
//   scan      each thread turns two tokens per stage into G exact distances
//             (estimator.cpp:45-59), kept as u16 in shared memory and counted
//             in a per-CTA 512-bin histogram per q-head
//   select    cluster barrier; every rank reads the C histograms over DSMEM,
//             derives the global threshold T (k-th smallest distance), how many
//             ties at T earlier ranks take and its own output offset; then an
//             order-preserving warp compaction of its own tokens (top_k
//             semantics, estimator.cpp:75-90: (score, index) order)
//   attend    each rank attends over its own selected rows (gather of K, V by
//             index, fp32 online softmax), pushes (m, l, o[128]) into the
//             merging rank's shared memory over DSMEM; cluster barrier;
//             log-sum-exp merge -> out (attention.cpp:8-45 semantics)
//
// Indices are bit-exact by construction: the selection is computed from the
// exact integer distances with the reference's total order, no approximation.
#pragma once
#include "ops.cuh"

namespace adamas_dev {

constexpr int kFusedThreads = 512;
constexpr int kFusedWarps = kFusedThreads / 32;
constexpr int kStageTok = 1024;  // tokens per bulk-copy stage: 2 x 16 KB planes
constexpr int kStageBytes = kStageTok * 32;
constexpr int kMaxStages = 16;   // ring depth cap (runtime: FusedParams::stages)
constexpr int kHistBins = 512;   // 2-bit L1 distances at d = 128 are <= 384
constexpr int kMaxG = 8;
constexpr int kMaxSeqs = 64;
constexpr int kPartStride = 132;  // floats per partial: m, l, pad, pad, o[128]
constexpr int kFusedUnsupported = -100;

struct FusedSeq {
  uint4* codes;  // this sequence's cache: [n_kv][2 planes][cap] x 16 B
  void* K;       // [n_kv][cap][128]
  void* V;
  int64_t cap;
  int64_t s_old;  // tokens in the cache before this step's append
};

struct FusedParams {
  int n_seqs, n_kv, C, chunk, budget, stages;
  int exact_encode;  // 1: always the sequential fp64 sum (diagnostics / tests)
  int dbg;           // diagnostics only: bit0 no L2 prefetch, bit1 no idx stores, bit2 skip pass 2
  const void* q;      // [n_seqs][n_q][128]
  const void* k_new;  // [n_seqs][n_kv][128]
  const void* v_new;
  float* out;    // [n_seqs][n_q][128]
  int32_t* idx;  // [n_seqs][n_q][budget] or null
  int* status;
  unsigned long long* trace;  // optional per-CTA phase timestamps (diagnostics)
  FusedSeq seq[kMaxSeqs];
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long global_ns() {
  // SM cycle counter: exact within a CTA (phase durations), not across SMs
  return (unsigned long long)clock64();
}
// BAR.SYNC on sm_100 blocks lazily (at the next access to barrier-protected
// state), so a stamp taken right after __syncthreads() would record the
// barrier's issue, not its release: the volatile shared load forces the wait.
#define ADAMAS_TRACE(i)                                                              \
  do {                                                                               \
    if (p.trace != nullptr && threadIdx.x == 0) {                                    \
      __shared__ volatile int trace_sink;                                            \
      const int sink = trace_sink;                                                   \
      p.trace[blockIdx.x * 16 + (i)] = global_ns() + (unsigned long long)(sink & 0); \
    }                                                                                \
  } while (0)

// Dynamic shared-memory carve-up, identical on host and device.
struct FusedSmem {
  uint32_t stage, dist, gmin, hist, hist_all, sel, inbox, wpart, qf, qcode, sq, bars, total;
  __host__ __device__ static uint32_t align(uint32_t x, uint32_t a) { return (x + a - 1u) & ~(a - 1u); }
  __host__ __device__ FusedSmem(int G, int C, int chunk, int selcap, int stages) {
    uint32_t o = 0;
    stage = o; o += (uint32_t)stages * kStageBytes;
    dist = o;  o = align(o + (uint32_t)G * chunk * 2, 16);
    gmin = o;  o = align(o + (uint32_t)G * (chunk / 32) * 2, 16);  // min distance per 32-token group
    hist = o;  o += (uint32_t)G * kHistBins * 4;
    hist_all = o; o += (uint32_t)C * G * kHistBins * 2;  // u16 histograms received from every rank
    sel = o;   o = align(o + (uint32_t)G * selcap * 4, 16);
    inbox = o; o += (uint32_t)C * G * kPartStride * 4;
    wpart = o; o += kFusedWarps * kPartStride * 4;
    qf = o;    o += (uint32_t)G * kHeadDim * 4;  // the G query heads as fp32
    o = align(o, 32);
    qcode = o; o += (uint32_t)(G + 1) * 32;
    sq = o;    o += (uint32_t)(G + 1) * kHeadDim * 8;
    bars = o;  o += (kMaxStages + 2) * 8;  // ring, hist exchange, partial exchange
    total = o;
  }
};

// Exclusive CTA-wide scan (thread order) of N ints per thread.
template <int N>
__device__ __forceinline__ void block_scan(int (&v)[N], int (&excl)[N], int (&total)[N], int* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl[N];
#pragma unroll
  for (int i = 0; i < N; ++i) incl[i] = v[i];
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int o = __shfl_up_sync(kFull, incl[i], m);
      if (lane >= m) incl[i] += o;
    }
  }
  if (lane == 31) {
#pragma unroll
    for (int i = 0; i < N; ++i) scratch[i * kFusedWarps + warp] = incl[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    int before = 0, sum = 0;
    for (int w = 0; w < kFusedWarps; ++w) {
      const int x = scratch[i * kFusedWarps + w];
      before += w < warp ? x : 0;
      sum += x;
    }
    excl[i] = before + incl[i] - v[i];
    total[i] = sum;
  }
  __syncthreads();
}

template <typename T, int G>
__global__ void __launch_bounds__(kFusedThreads, 1) fused_decode_kernel(const __grid_constant__ FusedParams p) {
  static_assert(G >= 1 && G <= kMaxG && (kFusedWarps % G) == 0, "G must divide the warp count");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ int scan_scratch[2 * kMaxG * kFusedWarps];
  __shared__ int sc[kMaxG][4];  // per q-head: T, below, pre_lt, pre_eq
  __shared__ int nsel[kMaxG];
  const int C = p.C;
  const int rank = (int)cluster_rank();
  const int unit = blockIdx.x / C;
  const int si = unit / p.n_kv, hk = unit % p.n_kv;
  const int n_q = p.n_kv * G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  const int64_t cap = p.seq[si].cap;
  const int64_t s_old = p.seq[si].s_old;
  const int64_t S = s_old + 1;
  const int64_t start = (int64_t)rank * p.chunk;
  const int64_t end = min(S, start + (int64_t)p.chunk);
  const int len = end > start ? (int)(end - start) : 0;
  const int mem_len = (int)max((int64_t)0, min(end, s_old) - start);  // already in HBM
  const bool has_new = (s_old >= start) && (s_old < end);
  const int selcap = min(p.budget, p.chunk);
  const int ring = p.stages;

  const FusedSmem L(G, C, p.chunk, selcap, ring);
  uint4* stage = reinterpret_cast<uint4*>(smem + L.stage);
  uint16_t* dist = reinterpret_cast<uint16_t*>(smem + L.dist);
  uint16_t* gmin = reinterpret_cast<uint16_t*>(smem + L.gmin);
  const int ngroups_cap = p.chunk / 32;
  int* hist = reinterpret_cast<int*>(smem + L.hist);
  uint16_t* hist_all = reinterpret_cast<uint16_t*>(smem + L.hist_all);
  int* sel = reinterpret_cast<int*>(smem + L.sel);
  float* inbox = reinterpret_cast<float*>(smem + L.inbox);
  float* wpart = reinterpret_cast<float*>(smem + L.wpart);
  float* qfs = reinterpret_cast<float*>(smem + L.qf);
  Code* qcode = reinterpret_cast<Code*>(smem + L.qcode);
  double* sqs = reinterpret_cast<double*>(smem + L.sq);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* hist_bar = bars + kMaxStages;
  uint64_t* inbox_bar = bars + kMaxStages + 1;
  int n_owned = 0;  // q-heads whose final merge this rank performs
  for (int g = rank; g < G; g += C) ++n_owned;

  uint4* planes = p.seq[si].codes + (int64_t)hk * 2 * cap;  // lo plane; hi = +cap
  const uint4* lo_g = planes + start;
  const uint4* hi_g = planes + cap + start;

  // ---------------------------------------------------------------- prologue
  ADAMAS_TRACE(0);
  if (p.trace != nullptr && threadIdx.x == 0) p.trace[blockIdx.x * 16 + 14] = globaltimer_ns();
  const int n_stages = (mem_len + kStageTok - 1) / kStageTok;
  constexpr int kIssueWarp = kFusedWarps - 1;
  auto issue = [&](int st) {
    const int slot = st % ring;
    const int ntok = min(kStageTok, mem_len - st * kStageTok);
    const uint32_t bytes = (uint32_t)ntok * 16u;
    uint4* dst = stage + (size_t)slot * (kStageBytes / 16);
    mbar_expect_tx(&bars[slot], 2u * bytes);
    bulk_g2s(dst, lo_g + (int64_t)st * kStageTok, bytes, &bars[slot]);
    bulk_g2s(dst + kStageTok, hi_g + (int64_t)st * kStageTok, bytes, &bars[slot]);
  };
  if (warp == kIssueWarp && lane == 0) {  // the code stream starts before anything else
    for (int s = 0; s < ring; ++s) mbar_init(&bars[s], 1);
    mbar_init(hist_bar, 1);
    mbar_init(inbox_bar, 1);
    mbar_fence_init();
    for (int st = 0; st < min(ring, n_stages); ++st) issue(st);
    // bytes this CTA will receive over DSMEM: every rank's u16 histograms, and
    // C partials per q-head it merges
    mbar_expect_tx(hist_bar, (uint32_t)(C * G * kHistBins * 2));
    if (n_owned) mbar_expect_tx(inbox_bar, (uint32_t)(n_owned * C * kPartStride * 4));
  }
  for (int i = tid; i < G * kHistBins; i += kFusedThreads) hist[i] = 0;
  for (int i = tid; i < G * ngroups_cap; i += kFusedThreads) gmin[i] = 0xffff;
  ADAMAS_TRACE(1);

  if (warp < G) {  // encode query head hk * G + warp (sweep.cpp:92-94)
    const T* qp = reinterpret_cast<const T*>(p.q) + ((int64_t)si * n_q + (int64_t)hk * G + warp) * kHeadDim;
    float f[4];
    Raw4<T>::to_float(Raw4<T>::load(qp + lane * 4), f);
    *reinterpret_cast<float4*>(qfs + warp * kHeadDim + lane * 4) = make_float4(f[0], f[1], f[2], f[3]);
    Code c;
    if (!encode128_warp(f, sqs + warp * kHeadDim, c, !p.exact_encode) && lane == 0)
      atomicOr(p.status, kStatusDegenerate);
    if (lane == 0) qcode[warp] = c;
  }
  if (has_new && warp == G) {  // append (kv_cache.cpp:62-71)
    const int64_t vrow = (int64_t)si * p.n_kv + hk;
    const T* kp = reinterpret_cast<const T*>(p.k_new) + vrow * kHeadDim;
    const T* vp = reinterpret_cast<const T*>(p.v_new) + vrow * kHeadDim;
    const auto kr = Raw4<T>::load(kp + lane * 4);
    const auto vr = Raw4<T>::load(vp + lane * 4);
    const int64_t row = (int64_t)hk * cap + s_old;
    Raw4<T>::store(reinterpret_cast<T*>(p.seq[si].K) + row * kHeadDim + lane * 4, kr);
    Raw4<T>::store(reinterpret_cast<T*>(p.seq[si].V) + row * kHeadDim + lane * 4, vr);
    float f[4];
    Raw4<T>::to_float(kr, f);
    Code c;
    if (!encode128_warp(f, sqs + G * kHeadDim, c, !p.exact_encode) && lane == 0)
      atomicOr(p.status, kStatusDegenerate);
    if (lane == 0) {
      qcode[G] = c;
      store_code(planes, cap, s_old, c);
    }
  }
  __syncthreads();
  cluster_arrive_relaxed();  // "my mbarriers are initialized"; waited on before the first DSMEM store
  QCode qc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) qc[g] = make_qcode(qcode[g]);

  // ---------------------------------------------------------------- scan
  ADAMAS_TRACE(2);
  for (int st = 0; st < n_stages; ++st) {
    const int slot = st % ring;
    mbar_wait(&bars[slot], (uint32_t)(st / ring) & 1u);
    const uint4* slo = stage + (size_t)slot * (kStageBytes / 16);
    const uint4* shi = slo + kStageTok;
    const int base = st * kStageTok;
    const int ntok = min(kStageTok, mem_len - base);
    uint4 a[2], b[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = tid + u * kFusedThreads;
      if (j < ntok) { a[u] = slo[j]; b[u] = shi[j]; }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = tid + u * kFusedThreads;
      const bool valid = j < ntok;
      const uint32_t lo[4] = {a[u].x, a[u].y, a[u].z, a[u].w}, hi[4] = {b[u].x, b[u].y, b[u].z, b[u].w};
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint32_t d = valid ? l1_distance(qc[g], lo, hi) : 0xffffu;
        if (valid) {
          dist[g * p.chunk + base + j] = (uint16_t)d;
          atomicAdd(&hist[g * kHistBins + d], 1);
        }
        // per 32-token group minimum: lets the compaction skip groups above T
        const uint32_t m = __reduce_min_sync(kFull, d);
        if (lane == 0 && (base + j) < p.chunk) gmin[g * ngroups_cap + ((base + j) >> 5)] = (uint16_t)m;
      }
    }
    __syncthreads();
    if (warp == kIssueWarp && lane == 0 && st + ring < n_stages) issue(st + ring);
  }
  if (has_new && tid < G) {  // the appended token is a candidate
    const Code nc = qcode[G];
    const uint32_t d = l1_distance(make_qcode(qcode[tid]), nc.lo, nc.hi);
    const int lt = (int)(s_old - start);
    dist[tid * p.chunk + lt] = (uint16_t)d;
    atomicAdd(&hist[tid * kHistBins + d], 1);
    uint16_t& gm = gmin[tid * ngroups_cap + (lt >> 5)];
    gm = (uint16_t)min((uint32_t)gm, d);
  }
  ADAMAS_TRACE(3);
  __syncthreads();  // local histogram final
  // Push this rank's histograms (as u16, counts <= chunk < 2^16) into every
  // rank's hist_all[rank] with st.async; each receiver's mbarrier counts bytes.
  cluster_wait();
  if (tid < G * (kHistBins / 8)) {
    const int g = tid / (kHistBins / 8), b0 = (tid % (kHistBins / 8)) * 8;
    const int4 h0 = *reinterpret_cast<const int4*>(hist + g * kHistBins + b0);
    const int4 h1 = *reinterpret_cast<const int4*>(hist + g * kHistBins + b0 + 4);
    const uint32_t w0 = (uint32_t)h0.x | ((uint32_t)h0.y << 16), w1 = (uint32_t)h0.z | ((uint32_t)h0.w << 16);
    const uint32_t w2 = (uint32_t)h1.x | ((uint32_t)h1.y << 16), w3 = (uint32_t)h1.z | ((uint32_t)h1.w << 16);
    const uint32_t local = smem_addr(hist_all + ((size_t)rank * G + g) * kHistBins + b0);
    for (int r = 0; r < C; ++r)
      st_async_v4(mapa_shared(local, r), w0, w1, w2, w3, mapa_shared(smem_addr(hist_bar), r));
  }
  mbar_wait(hist_bar, 0);
  ADAMAS_TRACE(4);

  // ---------------------------------------------------------------- threshold
  // Warp g (g < G) finds head g's threshold T = smallest distance whose
  // cumulative count over all ranks reaches k: lane l owns bins 16l..16l+15,
  // a warp scan orders the lanes, the owning lane walks its 16 bins.
  const int k_eff = (int)min((int64_t)p.budget, S);
  if (warp < G) {
    const int g = warp;
    int tot[16], pre[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) { tot[i] = 0; pre[i] = 0; }
    for (int r = 0; r < C; ++r) {
      const uint4* h = reinterpret_cast<const uint4*>(hist_all + ((size_t)r * G + g) * kHistBins + lane * 16);
      const uint4 a = h[0], b = h[1];
      const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int v = (int)((w[i >> 1] >> (16 * (i & 1))) & 0xffffu);
        tot[i] += v;
        pre[i] += r < rank ? v : 0;
      }
    }
    int lt = 0, lp = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) { lt += tot[i]; lp += pre[i]; }
    int it = lt, ip = lp;
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      const int a2 = __shfl_up_sync(kFull, it, m), b2 = __shfl_up_sync(kFull, ip, m);
      if (lane >= m) { it += a2; ip += b2; }
    }
    int c = it - lt, cp = ip - lp;  // exclusive: counts in lower bins
    if (c < k_eff && c + lt >= k_eff) {
      bool done = false;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (!done && c + tot[i] >= k_eff) {
          sc[g][0] = lane * 16 + i;  // T
          sc[g][1] = c;              // count of distances < T over the whole head
          sc[g][2] = cp;             // count of distances < T in ranks before this one
          sc[g][3] = pre[i];         // count of distances == T in ranks before this one
          done = true;
        }
        c += tot[i];
        cp += pre[i];
      }
    }
  }
  __syncthreads();
  ADAMAS_TRACE(5);

  // ---------------------------------------------------------------- compaction
  // Thread t of head g (TG = 512 / G threads per head) owns a contiguous run
  // of 32-token groups; a group whose minimum distance exceeds T holds no
  // selected token and costs one shared load. Candidate groups are evaluated
  // with SWAR on u16 pairs: (K - x) & 0x80008000 has a guard bit set exactly
  // where x <= thr (K = thr in both halves | 0x80008000; distances < 2^15).
  // Count -> one CTA scan in index order -> emit.
  {
    constexpr int TG = kFusedThreads / G;
    const int g = tid / TG, t_in = tid % TG;
    const int ngroups = (len + 31) >> 5;
    const int gpt = (ngroups + TG - 1) / TG;
    const int grp0 = min(ngroups, t_in * gpt), grp1 = min(ngroups, grp0 + gpt);
    const int thr = sc[g][0], below = sc[g][1], pre_lt = sc[g][2], pre_eq = sc[g][3];
    const int need = k_eff - below;               // ties at T the whole head takes
    const int eq_budget = max(0, need - pre_eq);  // ... of which this rank may take
    const int out_off = pre_lt + min(pre_eq, need);
    const uint16_t* dg = dist + g * p.chunk;
    const uint16_t* gm = gmin + g * ngroups_cap;
    const uint32_t kle = ((uint32_t)thr * 0x00010001u) | 0x80008000u;  // x <= thr
    const uint32_t klt = thr > 0 ? (((uint32_t)(thr - 1) * 0x00010001u) | 0x80008000u) : 0u;  // x < thr
    // 32-bit masks (bit i = token i of the group) of x < thr and x == thr
    auto group_masks = [&](int grp, uint32_t& ltm, uint32_t& eqm) {
      const uint4* src = reinterpret_cast<const uint4*>(dg + grp * 32);
      uint32_t le = 0, lt = 0;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const uint4 v4 = src[q4];
        const uint32_t w[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = (q4 * 4 + e) * 2;
          const uint32_t a = (kle - w[e]) & 0x80008000u, b = thr > 0 ? ((klt - w[e]) & 0x80008000u) : 0u;
          le |= ((a >> 15) & 1u) << i | (a >> 31) << (i + 1);
          lt |= ((b >> 15) & 1u) << i | (b >> 31) << (i + 1);
        }
      }
      const int valid = len - grp * 32;  // tokens of this group inside the rank's range
      const uint32_t vm = valid >= 32 ? 0xffffffffu : ((1u << valid) - 1u);
      ltm = lt & vm;
      eqm = (le & ~lt) & vm;
    };
    const T* Kg = reinterpret_cast<const T*>(p.seq[si].K) + ((int64_t)hk * cap + start) * kHeadDim;
    const T* Vg = reinterpret_cast<const T*>(p.seq[si].V) + ((int64_t)hk * cap + start) * kHeadDim;
    int my_lt = 0, my_eq = 0;
    for (int grp = grp0; grp < grp1; ++grp) {
      if (gm[grp] > thr) continue;
      uint32_t ltm, eqm;
      group_masks(grp, ltm, eqm);
      my_lt += __popc(ltm);
      my_eq += __popc(eqm);
      for (uint32_t m = (p.dbg & 1) ? 0u : (ltm | eqm); m; m &= m - 1) {  // warm L2 for the gather
        const int t = grp * 32 + __ffs(m) - 1;
        const char* kp = reinterpret_cast<const char*>(Kg + (int64_t)t * kHeadDim);
        const char* vp = reinterpret_cast<const char*>(Vg + (int64_t)t * kHeadDim);
#pragma unroll
        for (int c = 0; c < (int)(kHeadDim * sizeof(T)); c += 128) {
          prefetch_l2(kp + c);
          prefetch_l2(vp + c);
        }
      }
    }
    int lt_before = 0, eq_before = 0;
    {
      int v[2 * G], ex[2 * G], sum[2 * G];
#pragma unroll
      for (int g2 = 0; g2 < G; ++g2) { v[2 * g2] = g2 == g ? my_lt : 0; v[2 * g2 + 1] = g2 == g ? my_eq : 0; }
      block_scan<2 * G>(v, ex, sum, scan_scratch);
#pragma unroll
      for (int g2 = 0; g2 < G; ++g2) {
        if (g2 == g) { lt_before = ex[2 * g2]; eq_before = ex[2 * g2 + 1]; }
        if (tid == 0) nsel[g2] = min(sum[2 * g2] + min(sum[2 * g2 + 1], max(0, k_eff - sc[g2][1] - sc[g2][3])), selcap);
      }
    }
    ADAMAS_TRACE(6);
    if (my_lt | my_eq) {
      int32_t* idx_row = (p.idx && !(p.dbg & 2))
                             ? p.idx + ((int64_t)si * n_q + (int64_t)hk * G + g) * p.budget + out_off
                             : nullptr;
      int pos = lt_before + min(eq_before, eq_budget);
      int eq_seen = eq_before;
      for (int grp = grp0; grp < grp1; ++grp) {
        if (gm[grp] > thr) continue;
        uint32_t ltm, eqm;
        group_masks(grp, ltm, eqm);
        for (uint32_t m = ltm | eqm; m; m &= m - 1) {
          const int i = __ffs(m) - 1;
          if ((eqm >> i) & 1u) {
            if (eq_seen++ >= eq_budget) continue;  // ties beyond the budget are not taken
          }
          const int tok = (int)start + grp * 32 + i;
          if (pos < selcap) sel[g * selcap + pos] = tok;
          if (idx_row) idx_row[pos] = tok;
          ++pos;
        }
      }
    }
    if (rank == 0 && p.idx && t_in == 0) {  // estimator.cpp:80 caps the selection at S
      int32_t* row = p.idx + ((int64_t)si * n_q + (int64_t)hk * G + g) * p.budget;
      for (int i = k_eff; i < p.budget; ++i) row[i] = -1;
    }
  }
  __syncthreads();
  ADAMAS_TRACE(7);

  // ---------------------------------------------------------------- attend
  {
    constexpr int WG = kFusedWarps / G;  // warps per q-head
    const int g = warp % G, sub = warp / G;
    const int ns = nsel[g];
    const int hq = hk * G + g;
    const float4 q4 = *reinterpret_cast<const float4*>(qfs + g * kHeadDim + lane * 4);
    float qf[4] = {q4.x, q4.y, q4.z, q4.w};
    const float scale = 0.088388347648318440f * kLog2e;  // 1/sqrt(128), log2 units
#pragma unroll
    for (int j = 0; j < 4; ++j) qf[j] *= scale;
    const T* Kh = reinterpret_cast<const T*>(p.seq[si].K) + (int64_t)hk * cap * kHeadDim + lane * 4;
    const T* Vh = reinterpret_cast<const T*>(p.seq[si].V) + (int64_t)hk * cap * kHeadDim + lane * 4;
    float m = -INFINITY, l = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
    constexpr int B = 4;  // rows in flight per warp
    for (int r0 = sub; r0 < ns; r0 += WG * B) {
      typename Raw4<T>::V kr[B], vr[B];
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int r = r0 + b * WG;
        if (r < ns) {
          const int64_t t = sel[g * selcap + r];
          kr[b] = Raw4<T>::load(Kh + t * kHeadDim);
          vr[b] = Raw4<T>::load(Vh + t * kHeadDim);
        }
      }
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int r = r0 + b * WG;
        if (r < ns) {
          float kf[4], vf[4];
          Raw4<T>::to_float(kr[b], kf);
          Raw4<T>::to_float(vr[b], vf);
          const float s = warp_sum(qf[0] * kf[0] + qf[1] * kf[1] + qf[2] * kf[2] + qf[3] * kf[3]);
          const float mn = fmaxf(m, s);
          const float corr = exp2f(m - mn);
          const float pr = exp2f(s - mn);
          l = l * corr + pr;
#pragma unroll
          for (int j = 0; j < 4; ++j) o[j] = o[j] * corr + pr * vf[j];
          m = mn;
        }
      }
    }
    ADAMAS_TRACE(8);
    float* wp = wpart + warp * kPartStride;
    if (lane == 0) { wp[0] = m; wp[1] = l; }
#pragma unroll
    for (int j = 0; j < 4; ++j) wp[4 + lane * 4 + j] = o[j];
    __syncthreads();
    if (sub == 0) {  // combine this head's WG warp partials, push to the merging rank
      const float* mine = wpart + (lane * G + g) * kPartStride;
      const float ml = lane < WG ? mine[0] : -INFINITY, ll = lane < WG ? mine[1] : 0.f;
      float M = ll > 0.f ? ml : -INFINITY;
#pragma unroll
      for (int m2 = 16; m2 > 0; m2 >>= 1) M = fmaxf(M, __shfl_xor_sync(kFull, M, m2));
      const float cl = ll > 0.f ? exp2f(ml - M) : 0.f;
      const float Lsum = warp_sum(ll * cl);
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int s2 = 0; s2 < WG; ++s2) {
        const float c = __shfl_sync(kFull, cl, s2);
        const float4 v4 = *reinterpret_cast<const float4*>(wpart + (s2 * G + g) * kPartStride + 4 + lane * 4);
        acc[0] += v4.x * c; acc[1] += v4.y * c; acc[2] += v4.z * c; acc[3] += v4.w * c;
      }
      // push (M, L, o[128]) into the merging rank's inbox[rank][g] (528 B)
      const uint32_t local = smem_addr(inbox + (rank * G + g) * kPartStride);
      const uint32_t dst = mapa_shared(local, (uint32_t)(g % C));
      const uint32_t bar = mapa_shared(smem_addr(inbox_bar), (uint32_t)(g % C));
      if (lane == 0) st_async_v4(dst, __float_as_uint(M), __float_as_uint(Lsum), 0u, 0u, bar);
      st_async_v4(dst + 16 + lane * 16, __float_as_uint(acc[0]), __float_as_uint(acc[1]), __float_as_uint(acc[2]),
                  __float_as_uint(acc[3]), bar);
    }
  }
  ADAMAS_TRACE(9);
  if (n_owned) mbar_wait(inbox_bar, 0);  // all C partials of the heads this rank merges
  ADAMAS_TRACE(10);

  // ---------------------------------------------------------------- merge
  for (int g = warp; g < G; g += kFusedWarps) {
    if (g % C != rank) continue;
    float M = -INFINITY;
    for (int r = 0; r < C; ++r) {
      const float* q2 = inbox + (r * G + g) * kPartStride;
      if (q2[1] > 0.f) M = fmaxf(M, q2[0]);
    }
    float Lsum = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int r = 0; r < C; ++r) {
      const float* q2 = inbox + (r * G + g) * kPartStride;
      if (!(q2[1] > 0.f)) continue;
      const float c = exp2f(q2[0] - M);
      Lsum += q2[1] * c;
      const float4 v4 = *reinterpret_cast<const float4*>(q2 + 4 + lane * 4);
      acc[0] += v4.x * c; acc[1] += v4.y * c; acc[2] += v4.z * c; acc[3] += v4.w * c;
    }
    const float inv = 1.f / Lsum;
    float* op = p.out + ((int64_t)si * n_q + (int64_t)hk * G + g) * kHeadDim + lane * 4;
    *reinterpret_cast<float4*>(op) = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
  }
  ADAMAS_TRACE(11);
  if (p.trace != nullptr && threadIdx.x == 0) p.trace[blockIdx.x * 16 + 15] = globaltimer_ns();
}

}  // namespace adamas_dev
