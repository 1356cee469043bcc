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
  const void* q;      // [n_seqs][n_q][128]
  const void* k_new;  // [n_seqs][n_kv][128]
  const void* v_new;
  float* out;    // [n_seqs][n_q][128]
  int32_t* idx;  // [n_seqs][n_q][budget] or null
  int* status;
  unsigned long long* trace;  // optional per-CTA phase timestamps (diagnostics)
  FusedSeq seq[kMaxSeqs];
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define ADAMAS_TRACE(i) \
  do { if (p.trace != nullptr && threadIdx.x == 0) p.trace[blockIdx.x * 16 + (i)] = global_ns(); } while (0)

// Dynamic shared-memory carve-up, identical on host and device.
struct FusedSmem {
  uint32_t stage, dist, hist, hist_all, sel, inbox, wpart, qcode, sq, bars, total;
  __host__ __device__ static uint32_t align(uint32_t x, uint32_t a) { return (x + a - 1u) & ~(a - 1u); }
  __host__ __device__ FusedSmem(int G, int C, int chunk, int selcap, int stages) {
    uint32_t o = 0;
    stage = o; o += (uint32_t)stages * kStageBytes;
    dist = o;  o = align(o + (uint32_t)G * chunk * 2, 16);
    hist = o;  o += (uint32_t)G * kHistBins * 4;
    hist_all = o; o += (uint32_t)C * G * kHistBins * 2;  // u16 histograms received from every rank
    sel = o;   o = align(o + (uint32_t)G * selcap * 4, 16);
    inbox = o; o += (uint32_t)C * G * kPartStride * 4;
    wpart = o; o += kFusedWarps * kPartStride * 4;
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
  __shared__ int warp_cnt[kFusedWarps][2];
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
  int* hist = reinterpret_cast<int*>(smem + L.hist);
  uint16_t* hist_all = reinterpret_cast<uint16_t*>(smem + L.hist_all);
  int* sel = reinterpret_cast<int*>(smem + L.sel);
  float* inbox = reinterpret_cast<float*>(smem + L.inbox);
  float* wpart = reinterpret_cast<float*>(smem + L.wpart);
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
  ADAMAS_TRACE(1);

  if (warp < G) {  // encode query head hk * G + warp (sweep.cpp:92-94)
    const T* qp = reinterpret_cast<const T*>(p.q) + ((int64_t)si * n_q + (int64_t)hk * G + warp) * kHeadDim;
    float f[4];
    Raw4<T>::to_float(Raw4<T>::load(qp + lane * 4), f);
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
      if (j < ntok) {
        const uint32_t lo[4] = {a[u].x, a[u].y, a[u].z, a[u].w}, hi[4] = {b[u].x, b[u].y, b[u].z, b[u].w};
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const uint32_t d = l1_distance(qc[g], lo, hi);
          dist[g * p.chunk + base + j] = (uint16_t)d;
          atomicAdd(&hist[g * kHistBins + d], 1);
        }
      }
    }
    __syncthreads();
    if (warp == kIssueWarp && lane == 0 && st + ring < n_stages) issue(st + ring);
  }
  if (has_new && tid < G) {  // the appended token is a candidate
    const Code nc = qcode[G];
    const uint32_t d = l1_distance(make_qcode(qcode[tid]), nc.lo, nc.hi);
    dist[tid * p.chunk + (int)(s_old - start)] = (uint16_t)d;
    atomicAdd(&hist[tid * kHistBins + d], 1);
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
  // thread t owns distance bin t of every q-head
  const int k_eff = (int)min((int64_t)p.budget, S);
  {
    int tot[G], pre[G];
#pragma unroll
    for (int g = 0; g < G; ++g) { tot[g] = 0; pre[g] = 0; }
    for (int r = 0; r < C; ++r) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int h = hist_all[((size_t)r * G + g) * kHistBins + tid];
        tot[g] += h;
        pre[g] += r < rank ? h : 0;
      }
    }
    ADAMAS_TRACE(5);
    int v[2 * G], ex[2 * G], sum[2 * G];
#pragma unroll
    for (int g = 0; g < G; ++g) { v[g] = tot[g]; v[G + g] = pre[g]; }
    block_scan<2 * G>(v, ex, sum, scan_scratch);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (ex[g] < k_eff && ex[g] + tot[g] >= k_eff) {  // this bin holds the k-th smallest
        sc[g][0] = tid;        // T
        sc[g][1] = ex[g];      // count of distances < T over the whole head
        sc[g][2] = ex[G + g];  // count of distances < T in ranks before this one
        sc[g][3] = pre[g];     // count of distances == T in ranks before this one
      }
    }
  }
  __syncthreads();
  ADAMAS_TRACE(6);

  // ---------------------------------------------------------------- compaction
  // Warp w serves q-head g = w % G over sub-range w / G of this rank's tokens;
  // lane l reads 8 consecutive distances per 256-token step, so the
  // (sub-range, step, lane) order is index order. Pass 1 counts (< T, == T)
  // per warp; pass 2 re-walks with a packed warp scan and emits in order.
  {
    constexpr int WG = kFusedWarps / G;
    const int g = warp % G, sub = warp / G;
    const int per_warp = ((len + WG - 1) / WG + 255) / 256 * 256;
    const int wbeg = sub * per_warp, wend = min(len, wbeg + per_warp);
    const int thr = sc[g][0], below = sc[g][1], pre_lt = sc[g][2], pre_eq = sc[g][3];
    const int need = k_eff - below;               // ties at T the whole head takes
    const int eq_budget = max(0, need - pre_eq);  // ... of which this rank may take
    const int out_off = pre_lt + min(pre_eq, need);
    const uint16_t* dg = dist + g * p.chunk;
    auto masks = [&](int t0, uint32_t& ltm, uint32_t& eqm) {
      ltm = 0;
      eqm = 0;
      if (t0 < wend) {
        const uint4 vv = *reinterpret_cast<const uint4*>(dg + t0);
        const uint32_t w[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int d = (int)((w[e >> 1] >> (16 * (e & 1))) & 0xffffu);
          const bool valid = t0 + e < wend;
          ltm |= (uint32_t)(valid && d < thr) << e;
          eqm |= (uint32_t)(valid && d == thr) << e;
        }
      }
    };
    const T* Kg = reinterpret_cast<const T*>(p.seq[si].K) + ((int64_t)hk * cap + start) * kHeadDim;
    const T* Vg = reinterpret_cast<const T*>(p.seq[si].V) + ((int64_t)hk * cap + start) * kHeadDim;
    unsigned cnt = 0;  // packed: lt in bits 0..15, eq in bits 16..31
    for (int t0 = wbeg + lane * 8; t0 - lane * 8 < wend; t0 += 256) {
      uint32_t ltm, eqm;
      masks(t0, ltm, eqm);
      cnt += (unsigned)__popc(ltm) | ((unsigned)__popc(eqm) << 16);
      // candidates (d <= T): start pulling their K and V rows into L2 now, so
      // the gather after the compaction hits L2 instead of HBM
      for (uint32_t m = ltm | eqm; m; m &= m - 1) {
        const int t = t0 + __ffs(m) - 1;
        prefetch_l2_bulk(Kg + (int64_t)t * kHeadDim, kHeadDim * sizeof(T));
        prefetch_l2_bulk(Vg + (int64_t)t * kHeadDim, kHeadDim * sizeof(T));
      }
    }
    cnt = __reduce_add_sync(kFull, cnt);
    if (lane == 0) { warp_cnt[warp][0] = (int)(cnt & 0xffffu); warp_cnt[warp][1] = (int)(cnt >> 16); }
    __syncthreads();
    ADAMAS_TRACE(7);
    int run_lt = 0, run_eq = 0, tot_lt = 0, tot_eq = 0;
    for (int s2 = 0; s2 < WG; ++s2) {
      const int w2 = s2 * G + g;
      if (s2 < sub) { run_lt += warp_cnt[w2][0]; run_eq += warp_cnt[w2][1]; }
      tot_lt += warp_cnt[w2][0];
      tot_eq += warp_cnt[w2][1];
    }
    int32_t* idx_row = p.idx ? p.idx + ((int64_t)si * n_q + (int64_t)hk * G + g) * p.budget + out_off : nullptr;
    for (int t0 = wbeg + lane * 8; t0 - lane * 8 < wend && cnt != 0; t0 += 256) {
      uint32_t ltm, eqm;
      masks(t0, ltm, eqm);
      if (__ballot_sync(kFull, (ltm | eqm) != 0) == 0) continue;
      const unsigned packed = (unsigned)__popc(ltm) | ((unsigned)__popc(eqm) << 16);
      unsigned incl = packed;
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        const unsigned o = __shfl_up_sync(kFull, incl, m);
        if (lane >= m) incl += o;
      }
      const unsigned excl = incl - packed;
      const unsigned step_tot = __shfl_sync(kFull, incl, 31);
      if (ltm | eqm) {
        const int lt_before = run_lt + (int)(excl & 0xffffu), eq_before = run_eq + (int)(excl >> 16);
        int pos = lt_before + min(eq_before, eq_budget);
        int eq_seen = eq_before;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          bool take = (ltm >> e) & 1u;
          if ((eqm >> e) & 1u) take = eq_seen++ < eq_budget;
          if (take) {
            const int tok = (int)start + t0 + e;
            if (pos < selcap) sel[g * selcap + pos] = tok;
            if (idx_row) idx_row[pos] = tok;
            ++pos;
          }
        }
      }
      run_lt += (int)(step_tot & 0xffffu);
      run_eq += (int)(step_tot >> 16);
    }
    if (sub == 0 && lane == 0) nsel[g] = min(tot_lt + min(tot_eq, eq_budget), selcap);  // rows to attend
    if (rank == 0 && p.idx && sub == 0) {  // estimator.cpp:80 caps the selection at S
      int32_t* row = p.idx + ((int64_t)si * n_q + (int64_t)hk * G + g) * p.budget;
      for (int i = k_eff + lane; i < p.budget; i += 32) row[i] = -1;
    }
  }
  __syncthreads();
  ADAMAS_TRACE(8);

  // ---------------------------------------------------------------- attend
  {
    constexpr int WG = kFusedWarps / G;  // warps per q-head
    const int g = warp % G, sub = warp / G;
    const int ns = nsel[g];
    const int hq = hk * G + g;
    const T* qp = reinterpret_cast<const T*>(p.q) + ((int64_t)si * n_q + hq) * kHeadDim;
    float qf[4];
    Raw4<T>::to_float(Raw4<T>::load(qp + lane * 4), qf);
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
    ADAMAS_TRACE(9);
    float* wp = wpart + warp * kPartStride;
    if (lane == 0) { wp[0] = m; wp[1] = l; }
#pragma unroll
    for (int j = 0; j < 4; ++j) wp[4 + lane * 4 + j] = o[j];
    __syncthreads();
    if (sub == 0) {  // combine this head's WG warp partials, push to the merging rank
      float M = -INFINITY;
      for (int s2 = 0; s2 < WG; ++s2) {
        const float* q2 = wpart + (s2 * G + g) * kPartStride;
        if (q2[1] > 0.f) M = fmaxf(M, q2[0]);
      }
      float Lsum = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
      for (int s2 = 0; s2 < WG; ++s2) {
        const float* q2 = wpart + (s2 * G + g) * kPartStride;
        if (!(q2[1] > 0.f)) continue;
        const float c = exp2f(q2[0] - M);
        Lsum += q2[1] * c;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] += q2[4 + lane * 4 + j] * c;
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
  ADAMAS_TRACE(10);
  if (n_owned) mbar_wait(inbox_bar, 0);  // all C partials of the heads this rank merges
  ADAMAS_TRACE(11);

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
  ADAMAS_TRACE(12);
}

}  // namespace adamas_dev
