// fused_decode.cuh — one Adamas decode step of one layer in ONE launch.
//
// Work unit = (sequence, kv-head) with its G = n_q / n_kv query heads. A
// thread-block cluster of C CTAs owns a unit; CTA rank r owns the contiguous
// token range [r * chunk, min(S, (r + 1) * chunk)) where S includes the token
// appended by this very step (Alg. 1: update before estimate).
//
//   prologue  warps 0..G-1 encode the G query heads (fp64 FWHT + RMS
//             thresholds, bit-exact); the rank owning position S-1 encodes the
//             new key and appends (k, v, code) to the cache (kv_cache.cpp:62-71)
//   scan      bulk-copy (TMA engine) ring streams the range's lo/hi code planes
//             HBM -> smem; every token's G distances (estimator.cpp:45-59) go
//             to a u16 smem array and a per-CTA 512-bin smem histogram
//   select    cluster barrier; every rank reads all C histograms over DSMEM and
//             derives the global threshold T (k-th smallest), how many ties at
//             T the ranks before it take, and its output offset; then an
//             order-preserving warp-ballot compaction of its own tokens
//             (top_k semantics, estimator.cpp:75-90: (score, index) order)
//   attend    each rank attends over its own selected rows (gather of K, V by
//             index, fp32 online softmax) and pushes (m, l, o[128]) into the
//             merging rank's smem over DSMEM; cluster barrier; log-sum-exp
//             merge -> out (attention.cpp:8-45 semantics)
//
// Indices are bit-exact by construction: the selection is computed from the
// exact integer distances with the reference's total order, no approximation.
#pragma once
#include <cooperative_groups.h>

#include "ops.cuh"

namespace adamas_dev {
namespace cg = cooperative_groups;

constexpr int kFusedThreads = 256;
constexpr int kFusedWarps = kFusedThreads / 32;
constexpr int kStageTok = 512;  // tokens per bulk-copy stage: 2 x 8 KB planes
constexpr int kStages = 4;
constexpr int kHistBins = 512;  // 2-bit L1 distances at d = 128 are <= 384
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
  int n_seqs, n_kv, C, chunk, budget;
  const void* q;      // [n_seqs][n_q][128]
  const void* k_new;  // [n_seqs][n_kv][128]
  const void* v_new;
  float* out;    // [n_seqs][n_q][128]
  int32_t* idx;  // [n_seqs][n_q][budget] or null
  int* status;
  FusedSeq seq[kMaxSeqs];
};

// Dynamic shared-memory carve-up, identical on host and device.
struct FusedSmem {
  uint32_t stage, dist, hist, sel, inbox, wpart, qcode, sq, bars, scal, total;
  __host__ __device__ static uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }
  __host__ __device__ FusedSmem(int G, int C, int chunk, int selcap) {
    uint32_t o = 0;
    stage = o; o += kStages * kStageTok * 32;
    dist = o;  o = align16(o + (uint32_t)G * chunk * 2);
    hist = o;  o += (uint32_t)G * kHistBins * 4;
    sel = o;   o = align16(o + (uint32_t)G * selcap * 4);
    inbox = o; o += (uint32_t)C * G * kPartStride * 4;
    wpart = o; o += kFusedWarps * kPartStride * 4;
    o = (o + 31u) & ~31u;
    qcode = o; o += (uint32_t)(G + 1) * 32;
    sq = o;    o += kFusedWarps * kHeadDim * 8;
    bars = o;  o += kStages * 8;
    scal = o;  o += 64 * 4;
    total = o;
  }
};

// Exclusive scan over the CTA of up to three ints (thread order).
__device__ __forceinline__ void block_scan3(int a, int b, int c, int* scratch /*3*32*/, int& ea, int& eb,
                                            int& ec) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int ia = a, ib = b, ic = c;
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    const int ta = __shfl_up_sync(kFull, ia, m), tb = __shfl_up_sync(kFull, ib, m),
              tc = __shfl_up_sync(kFull, ic, m);
    if (lane >= m) { ia += ta; ib += tb; ic += tc; }
  }
  if (lane == 31) { scratch[warp] = ia; scratch[32 + warp] = ib; scratch[64 + warp] = ic; }
  __syncthreads();
  int wa = 0, wb = 0, wc = 0;
  for (int w = 0; w < warp; ++w) { wa += scratch[w]; wb += scratch[32 + w]; wc += scratch[64 + w]; }
  __syncthreads();
  ea = wa + ia - a;
  eb = wb + ib - b;
  ec = wc + ic - c;
}

template <typename T, int G>
__global__ void __launch_bounds__(kFusedThreads, 1) fused_decode_kernel(const __grid_constant__ FusedParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int C = p.C;
  const int rank = (int)cluster.block_rank();
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

  const FusedSmem L(G, C, p.chunk, selcap);
  uint4* stage = reinterpret_cast<uint4*>(smem + L.stage);
  uint16_t* dist = reinterpret_cast<uint16_t*>(smem + L.dist);
  int* hist = reinterpret_cast<int*>(smem + L.hist);
  int* sel = reinterpret_cast<int*>(smem + L.sel);
  float* inbox = reinterpret_cast<float*>(smem + L.inbox);
  float* wpart = reinterpret_cast<float*>(smem + L.wpart);
  Code* qcode = reinterpret_cast<Code*>(smem + L.qcode);
  double* sqs = reinterpret_cast<double*>(smem + L.sq);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  int* scal = reinterpret_cast<int*>(smem + L.scal);

  uint4* planes = p.seq[si].codes + (int64_t)hk * 2 * cap;  // lo plane; hi = +cap
  const uint4* lo_g = planes + start;
  const uint4* hi_g = planes + cap + start;

  // ---------------------------------------------------------------- prologue
  for (int i = tid; i < G * kHistBins; i += kFusedThreads) hist[i] = 0;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int n_stages = (mem_len + kStageTok - 1) / kStageTok;
  auto issue = [&](int st) {
    const int slot = st % kStages;
    const int ntok = min(kStageTok, mem_len - st * kStageTok);
    const uint32_t bytes = (uint32_t)ntok * 16u;
    mbar_expect_tx(&bars[slot], 2u * bytes);
    bulk_g2s(stage + slot * 2 * kStageTok, lo_g + (int64_t)st * kStageTok, bytes, &bars[slot]);
    bulk_g2s(stage + slot * 2 * kStageTok + kStageTok, hi_g + (int64_t)st * kStageTok, bytes, &bars[slot]);
  };
  if (tid == 0)
    for (int st = 0; st < min(kStages, n_stages); ++st) issue(st);

  if (warp < G) {  // encode query head hk * G + warp (sweep.cpp:92-94)
    const T* qp = reinterpret_cast<const T*>(p.q) + ((int64_t)si * n_q + (int64_t)hk * G + warp) * kHeadDim;
    float f[4];
    Raw4<T>::to_float(Raw4<T>::load(qp + lane * 4), f);
    Code c;
    if (!encode128_warp(f, sqs + warp * kHeadDim, c) && lane == 0) atomicOr(p.status, kStatusDegenerate);
    if (lane == 0) qcode[warp] = c;
  }
  if (has_new && warp == (G % kFusedWarps)) {  // append (kv_cache.cpp:62-71)
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
    if (!encode128_warp(f, sqs + warp * kHeadDim, c) && lane == 0) atomicOr(p.status, kStatusDegenerate);
    if (lane == 0) {
      qcode[G] = c;
      store_code(planes, cap, s_old, c);
    }
  }
  __syncthreads();
  QCode qc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) qc[g] = make_qcode(qcode[g]);

  // ---------------------------------------------------------------- scan
  for (int st = 0; st < n_stages; ++st) {
    const int slot = st % kStages;
    mbar_wait(&bars[slot], (uint32_t)(st / kStages) & 1u);
    const uint4* slo = stage + slot * 2 * kStageTok;
    const uint4* shi = slo + kStageTok;
    const int base = st * kStageTok;
    const int ntok = min(kStageTok, mem_len - base);
    for (int j = tid; j < ntok; j += kFusedThreads) {
      const uint4 a = slo[j], b = shi[j];
      const uint32_t lo[4] = {a.x, a.y, a.z, a.w}, hi[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint32_t d = l1_distance(qc[g], lo, hi);
        dist[g * p.chunk + base + j] = (uint16_t)d;
        atomicAdd(&hist[g * kHistBins + d], 1);
      }
    }
    __syncthreads();
    if (tid == 0 && st + kStages < n_stages) issue(st + kStages);
  }
  if (has_new && tid < G) {  // the appended token is a candidate
    const Code nc = qcode[G];
    const uint32_t d = l1_distance(make_qcode(qcode[tid]), nc.lo, nc.hi);
    dist[tid * p.chunk + (int)(s_old - start)] = (uint16_t)d;
    atomicAdd(&hist[tid * kHistBins + d], 1);
  }
  cluster.sync();  // #1: every rank's histogram is final

  // ---------------------------------------------------------------- select
  const int k_eff = (int)min((int64_t)p.budget, S);
  int* sc = scal;  // per g: [0] T, [1] below, [2] pre_lt, [3] pre_eq, [4] own_lt, [5] own_eq
  __shared__ int scan_scratch[96];
  __shared__ int row_tot[2];
#pragma unroll 1
  for (int g = 0; g < G; ++g) {
    const int b0 = 2 * tid, b1 = 2 * tid + 1;
    int tot0 = 0, tot1 = 0, pre0 = 0, pre1 = 0;
    for (int r = 0; r < C; ++r) {
      const int* rh = cluster.map_shared_rank(hist, r) + g * kHistBins;
      const int2 h = *reinterpret_cast<const int2*>(rh + b0);
      tot0 += h.x;
      tot1 += h.y;
      if (r < rank) { pre0 += h.x; pre1 += h.y; }
    }
    const int own0 = hist[g * kHistBins + b0], own1 = hist[g * kHistBins + b1];
    int etot, epre, eown;
    block_scan3(tot0 + tot1, pre0 + pre1, own0 + own1, scan_scratch, etot, epre, eown);
    if (etot < k_eff && etot + tot0 >= k_eff) {
      sc[g * 6 + 0] = b0; sc[g * 6 + 1] = etot; sc[g * 6 + 2] = epre; sc[g * 6 + 3] = pre0;
      sc[g * 6 + 4] = eown; sc[g * 6 + 5] = own0;
    } else if (etot + tot0 < k_eff && etot + tot0 + tot1 >= k_eff) {
      sc[g * 6 + 0] = b1; sc[g * 6 + 1] = etot + tot0; sc[g * 6 + 2] = epre + pre0; sc[g * 6 + 3] = pre1;
      sc[g * 6 + 4] = eown + own0; sc[g * 6 + 5] = own1;
    }
  }
  __syncthreads();

  // order-preserving compaction: warp w walks 256-token slabs of its range
  const int n_slab = (len + 255) / 256;
#pragma unroll 1
  for (int g = 0; g < G; ++g) {
    const int thr = sc[g * 6 + 0], below = sc[g * 6 + 1], pre_lt = sc[g * 6 + 2], pre_eq = sc[g * 6 + 3];
    const int need = k_eff - below;                     // ties at T the whole head takes
    const int eq_budget = max(0, need - pre_eq);        // ... of which this rank may take
    const int out_off = pre_lt + min(pre_eq, need);     // selected tokens in earlier ranks
    const uint16_t* dg = dist + g * p.chunk;
    // rows of kFusedWarps slabs in index order; thread order == token order
    int run_lt = 0, run_eq = 0;  // CTA-wide counts before the current slab row
    for (int row0 = 0; row0 < n_slab; row0 += kFusedWarps) {
      const int sl = row0 + warp;
      const int t0 = sl * 256 + lane * 8;
      int lt = 0, eq = 0;
      uint32_t ltm = 0, eqm = 0;
      if (sl < n_slab && t0 < len) {
        const uint4 v = *reinterpret_cast<const uint4*>(dg + t0);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int d = (int)((w[e >> 1] >> (16 * (e & 1))) & 0xffffu);
          const bool valid = t0 + e < len;
          if (valid && d < thr) ltm |= 1u << e;
          if (valid && d == thr) eqm |= 1u << e;
        }
        lt = __popc(ltm);
        eq = __popc(eqm);
      }
      int elt, eeq, dummy;
      block_scan3(lt, eq, 0, scan_scratch, elt, eeq, dummy);
      // CTA-wide exclusive counts for this lane's 8 tokens
      const int lt_before = run_lt + elt, eq_before = run_eq + eeq;
      int pos = lt_before + min(eq_before, eq_budget);
      int eq_seen = eq_before;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        bool take = (ltm >> e) & 1u;
        if ((eqm >> e) & 1u) {
          take = eq_seen < eq_budget;
          ++eq_seen;
        }
        if (take) {
          const int tok = (int)start + t0 + e;
          if (pos < selcap) sel[g * selcap + pos] = tok;
          if (p.idx) p.idx[((int64_t)si * n_q + (int64_t)hk * G + g) * p.budget + out_off + pos] = tok;
          ++pos;
        }
      }
      // totals of this row of slabs
      if (tid == kFusedThreads - 1) { row_tot[0] = elt + lt; row_tot[1] = eeq + eq; }
      __syncthreads();
      run_lt += row_tot[0];
      run_eq += row_tot[1];
      __syncthreads();
    }
    if (tid == 0) scal[48 + g] = min(run_lt + min(run_eq, eq_budget), selcap);  // rows this rank attends
  }
  if (rank == 0 && p.idx) {  // estimator.cpp:80 caps the selection at S
    for (int g = 0; g < G; ++g)
      for (int i = k_eff + tid; i < p.budget; i += kFusedThreads)
        p.idx[((int64_t)si * n_q + (int64_t)hk * G + g) * p.budget + i] = -1;
  }
  __syncthreads();

  // ---------------------------------------------------------------- attend
  {
    constexpr int WG = kFusedWarps / G;  // warps per q-head
    const int g = warp % G, sub = warp / G;
    const int nsel = scal[48 + g];
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
    for (int r0 = sub; r0 < nsel; r0 += WG * B) {
      typename Raw4<T>::V kr[B], vr[B];
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int r = r0 + b * WG;
        if (r < nsel) {
          const int64_t t = sel[g * selcap + r];
          kr[b] = Raw4<T>::load(Kh + t * kHeadDim);
          vr[b] = Raw4<T>::load(Vh + t * kHeadDim);
        }
      }
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int r = r0 + b * WG;
        if (r < nsel) {
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
    float* wp = wpart + warp * kPartStride;
    if (lane == 0) { wp[0] = m; wp[1] = l; }
#pragma unroll
    for (int j = 0; j < 4; ++j) wp[4 + lane * 4 + j] = o[j];
    __syncthreads();
    if (sub == 0) {  // combine this head's WG warp partials, push to the merging rank
      float M = -INFINITY;
      for (int s2 = 0; s2 < WG; ++s2) M = fmaxf(M, wpart[(s2 * G + g) * kPartStride]);
      float Lsum = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
      for (int s2 = 0; s2 < WG; ++s2) {
        const float* q2 = wpart + (s2 * G + g) * kPartStride;
        if (q2[1] == 0.f) continue;
        const float c = exp2f(q2[0] - M);
        Lsum += q2[1] * c;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] += q2[4 + lane * 4 + j] * c;
      }
      float* dst = cluster.map_shared_rank(inbox, g % C) + (rank * G + g) * kPartStride;
      if (lane == 0) { dst[0] = M; dst[1] = Lsum; }
      *reinterpret_cast<float4*>(dst + 4 + lane * 4) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    }
  }
  cluster.sync();  // #2: partials delivered; no rank touches remote smem after this

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
      const float4 v = *reinterpret_cast<const float4*>(q2 + 4 + lane * 4);
      acc[0] += v.x * c; acc[1] += v.y * c; acc[2] += v.z * c; acc[3] += v.w * c;
    }
    const float inv = 1.f / Lsum;
    float* op = p.out + ((int64_t)si * n_q + (int64_t)hk * G + g) * kHeadDim + lane * 4;
    *reinterpret_cast<float4*>(op) = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
  }
}

}  // namespace adamas_dev
