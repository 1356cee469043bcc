// harness_select.cuh — f3: the GPU backend for the sweep
// harness's selection step, in the harness's own arithmetic (fp64 inputs) at
// every head_dim the harness accepts (power of two, 2..1024) and every code
// width the reference quantizer has (1, 2, 3 bits):
//
//   hsel_encode_kernel      build_cache (sweep.cpp:38-50) / encode (sweep.cpp:32-36):
//                           fwht (kernels_scalar.cpp:11-35), compute_thresholds
//                           (quantizer.cpp:40-64), bucketize (quantizer.cpp:74-85)
//   hsel_score_kernel       score_all (estimator.cpp:45-73), l1/l2 over 1/2-bit
//                           planes (kernels_scalar.cpp:65-97) or 3-bit bytes (:99-115)
//   hsel_topk_kernel        top_k (estimator.cpp:75-90) and top_k_by_score
//                           (baselines.cpp:21-32) as one radix select
//   hsel_dot_kernel         the oracle policy's dot scores (sweep.cpp:202-204, common.hpp:65-69)
//   hsel_page_*_kernel      quest: PageSummaries::append / page_scores / page_select
//                           (baselines.cpp:40-91)
//   hsel_attention_kernel   full_attention (attention.cpp:8-38) over all rows or a
//                           selection (attend_subset, sweep.cpp:120-131)
//
// Every fp64 operation is a correctly rounded __d*_rn intrinsic in the
// reference's order (the reference is built without contraction), so codes,
// distances, dot scores and page scores are bit-identical to the reference's.
// The attention uses CUDA's exp(), which may differ from libm's in the last
// place: its output is checked to a tolerance, not bitwise.
#pragma once

#include "common.cuh"

namespace adamas_dev {

constexpr int kHselMaxDim = 1024;
constexpr int kHselWarps = 4;  // encode: one vector per warp
// quantizer.cpp:12-14
constexpr double kQ18 = 1.1503493803760081783;
constexpr double kQ38 = 0.31863936396437516302;

// per-call status bits (hsel device status word)
constexpr int kHselZero = 1;       // "degenerate scale: input vector is all zeros" (quantizer.cpp:47)
constexpr int kHselNonFinite = 2;  // "non-finite input to compute_thresholds" (quantizer.cpp:46)

// Element placement. A vector of D = 32 E elements (E >= 1) lives in one warp,
// element j = lane * E + e in lane `lane`, register e; D < 32 uses lanes
// 0..D-1 with E = 1. Code plane word e holds bit `lane` = element lane*E + e:
// a fixed permutation of the reference's packing order. Distances are sums of
// per-element terms and query and keys are permuted alike, so they are
// unchanged; hsel_codes_ref_kernel undoes the permutation for export.
__host__ __device__ constexpr int hsel_words(int D) { return D >= 32 ? D / 32 : 1; }

// fwht_scalar (kernels_scalar.cpp:11-21): stage h pairs j, j + h (bit h of j
// clear) -> ((a + b) c, (a - b) c), c = 1/sqrt(2), stages h = 1, 2, 4, ...
template <int E>
__device__ __forceinline__ void hsel_fwht(double (&x)[E], int D) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int h = 1; h < E; h <<= 1) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e & h) continue;
      const double a = x[e], b = x[e + h];
      x[e] = __dmul_rn(__dadd_rn(a, b), kInvSqrt2);
      x[e + h] = __dmul_rn(__dsub_rn(a, b), kInvSqrt2);
    }
  }
  for (int m = 1; m * E < D; m <<= 1) {  // h = m E: partner lane ^ m, same register
    const bool upper = (lane & m) != 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const double p = __shfl_xor_sync(kFull, x[e], m);
      x[e] = upper ? __dmul_rn(__dsub_rn(p, x[e]), kInvSqrt2) : __dmul_rn(__dadd_rn(x[e], p), kInvSqrt2);
    }
  }
}

// One warp per vector. planes: [n_vec][2][W] u32 (low code bit, low ^ high
// bit) for bits 1 and 2; bytes: [n_vec][D] (the reference's CodeVector) for 3.
template <int E, int BITS>
__global__ void __launch_bounds__(kHselWarps * 32)
hsel_encode_kernel(const double* __restrict__ x, int64_t n_vec, int D, int hadamard,
                   uint32_t* __restrict__ planes, uint8_t* __restrict__ bytes, int* __restrict__ status) {
  __shared__ double sq[kHselWarps][32 * E];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int bits = BITS;
  const bool active = lane * E < D;
  const int W = hsel_words(D);
  for (int64_t v = (int64_t)blockIdx.x * kHselWarps + warp; v < n_vec; v += (int64_t)gridDim.x * kHselWarps) {
    double r[E];
    const double* src = x + v * D + lane * E;
#pragma unroll
    for (int e = 0; e < E; ++e) r[e] = active ? src[e] : 0.0;
    if (hadamard) hsel_fwht<E>(r, D);
    // compute_thresholds: sum of squares in index order 0..D-1 (quantizer.cpp:43-44).
    // Fast path: a shuffle-tree sum of the same exact products. Two summation
    // orders of n <= 1024 non-negative terms agree to 2 (n - 1) u < 2.3e-13
    // relative, so sigma and every threshold k * sigma agree to < 2e-13; the
    // codes can only differ for an element within that distance of a nonzero
    // threshold (0 does not depend on sigma). If any element is within 1e-12
    // relative of one, or the sum is near the ends of the fp64 range, the warp
    // takes the exact sequential sum instead.
    double sqv[E];
    double s4 = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      sqv[e] = active ? __dmul_rn(r[e], r[e]) : 0.0;
      s4 = __dadd_rn(s4, sqv[e]);
    }
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) s4 = __dadd_rn(s4, __shfl_xor_sync(kFull, s4, m));
    double sigma = __dsqrt_rn(__ddiv_rn(s4, (double)D));
    bool near = !(s4 > 1e-290 && s4 < 1e300);
    if (bits >= 2) {
      const double t28 = __dmul_rn(kQ28, sigma);
      const double t18 = __dmul_rn(kQ18, sigma), t38 = __dmul_rn(kQ38, sigma);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const double a = fabs(r[e]);
        near |= fabs(a - t28) <= 1e-12 * t28;
        if (bits == 3) near |= fabs(a - t18) <= 1e-12 * t18 || fabs(a - t38) <= 1e-12 * t38;
      }
    }
    if (__any_sync(kFull, near)) {
      if (active) {
#pragma unroll
        for (int e = 0; e < E; ++e) sq[warp][lane * E + e] = sqv[e];
      }
      __syncwarp();
      if (lane == 0) {
        double acc = 0.0;
        for (int j = 0; j < D; ++j) acc = __dadd_rn(acc, sq[warp][j]);
        sigma = __dsqrt_rn(__ddiv_rn(acc, (double)D));
      }
      sigma = __shfl_sync(kFull, sigma, 0);
      __syncwarp();  // sq is rewritten for the next vector
    }
    const int bad = !isfinite(sigma) ? kHselNonFinite : (sigma == 0.0 ? kHselZero : 0);
    if (bad && lane == 0) atomicOr(status, bad);
    // thresholds (quantizer.cpp:52-62): -k s is (-k) s, exactly -(k s)
    double t[7];
    int nt;
    if (bits == 1) {
      nt = 1;
      t[0] = 0.0;
    } else if (bits == 2) {
      nt = 3;
      t[0] = __dmul_rn(-kQ28, sigma);
      t[1] = 0.0;
      t[2] = __dmul_rn(kQ28, sigma);
    } else {
      nt = 7;
      t[0] = __dmul_rn(-kQ18, sigma);
      t[1] = __dmul_rn(-kQ28, sigma);
      t[2] = __dmul_rn(-kQ38, sigma);
      t[3] = 0.0;
      t[4] = __dmul_rn(kQ38, sigma);
      t[5] = __dmul_rn(kQ28, sigma);
      t[6] = __dmul_rn(kQ18, sigma);
    }
    uint32_t code[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      uint32_t lvl = 0;
#pragma unroll
      for (int b = 0; b < 7; ++b) lvl += (b < nt && r[e] > t[b]) ? 1u : 0u;  // bucketize: # thresholds below
      code[e] = (active && !bad) ? lvl : 0u;
    }
    if (bits == 3) {
      if (active) {
#pragma unroll
        for (int e = 0; e < E; ++e) bytes[v * D + lane * E + e] = (uint8_t)code[e];
      }
    } else {
      uint32_t mylo = 0, myx = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t lo = __ballot_sync(kFull, code[e] & 1u);
        const uint32_t hi = __ballot_sync(kFull, (code[e] >> 1) & 1u);
        if (lane == e) {
          mylo = lo;
          myx = lo ^ hi;
        }
      }
      if (lane < W) {
        planes[(v * 2 + 0) * W + lane] = mylo;
        planes[(v * 2 + 1) * W + lane] = myx;
      }
    }
  }
}

// Reference-format export: PackedCodes words (quantizer.cpp:87-117: code i at
// bits * (i % per_word) of word i / per_word, zero padded) for bits 1 and 2, the
// CodeVector bytes for 3. One thread per output word / byte.
__global__ void hsel_codes_ref_kernel(const uint32_t* __restrict__ planes, const uint8_t* __restrict__ bytes,
                                      int64_t n_vec, int D, int bits, void* __restrict__ out) {
  const int W = hsel_words(D);
  const int E = D >= 32 ? D / 32 : 1;
  if (bits == 3) {
    uint8_t* o = static_cast<uint8_t*>(out);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_vec * D; i += (int64_t)gridDim.x * blockDim.x)
      o[i] = bytes[i];
    return;
  }
  const int per_word = 16 / bits;
  const int nwords = (D + per_word - 1) / per_word;
  uint16_t* o = static_cast<uint16_t*>(out);
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_vec * nwords;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = g / nwords;
    const int w = (int)(g % nwords);
    const uint32_t* lo = planes + v * 2 * W;
    const uint32_t* xx = lo + W;
    uint32_t word = 0;
    for (int s = 0; s < per_word; ++s) {
      const int i = w * per_word + s;
      if (i >= D) break;
      const int ln = i / E, e = i % E;
      const uint32_t l = (lo[e] >> ln) & 1u, h = ((lo[e] ^ xx[e]) >> ln) & 1u;
      word |= (l | (h << 1)) << (bits * s);
    }
    o[g] = (uint16_t)word;
  }
}

// ------------------------------------------------------------------ scores
// score_all: thread per (row, token). Row r reads instance r / rows_per_inst.
constexpr int kHselScoreThreads = 256;

template <int BITS, int METRIC>
__global__ void __launch_bounds__(kHselScoreThreads)
hsel_score_kernel(const uint32_t* __restrict__ planes, const uint8_t* __restrict__ bytes,
                  const uint32_t* __restrict__ qplanes, const uint8_t* __restrict__ qbytes, int64_t S, int D,
                  int64_t rows_per_inst, uint32_t* __restrict__ scores) {
  __shared__ uint32_t qs[kHselMaxDim / 4 + 64];
  const int64_t row = blockIdx.y;
  const int64_t inst = row / rows_per_inst;
  const int W = hsel_words(D);
  if (BITS == 3) {
    for (int i = threadIdx.x; i < D; i += blockDim.x) reinterpret_cast<uint8_t*>(qs)[i] = qbytes[row * D + i];
  } else {
    for (int i = threadIdx.x; i < 2 * W; i += blockDim.x) qs[i] = qplanes[row * 2 * W + i];
  }
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= S) return;
  uint32_t acc = 0;
  if (BITS == 3) {
    const uint8_t* k = bytes + (inst * S + t) * D;
    const uint8_t* q = reinterpret_cast<const uint8_t*>(qs);
    if (D >= 4) {
      for (int w = 0; w < D / 4; ++w) {
        const uint32_t a = reinterpret_cast<const uint32_t*>(q)[w];
        const uint32_t b = __ldg(reinterpret_cast<const uint32_t*>(k) + w);
        if (METRIC == kMetricManhattan) {
          acc = __vsadu4(a, b) + acc;  // kernels_scalar.cpp:99-106
        } else {
          const uint32_t d = __vabsdiffu4(a, b);  // kernels_scalar.cpp:108-115: sum of d^2
          acc = __dp4a(d, d, acc);
        }
      }
    } else {
      for (int i = 0; i < D; ++i) {
        const int d = (int)q[i] - (int)k[i];
        acc += METRIC == kMetricManhattan ? (uint32_t)(d < 0 ? -d : d) : (uint32_t)(d * d);
      }
    }
  } else {
    const uint32_t* klo = planes + (inst * S + t) * 2 * W;
    const uint32_t* kx = klo + W;
    for (int w = 0; w < W; ++w) {
      const uint32_t ql = qs[w], qx = qs[W + w];
      const uint32_t L = ql ^ __ldg(klo + w);
      if (BITS == 1) {
        acc += __popc(L);  // l1_1bit_words: popcount(q ^ k) for both metrics (estimator.cpp:51-52)
      } else {
        const uint32_t Hd = qx ^ __ldg(kx + w) ^ L;  // high-bit difference
        if (METRIC == kMetricManhattan) {
          acc += __popc(L) + 2u * __popc(Hd & ~(L & qx));  // |a-b| = L + 2A (common.cuh l1_distance)
        } else {
          const uint32_t cr = Hd & L;  // (a-b)^2 = L + 4Hd + 4(Hd L ~X) - 4(Hd L X) (ops.cuh plane_distance)
          acc += __popc(L) + 4u * __popc(Hd) + 4u * __popc(cr & ~qx) - 4u * __popc(cr & qx);
        }
      }
    }
  }
  scores[row * S + t] = acc;
}

// -------------------------------------------------------------------- top-k
// One CTA per row, radix select over order keys (8-bit digits, high to low):
// the k smallest keys under (key, index), ties toward the smaller index, written
// as ascending indices (no sort: an order-preserving compaction). MODE 0: u32
// distances ascending (top_k, estimator.cpp:75-90); MODE 1: fp64 scores
// descending (top_k_by_score, baselines.cpp:21-32; -0.0 and +0.0 compare equal
// there, so both map to the key of +0.0).
constexpr int kHselTopkThreads = 1024;

template <int MODE>
__device__ __forceinline__ uint64_t hsel_key(const void* scores, int64_t i) {
  if (MODE == 0) return static_cast<const uint32_t*>(scores)[i];
  double s = static_cast<const double*>(scores)[i];
  if (s == 0.0) s = 0.0;
  const uint64_t u = (uint64_t)__double_as_longlong(s);
  const uint64_t ord = (u >> 63) ? ~u : (u | 0x8000000000000000ull);  // ascending in value
  return ~ord;                                                           // descending in value
}

__device__ __forceinline__ int64_t hsel_block_flag_scan(bool flag, int* scratch, int64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t b = __ballot_sync(kFull, flag);
  if (lane == 0) scratch[warp] = __popc(b);
  __syncthreads();
  int before = 0, sum = 0;
  for (int w = 0; w < nwarps; ++w) {
    const int v = scratch[w];
    before += (w < warp) ? v : 0;
    sum += v;
  }
  __syncthreads();
  *total = sum;
  return before + __popc(b & ((1u << lane) - 1u));
}

template <int MODE>
__global__ void __launch_bounds__(kHselTopkThreads)
hsel_topk_kernel(const void* __restrict__ scores, int64_t n, int64_t k, int64_t* __restrict__ idx) {
  __shared__ unsigned hist[256];
  __shared__ int scratch[32];
  __shared__ uint64_t s_prefix;
  __shared__ int64_t s_need;
  const int64_t row = blockIdx.x;
  const void* s = MODE == 0 ? (const void*)(static_cast<const uint32_t*>(scores) + row * n)
                            : (const void*)(static_cast<const double*>(scores) + row * n);
  int64_t* out = idx + row * k;
  const int64_t keep = k < n ? k : n;
  for (int64_t i = keep + threadIdx.x; i < k; i += blockDim.x) out[i] = -1;
  if (k >= n) {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = i;
    return;
  }
  if (k == 0) return;
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_need = k;
  }
  constexpr int kBits = MODE == 0 ? 32 : 64;
  for (int shift = kBits - 8; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint64_t prefix = s_prefix;
    const uint64_t hi_mask = shift + 8 >= 64 ? 0ull : (~0ull << (shift + 8));
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint64_t key = hsel_key<MODE>(s, i);
      if ((key & hi_mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // digit whose cumulative count reaches the remaining need
      const int lane = threadIdx.x;
      unsigned c[8], sum = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = hist[lane * 8 + j];
        sum += c[j];
      }
      unsigned incl = sum;
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        const unsigned o = __shfl_up_sync(kFull, incl, m);
        if (lane >= m) incl += o;
      }
      const int64_t need = s_need;
      unsigned before = incl - sum;
      bool found = false;
      int digit = 0;
      unsigned below = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (!found && (int64_t)before < need && (int64_t)(before + c[j]) >= need) {
          found = true;
          digit = lane * 8 + j;
          below = before;
        }
        before += c[j];
      }
      __syncwarp();
      if (found) {
        s_prefix = prefix | ((uint64_t)digit << shift);
        s_need = need - below;
      }
    }
    __syncthreads();
  }
  const uint64_t T = s_prefix;
  const int64_t need = s_need;  // keys equal to T to take, in index order
  int64_t eq_seen = 0, taken = 0;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const uint64_t key = i < n ? hsel_key<MODE>(s, i) : ~0ull;
    const bool eq = (i < n) && key == T;
    int64_t eq_total, take_total;
    const int64_t eq_before = eq_seen + hsel_block_flag_scan(eq, scratch, &eq_total);
    const bool take = (i < n) && (key < T || (eq && eq_before < need));
    const int64_t pos = taken + hsel_block_flag_scan(take, scratch, &take_total);
    if (take) out[pos] = i;
    eq_seen += eq_total;
    taken += take_total;
    if (taken >= keep) break;
  }
}

// --------------------------------------------------------------- dot scores
// dot(q, key) (common.hpp:65-69): acc += q_j k_j, j ascending, one thread per
// token; keys staged through shared memory 32 columns at a time (coalesced).
constexpr int kHselDotTok = 128;

__device__ __forceinline__ double hsel_dot_tile(const double* __restrict__ keys, const double* qs, int64_t S,
                                                int D, int64_t inst, int64_t t0, double (*tile)[33]) {
  double acc = 0.0;
  for (int j0 = 0; j0 < D; j0 += 32) {
    const int jw = D - j0 < 32 ? D - j0 : 32;
    for (int i = threadIdx.x; i < kHselDotTok * 32; i += kHselDotTok) {
      const int r = i >> 5, c = i & 31;
      const int64_t tr = t0 + r;
      tile[r][c] = (tr < S && c < jw) ? keys[(inst * S + tr) * D + j0 + c] : 0.0;
    }
    __syncthreads();
    for (int c = 0; c < jw; ++c) acc = __dadd_rn(acc, __dmul_rn(qs[j0 + c], tile[threadIdx.x][c]));
    __syncthreads();
  }
  return acc;
}

__global__ void __launch_bounds__(kHselDotTok)
hsel_dot_kernel(const double* __restrict__ q, const double* __restrict__ keys, int64_t S, int D,
                int64_t rows_per_inst, double* __restrict__ out) {
  __shared__ double qs[kHselMaxDim];
  __shared__ double tile[kHselDotTok][33];
  const int64_t row = blockIdx.y, inst = row / rows_per_inst;
  for (int j = threadIdx.x; j < D; j += blockDim.x) qs[j] = q[row * D + j];
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * kHselDotTok;
  const double acc = hsel_dot_tile(keys, qs, S, D, inst, t0, tile);
  if (t0 + threadIdx.x < S) out[row * S + t0 + threadIdx.x] = acc;
}

// ------------------------------------------------------------------- quest
// PageSummaries::append (baselines.cpp:40-54): per (instance, page, channel)
// the running std::min / std::max over the page's keys in token order.
__global__ void hsel_page_summary_kernel(const double* __restrict__ keys, int64_t n_inst, int64_t S, int D,
                                         int64_t page_size, double* __restrict__ mins, double* __restrict__ maxs) {
  const int64_t P = (S + page_size - 1) / page_size;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_inst * P * D;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(g % D);
    const int64_t p = (g / D) % P, inst = g / (D * P);
    const int64_t first = p * page_size, last = min(first + page_size, S);
    const double* k = keys + (inst * S) * D + j;
    double mn = k[first * D], mx = mn;
    for (int64_t i = first + 1; i < last; ++i) {
      const double v = k[i * D];
      mn = v < mn ? v : mn;  // std::min(mn, v)
      mx = mx < v ? v : mx;  // std::max(mx, v)
    }
    mins[g] = mn;
    maxs[g] = mx;
  }
}

// page_scores (baselines.cpp:57-69): s += std::max(q_j mn_j, q_j mx_j), j ascending.
// CTA = 128 pages of one query row; page summaries staged 16 channels at a time.
constexpr int kHselPageTile = 128;

__global__ void __launch_bounds__(kHselPageTile)
hsel_page_score_kernel(const double* __restrict__ q, const double* __restrict__ mins, const double* __restrict__ maxs,
                       int64_t rows_per_inst, int64_t P, int D, double* __restrict__ scores) {
  __shared__ double qs[kHselMaxDim];
  __shared__ double tmn[kHselPageTile][17], tmx[kHselPageTile][17];
  const int64_t row = blockIdx.y, inst = row / rows_per_inst;
  const int64_t p0 = (int64_t)blockIdx.x * kHselPageTile;
  for (int j = threadIdx.x; j < D; j += blockDim.x) qs[j] = q[row * D + j];
  const double* mn = mins + inst * P * D;
  const double* mx = maxs + inst * P * D;
  double sc = 0.0;
  for (int j0 = 0; j0 < D; j0 += 16) {
    const int jw = D - j0 < 16 ? D - j0 : 16;
    __syncthreads();
    for (int i = threadIdx.x; i < kHselPageTile * 16; i += kHselPageTile) {
      const int r = i >> 4, c = i & 15;
      const int64_t pr = p0 + r;
      const bool ok = pr < P && c < jw;
      tmn[r][c] = ok ? mn[pr * D + j0 + c] : 0.0;
      tmx[r][c] = ok ? mx[pr * D + j0 + c] : 0.0;
    }
    __syncthreads();
    for (int c = 0; c < jw; ++c) {
      const double a = __dmul_rn(qs[j0 + c], tmn[threadIdx.x][c]), b = __dmul_rn(qs[j0 + c], tmx[threadIdx.x][c]);
      sc = __dadd_rn(sc, a < b ? b : a);
    }
  }
  if (p0 + threadIdx.x < P) scores[row * P + p0 + threadIdx.x] = sc;
}

// page_select (baselines.cpp:71-91): the selected pages (ascending) expanded to
// their token ranges; only the last page can be partial and it sorts last.
__global__ void hsel_page_expand_kernel(const int64_t* __restrict__ pages, int64_t kp, int64_t S, int64_t page_size,
                                        int64_t budget, int64_t* __restrict__ idx, int64_t* __restrict__ counts) {
  const int64_t row = blockIdx.x;
  const int64_t* pr = pages + row * kp;
  int64_t* out = idx + row * budget;
  for (int64_t i = threadIdx.x; i < budget; i += blockDim.x) {
    const int64_t r = i / page_size, o = i % page_size;
    const int64_t t = r < kp ? pr[r] * page_size + o : S;
    out[i] = t < S ? t : -1;
  }
  if (threadIdx.x == 0) {
    const int64_t lastp = pr[kp - 1];
    counts[row] = kp * page_size - (lastp * page_size + page_size > S ? lastp * page_size + page_size - S : 0);
  }
}

__global__ void hsel_fill_kernel(int64_t* __restrict__ p, int64_t n, int64_t v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// --------------------------------------------------------------- attention
// full_attention (attention.cpp:8-38) over rows idx[0..count) (all S rows when
// idx is null): logits = dot(q, k_i) * (1 / sqrt(d)), peak, l_i = exp(l_i - peak),
// denom = sum in row order, out_j = sum_i (l_i / denom) v_ij in row order.
// One CTA per query row; logits in global scratch [rows][n_max].
constexpr int kHselAttnThreads = 256;

__global__ void __launch_bounds__(kHselAttnThreads)
hsel_attention_kernel(const double* __restrict__ q, const double* __restrict__ K, const double* __restrict__ V,
                      int64_t S, int D, int64_t rows_per_inst, const int64_t* __restrict__ idx, int64_t idx_stride,
                      const int64_t* __restrict__ counts, double* __restrict__ logits, int64_t n_max,
                      double* __restrict__ out) {
  __shared__ double red[kHselAttnThreads / 32];
  __shared__ double s_peak, s_denom;
  const int64_t row = blockIdx.x, inst = row / rows_per_inst;
  const int64_t n = idx ? (counts ? counts[row] : idx_stride) : S;
  const int64_t* ir = idx ? idx + row * idx_stride : nullptr;
  const double* qq = q + row * D;
  const double* Kb = K + inst * S * D;
  const double* Vb = V + inst * S * D;
  double* lg = logits + row * n_max;
  const double scale = __ddiv_rn(1.0, __dsqrt_rn((double)D));
  double mx = -INFINITY;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t t = ir ? ir[i] : i;
    const double* k = Kb + t * D;
    double acc = 0.0;
    for (int j = 0; j < D; ++j) acc = __dadd_rn(acc, __dmul_rn(qq[j], k[j]));
    const double l = __dmul_rn(acc, scale);
    lg[i] = l;
    mx = fmax(mx, l);
  }
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, m));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double p = red[0];
    for (int w = 1; w < kHselAttnThreads / 32; ++w) p = fmax(p, red[w]);
    s_peak = p;
  }
  __syncthreads();
  const double peak = s_peak;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) lg[i] = exp(__dsub_rn(lg[i], peak));
  __syncthreads();
  if (threadIdx.x == 0) {
    double den = 0.0;
    for (int64_t i = 0; i < n; ++i) den = __dadd_rn(den, lg[i]);
    s_denom = den;
  }
  __syncthreads();
  const double den = s_denom;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) lg[i] = __ddiv_rn(lg[i], den);
  __syncthreads();
  for (int j = threadIdx.x; j < D; j += blockDim.x) {
    double o = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const int64_t t = ir ? ir[i] : i;
      o = __dadd_rn(o, __dmul_rn(lg[i], Vb[t * D + j]));
    }
    out[row * D + j] = o;
  }
}

}  // namespace adamas_dev
