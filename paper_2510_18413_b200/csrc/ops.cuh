// ops.cuh — operator-level kernels behind the C ABI (one kernel per reference
// operator): encode+append, query encode, score_all, top_k, sparse_attention.
// The fused single-launch decode step lives in fused_decode.cuh.
#pragma once
#include "common.cuh"

namespace adamas_dev {

// ----------------------------------------------------------------- raw moves
template <typename T>
struct Raw4;  // four consecutive elements as one vector register
template <>
struct Raw4<float> {
  using V = float4;
  __device__ static __forceinline__ V load(const float* p) { return *reinterpret_cast<const float4*>(p); }
  __device__ static __forceinline__ void store(float* p, V v) { *reinterpret_cast<float4*>(p) = v; }
  __device__ static __forceinline__ void to_float(V v, float f[4]) {
    f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
  }
};
template <>
struct Raw4<__nv_bfloat16> {
  using V = uint2;
  __device__ static __forceinline__ V load(const __nv_bfloat16* p) { return *reinterpret_cast<const uint2*>(p); }
  __device__ static __forceinline__ void store(__nv_bfloat16* p, V v) { *reinterpret_cast<uint2*>(p) = v; }
  __device__ static __forceinline__ void to_float(V v, float f[4]) {
    f[0] = __uint_as_float(v.x << 16);
    f[1] = __uint_as_float(v.x & 0xffff0000u);
    f[2] = __uint_as_float(v.y << 16);
    f[3] = __uint_as_float(v.y & 0xffff0000u);
  }
};

// Reference-layout code byte of lane l (elements 4l..4l+3) -> four 2-bit codes.
// (PackedCodes words are little-endian u16, so byte l of the 32-byte row holds
// elements 4l..4l+3 at bit offsets 0, 2, 4, 6.)
__device__ __forceinline__ void planes_from_ref_byte(uint32_t byte, Code& out) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t c = (byte >> (2 * j)) & 3u;
    out.lo[j] = __ballot_sync(kFull, c & 1u);
    out.hi[j] = __ballot_sync(kFull, c >> 1);
  }
}
__device__ __forceinline__ uint32_t ref_byte_from_planes(const Code& c, int lane) {
  uint32_t b = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t code = ((c.lo[j] >> lane) & 1u) | (((c.hi[j] >> lane) & 1u) << 1);
    b |= code << (2 * j);
  }
  return b;
}
__device__ __forceinline__ uint32_t ref_byte_from_codes(const uint32_t code[4]) {
  return code[0] | (code[1] << 2) | (code[2] << 4) | (code[3] << 6);
}

// planes: the kv-head's lo plane base; the x plane (lo ^ hi) is `cap` records later.
__device__ __forceinline__ void store_code(uint4* planes, int64_t cap, int64_t t, const Code& c) {
  planes[t] = make_uint4(c.lo[0], c.lo[1], c.lo[2], c.lo[3]);
  planes[cap + t] = make_uint4(c.lo[0] ^ c.hi[0], c.lo[1] ^ c.hi[1], c.lo[2] ^ c.hi[2], c.lo[3] ^ c.hi[3]);
}
__device__ __forceinline__ Code load_code(const uint4* planes, int64_t cap, int64_t t) {
  const uint4 a = planes[t], b = planes[cap + t];
  Code c;
  c.lo[0] = a.x; c.lo[1] = a.y; c.lo[2] = a.z; c.lo[3] = a.w;
  c.hi[0] = a.x ^ b.x; c.hi[1] = a.y ^ b.y; c.hi[2] = a.z ^ b.z; c.hi[3] = a.w ^ b.w;
  return c;
}

// ----------------------------------------------------------------- append
// Bulk encode + append (the build_cache loop, sweep.cpp:38-50, and
// KvCache::update, kv_cache.cpp:62-71). A warp takes a block of kAppendNV
// consecutive tokens of ONE kv-head: their K/V rows are loaded (one 256-B row
// per vector for bf16, coalesced), encoded together (independent shuffle
// chains interleave), written to the head's rows, and their codes land as
// kAppendNV consecutive 16-B records per plane (lanes 0..NV-1: one coalesced
// store per plane). The next block's rows are loaded before the current one is
// encoded, so the HBM latency overlaps the encode.
constexpr int kAppendWarps = 8;
#ifndef ADAMAS_APPEND_NV
#define ADAMAS_APPEND_NV 2  // measured: 2 -> 434 us, 4 -> 465, 8 -> 610 for 32 heads x 32K (bf16)
#endif
constexpr int kAppendNV = ADAMAS_APPEND_NV;

template <typename T, bool kCoded>
__global__ void __launch_bounds__(kAppendWarps * 32)
append_kernel(const T* __restrict__ keys, const T* __restrict__ values,
              const uint16_t* __restrict__ codes_ref, int64_t n_vec, int n_kv, int64_t seq0,
              int64_t cap, T* __restrict__ K, T* __restrict__ V, uint4* __restrict__ codes,
              int* __restrict__ status) {
  __shared__ double sq[kAppendWarps][kHeadDim];
  constexpr int NV = kAppendNV;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n_tok = (int)(n_vec / n_kv);                  // < 2^31 (capacity bound)
  const int nblocks = (n_tok + NV - 1) / NV * n_kv;     // (token block, kv-head) pairs
  const int stride = gridDim.x * kAppendWarps;
  using R = typename Raw4<T>::V;
  auto load = [&](int b, R (&kr)[NV], R (&vr)[NV]) {
    const int h = b % n_kv;
    const int64_t t0 = (int64_t)(b / n_kv) * NV;
#pragma unroll
    for (int n = 0; n < NV; ++n) {
      const int64_t t = min(t0 + n, (int64_t)n_tok - 1);
      const int64_t off = (t * n_kv + h) * kHeadDim + lane * 4;
      kr[n] = Raw4<T>::load(keys + off);
      vr[n] = Raw4<T>::load(values + off);
    }
  };
  R kr[NV], vr[NV], krn[NV], vrn[NV];
  int b = blockIdx.x * kAppendWarps + warp;
  if (b < nblocks) load(b, kr, vr);
  for (; b < nblocks; b += stride) {
    if (b + stride < nblocks) load(b + stride, krn, vrn);  // the next block is in flight during this one
    const int h = b % n_kv;
    const int64_t t0 = (int64_t)(b / n_kv) * NV;
    const int nv = (int)min((int64_t)NV, (int64_t)n_tok - t0);
    Code c[NV];
    if constexpr (kCoded) {
#pragma unroll
      for (int n = 0; n < NV; ++n) {
        const int64_t t = min(t0 + n, (int64_t)n_tok - 1);
        planes_from_ref_byte(reinterpret_cast<const uint8_t*>(codes_ref + (t * n_kv + h) * 16)[lane], c[n]);
      }
    } else {
      float f[NV][4];
      int res[NV];
#pragma unroll
      for (int n = 0; n < NV; ++n) Raw4<T>::to_float(kr[n], f[n]);
      encode128_warp_f32n<NV>(f, c, res);
#pragma unroll
      for (int n = 0; n < NV; ++n) {
        if (res[n] < 0) res[n] = encode128_warp(f[n], sq[warp], c[n], true) ? 1 : 0;  // exact fallback
        if (res[n] == 0 && lane == 0 && n < nv) atomicOr(status, kStatusDegenerate);
      }
    }
    const int64_t row0 = (int64_t)h * cap + seq0 + t0;
#pragma unroll
    for (int n = 0; n < NV; ++n) {
      if (n < nv) {
        Raw4<T>::store(K + (row0 + n) * kHeadDim + lane * 4, kr[n]);
        Raw4<T>::store(V + (row0 + n) * kHeadDim + lane * 4, vr[n]);
      }
    }
    // codes: lane n < nv writes token t0 + n's record in both planes
    uint4 lo = make_uint4(0, 0, 0, 0), xx = lo;
#pragma unroll
    for (int n = 0; n < NV; ++n)
      if (lane == n) {
        lo = make_uint4(c[n].lo[0], c[n].lo[1], c[n].lo[2], c[n].lo[3]);
        xx = make_uint4(c[n].lo[0] ^ c[n].hi[0], c[n].lo[1] ^ c[n].hi[1], c[n].lo[2] ^ c[n].hi[2],
                        c[n].lo[3] ^ c[n].hi[3]);
      }
    if (lane < nv) {
      uint4* planes = codes + (int64_t)h * 2 * cap;
      planes[seq0 + t0 + lane] = lo;
      planes[cap + seq0 + t0 + lane] = xx;
    }
#pragma unroll
    for (int n = 0; n < NV; ++n) { kr[n] = krn[n]; vr[n] = vrn[n]; }
  }
}

// Sixteen consecutive elements (one lane's share of a vector in the 8-lane
// layout) as raw registers: 32 B (bf16) or 64 B (fp32).
template <typename T>
struct Raw16;
template <>
struct Raw16<__nv_bfloat16> {
  uint4 r[2];
  __device__ __forceinline__ void load(const __nv_bfloat16* p) {
    r[0] = __ldcs(reinterpret_cast<const uint4*>(p));
    r[1] = __ldcs(reinterpret_cast<const uint4*>(p) + 1);
  }
  __device__ __forceinline__ void store(__nv_bfloat16* p) const {
    reinterpret_cast<uint4*>(p)[0] = r[0];
    reinterpret_cast<uint4*>(p)[1] = r[1];
  }
  __device__ __forceinline__ void to_float(float (&f)[16]) const {
    const uint32_t w[8] = {r[0].x, r[0].y, r[0].z, r[0].w, r[1].x, r[1].y, r[1].z, r[1].w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
};
template <>
struct Raw16<float> {
  float4 r[4];
  __device__ __forceinline__ void load(const float* p) {
#pragma unroll
    for (int i = 0; i < 4; ++i) r[i] = __ldcs(reinterpret_cast<const float4*>(p) + i);
  }
  __device__ __forceinline__ void store(float* p) const {
#pragma unroll
    for (int i = 0; i < 4; ++i) reinterpret_cast<float4*>(p)[i] = r[i];
  }
  __device__ __forceinline__ void to_float(float (&f)[16]) const {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[4 * i] = r[i].x; f[4 * i + 1] = r[i].y; f[4 * i + 2] = r[i].z; f[4 * i + 3] = r[i].w;
    }
  }
};

// Bulk prefill (kv_cache.cpp:62-71 per vector, sweep.cpp:38-50's build loop):
// each warp encodes four consecutive input vectors per iteration through the
// 8-lane certified encoder (encode128_g8_f32: about half the instructions of
// the 32-lane route per vector, which made append_kernel issue-bound), copies
// their K / V rows into the cache and stores the codes; a group whose vector
// misses the certificate is re-encoded exactly by the whole warp. The next
// iteration's rows are loaded before this one is encoded.
constexpr int kAppend8Warps = 8;
template <typename T>
__global__ void __launch_bounds__(kAppend8Warps * 32)
append8_kernel(const T* __restrict__ keys, const T* __restrict__ values, int64_t n_vec, int n_kv, int64_t seq0,
               int64_t cap, T* __restrict__ K, T* __restrict__ V, uint4* __restrict__ codes,
               int* __restrict__ status) {
  __shared__ double sq[kAppend8Warps][kHeadDim];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, grp = lane >> 3, L = lane & 7;
  const int64_t stride = (int64_t)gridDim.x * kAppend8Warps * 4;
  int64_t b0 = ((int64_t)blockIdx.x * kAppend8Warps + warp) * 4;  // this warp's first vector
  Raw16<T> kr, vr, krn, vrn;
  auto load = [&](int64_t first, Raw16<T>& k, Raw16<T>& v) {
    const int64_t b = min(first + grp, n_vec - 1);
    k.load(keys + b * kHeadDim + L * 16);
    v.load(values + b * kHeadDim + L * 16);
  };
  if (b0 < n_vec) load(b0, kr, vr);
  for (; b0 < n_vec; b0 += stride) {
    if (b0 + stride < n_vec) load(b0 + stride, krn, vrn);
    const int64_t b = b0 + grp;
    const bool valid = b < n_vec;
    const int64_t t = n_vec <= 0x7fffffff ? (int64_t)((uint32_t)b / (uint32_t)n_kv) : b / n_kv;
    const int h = (int)(b - t * n_kv);
    float f[16];
    kr.to_float(f);
    Code c;
    const int res = encode128_g8_f32(f, c);
    const int64_t row = (int64_t)h * cap + seq0 + t;
    if (valid) {
      kr.store(K + row * kHeadDim + L * 16);
      vr.store(V + row * kHeadDim + L * 16);
    }
    uint4* planes = codes + (int64_t)h * 2 * cap;
    if (valid && res > 0 && L == 0) store_code(planes, cap, seq0 + t, c);
    // exact path (reference order, fp64) for vectors outside the certificate,
    // one at a time by the whole warp in the 4-elements-per-lane layout
    unsigned unsure = __ballot_sync(kFull, valid && res < 0 && L == 0);
    while (unsure) {
      const int g = (__ffs(unsure) - 1) >> 3;
      unsure &= unsure - 1;
      const int64_t bg = b0 + g;
      float e[4];
      Raw4<T>::to_float(Raw4<T>::load(keys + bg * kHeadDim + lane * 4), e);
      Code ce;
      const bool ok = encode128_warp(e, sq[warp], ce, true);
      if (lane == 0) {
        if (!ok) atomicOr(status, kStatusDegenerate);
        store_code(codes + (int64_t)(bg % n_kv) * 2 * cap, cap, seq0 + bg / n_kv, ce);
      }
    }
    kr = krn;
    vr = vrn;
  }
}

// ----------------------------------------------------------------- query encode
template <typename T>
__global__ void __launch_bounds__(kAppendWarps * 32)
encode_query_kernel(const T* __restrict__ q, int n_q, uint16_t* __restrict__ out_ref,
                    int* __restrict__ status) {
  __shared__ double sq[kAppendWarps][kHeadDim];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int h = blockIdx.x * kAppendWarps + warp;
  if (h >= n_q) return;
  float f[4];
  Raw4<T>::to_float(Raw4<T>::load(q + (int64_t)h * kHeadDim + lane * 4), f);
  Code c;
  const bool ok = encode128(f, sq[warp], c);
  if (!ok && lane == 0) atomicOr(status, kStatusDegenerate);
  reinterpret_cast<uint8_t*>(out_ref + (int64_t)h * 16)[lane] = (uint8_t)ref_byte_from_planes(c, lane);
}

// ----------------------------------------------------------------- codes out
__global__ void codes_to_ref_kernel(const uint4* __restrict__ codes, int n_kv, int64_t cap,
                                    int64_t start, int64_t n, uint16_t* __restrict__ out_ref) {
  const int lane = threadIdx.x & 31;
  const int64_t vec = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (vec >= (int64_t)n_kv * n) return;
  const int h = (int)(vec / n);
  const int64_t t = vec % n;
  const Code c = load_code(codes + (int64_t)h * 2 * cap, cap, start + t);
  reinterpret_cast<uint8_t*>(out_ref + vec * 16)[lane] = (uint8_t)ref_byte_from_planes(c, lane);
}

// ----------------------------------------------------------------- score_all
constexpr int kScoreThreads = 256;
constexpr int kScoreTokensPerThread = 4;

// Distance variants over the same bit planes (the
// reference's ablations, kernels.hpp:24-32): with L = al ^ bl and
// Hd = ah ^ bh = X ^ kx ^ L per element,
//   manhattan (2-bit)      |a-b|   = L + 2 (Hd & ~(L & X))
//   euclidean_sq (2-bit)   (a-b)^2 = L + 4 Hd + 4 (Hd & L & ~X) - 4 (Hd & L & X)
//   1-bit L1 (Hamming)     [ah != bh] = Hd: the 1-bit code (x > 0) is the
//                          2-bit code's high bit (both threshold at 0)
constexpr int kMetricManhattan = 0;
constexpr int kMetricEuclideanSq = 1;
constexpr int kMetricHamming1 = 2;

template <int METRIC>
__device__ __forceinline__ uint32_t plane_distance(const QCode& q, const uint32_t klo[4], const uint32_t kx[4]) {
  if (METRIC == kMetricManhattan) return l1_distance(q, klo, kx);
  uint32_t acc = 0;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const uint32_t L = q.lo[w] ^ klo[w];
    const uint32_t Hd = q.x[w] ^ kx[w] ^ L;
    if (METRIC == kMetricHamming1) {
      acc += __popc(Hd);
    } else {
      const uint32_t cr = Hd & L;
      acc += __popc(L) + 4u * __popc(Hd) + 4u * __popc(cr & ~q.x[w]) - 4u * __popc(cr & q.x[w]);
    }
  }
  return acc;
}

template <int METRIC>
__global__ void __launch_bounds__(kScoreThreads)
score_kernel(const uint4* __restrict__ codes, int64_t cap, int64_t S, int group,
             const uint16_t* __restrict__ q_ref, int32_t* __restrict__ scores) {
  __shared__ Code qs;
  const int hq = blockIdx.y;
  const int hk = hq / group;
  if (threadIdx.x < 32) {
    const uint32_t byte = reinterpret_cast<const uint8_t*>(q_ref + (int64_t)hq * 16)[threadIdx.x];
    Code c;
    planes_from_ref_byte(byte, c);
    if (threadIdx.x == 0) qs = c;
  }
  __syncthreads();
  const QCode q = make_qcode(qs);
  const uint4* lo_plane = codes + (int64_t)hk * 2 * cap;
  const uint4* x_plane = lo_plane + cap;
  const int64_t t0 = (int64_t)blockIdx.x * kScoreThreads * kScoreTokensPerThread + threadIdx.x;
#pragma unroll
  for (int i = 0; i < kScoreTokensPerThread; ++i) {
    const int64_t t = t0 + (int64_t)i * kScoreThreads;
    if (t < S) {
      uint32_t lo[4], x[4];
      ld_plane_nc(lo_plane + t, lo);
      ld_plane_nc(x_plane + t, x);
      scores[(int64_t)hq * S + t] = (int32_t)plane_distance<METRIC>(q, lo, x);
    }
  }
}

// ----------------------------------------------------------------- top_k
// One CTA per row: the k smallest int32 scores under the order (score, index)
// (estimator.cpp:75-90: any int32, ties toward the smaller index), as ascending
// indices. Radix select over order keys u = score ^ 0x80000000 (unsigned order =
// signed order), 8-bit digits from the highest digit in which the row's min and
// max keys differ (2-bit distances <= 384 take 2 passes, any int32 at most 4),
// then an order-preserving compaction of {key < T} plus the first
// (k - #below) indices with key == T. The output is ascending by construction;
// no sort.
constexpr int kTopkThreads = 1024;

// Exclusive prefix of a 0/1 flag over the CTA in thread order; returns the
// prefix and writes the CTA total to *total. `scratch` holds 32 ints.
__device__ __forceinline__ int block_flag_scan(bool flag, int* scratch, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t b = __ballot_sync(kFull, flag);
  const int in_warp = __popc(b & ((1u << lane) - 1u));
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
  return before + in_warp;
}

__device__ __forceinline__ uint32_t topk_key(int32_t v) { return (uint32_t)v ^ 0x80000000u; }

__global__ void __launch_bounds__(kTopkThreads)
topk_kernel(const int32_t* __restrict__ scores, int64_t n, int64_t k, int32_t* __restrict__ idx) {
  __shared__ unsigned hist[256];
  __shared__ int scratch[32];
  __shared__ uint32_t s_min[32], s_max[32];
  __shared__ uint32_t s_prefix;
  __shared__ int s_need;
  const int row = blockIdx.x;
  const int32_t* s = scores + (int64_t)row * n;
  int32_t* out = idx + (int64_t)row * k;
  const int64_t keep = k < n ? k : n;
  for (int64_t i = keep + threadIdx.x; i < k; i += blockDim.x) out[i] = -1;
  if (k >= n) {  // estimator.cpp:80 — everything, in order
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = (int32_t)i;
    return;
  }
  if (k == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // the row's key range: leading digits shared by every key need no pass
  uint32_t lo = 0xffffffffu, hi = 0u;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t u = topk_key(s[i]);
    lo = min(lo, u);
    hi = max(hi, u);
  }
  lo = __reduce_min_sync(kFull, lo);
  hi = __reduce_max_sync(kFull, hi);
  if (lane == 0) { s_min[warp] = lo; s_max[warp] = hi; }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    lo = __reduce_min_sync(kFull, lane < nw ? s_min[lane] : 0xffffffffu);
    hi = __reduce_max_sync(kFull, lane < nw ? s_max[lane] : 0u);
    if (lane == 0) {
      s_min[0] = lo;
      s_max[0] = hi;
      s_need = (int)k;
    }
  }
  __syncthreads();
  lo = s_min[0];
  hi = s_max[0];
  const uint32_t diff = lo ^ hi;
  int shift = diff ? ((31 - __clz(diff)) / 8) * 8 : -8;  // top digit in which keys differ
  if (threadIdx.x == 0) s_prefix = shift + 8 >= 32 ? 0u : (lo & (0xffffffffu << (shift + 8)));
  __syncthreads();
  for (; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t prefix = s_prefix;
    const uint32_t hi_mask = shift + 8 >= 32 ? 0u : (0xffffffffu << (shift + 8));
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t u = topk_key(s[i]);
      if ((u & hi_mask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (warp == 0) {  // digit whose cumulative count reaches the remaining need
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
      const int need = s_need;
      __syncwarp();  // every lane has read s_need before one lane rewrites it (racecheck)
      unsigned before = incl - sum;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if ((int)before < need && (int)(before + c[j]) >= need) {
          s_prefix = prefix | ((uint32_t)(lane * 8 + j) << shift);
          s_need = need - (int)before;
        }
        before += c[j];
      }
    }
    __syncthreads();
  }
  const uint32_t T = s_prefix;
  const int need = s_need;  // keys equal to T to take, in index order
  int eq_seen = 0, taken = 0;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const uint32_t u = i < n ? topk_key(s[i]) : 0xffffffffu;
    const bool eq = (i < n) && u == T;
    int eq_total;
    const int eq_before = eq_seen + block_flag_scan(eq, scratch, &eq_total);
    const bool take = (i < n) && (u < T || (eq && eq_before < need));
    int take_total;
    const int pos = taken + block_flag_scan(take, scratch, &take_total);
    if (take) out[pos] = (int32_t)i;
    eq_seen += eq_total;
    taken += take_total;
    if (taken >= keep) break;
  }
}

// ----------------------------------------------------------------- sparse attention
// One CTA per q-head; each warp walks rows warp, warp+8, ... with an online
// softmax over its rows (fp32), then the eight (m, l, o) partials are merged.
constexpr int kAttnWarps = 8;
constexpr float kLog2e = 1.4426950408889634f;

template <typename T>
__global__ void __launch_bounds__(kAttnWarps * 32)
attend_kernel(const T* __restrict__ K, const T* __restrict__ V, int64_t cap, int64_t seq_len, int group,
              const T* __restrict__ q, const int32_t* __restrict__ idx, int64_t k,
              float* __restrict__ out, float* __restrict__ lse, int* __restrict__ status) {
  __shared__ float sm[kAttnWarps], sl[kAttnWarps];
  __shared__ float so[kAttnWarps][kHeadDim];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hq = blockIdx.x, hk = hq / group;
  {  // KvCache::gather preconditions (kv_cache.cpp:90-91) and the empty selection
     // (attention.cpp:42): a row is a strictly increasing run of indices in
     // [0, seq_len), optionally followed by -1 entries only. A bad row latches
     // kStatusBadSelection and reads nothing.
    const int32_t* row = idx + (int64_t)hq * k;
    bool bad = false;
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x) {
      const int32_t t = row[i], prev = i > 0 ? row[i - 1] : -1;
      if (t >= 0) bad |= t >= seq_len || (i > 0 && prev < 0) || (i > 0 && prev >= t);
      else bad |= t != -1 || i == 0;
    }
    if (__syncthreads_or(bad)) {
      if (threadIdx.x == 0) atomicOr(status, kStatusBadSelection);
      if (warp == 0) {
        *reinterpret_cast<float4*>(out + (int64_t)hq * kHeadDim + lane * 4) = make_float4(NAN, NAN, NAN, NAN);
        if (lse != nullptr && lane == 0) { lse[2 * hq] = NAN; lse[2 * hq + 1] = 0.f; }
      }
      return;
    }
  }
  float qf[4];
  Raw4<T>::to_float(Raw4<T>::load(q + (int64_t)hq * kHeadDim + lane * 4), qf);
  // logits in log2 units: q.k / sqrt(128) * log2(e)
  const float scale = 0.088388347648318440f * kLog2e;
  const int32_t* row_idx = idx + (int64_t)hq * k;
  const T* Kh = K + (int64_t)hk * cap * kHeadDim;
  const T* Vh = V + (int64_t)hk * cap * kHeadDim;
  float m = -INFINITY, l = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t r = warp; r < k; r += kAttnWarps) {
    const int32_t t = row_idx[r];
    if (t < 0) break;
    float kf[4], vf[4];
    Raw4<T>::to_float(Raw4<T>::load(Kh + (int64_t)t * kHeadDim + lane * 4), kf);
    Raw4<T>::to_float(Raw4<T>::load(Vh + (int64_t)t * kHeadDim + lane * 4), vf);
    float dot = qf[0] * kf[0] + qf[1] * kf[1] + qf[2] * kf[2] + qf[3] * kf[3];
    dot = warp_sum(dot) * scale;
    const float mn = fmaxf(m, dot);
    const float corr = exp2f(m - mn);
    const float p = exp2f(dot - mn);
    l = l * corr + p;
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = o[j] * corr + p * vf[j];
    m = mn;
  }
  if (lane == 0) { sm[warp] = m; sl[warp] = l; }
#pragma unroll
  for (int j = 0; j < 4; ++j) so[warp][lane * 4 + j] = o[j];
  __syncthreads();
  if (warp == 0) {
    float M = -INFINITY;
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, sm[w]);
    float L = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int w = 0; w < kAttnWarps; ++w) {
      if (sl[w] == 0.f) continue;
      const float c = exp2f(sm[w] - M);
      L += sl[w] * c;
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] += so[w][lane * 4 + j] * c;
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    float4 res = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
    *reinterpret_cast<float4*>(out + (int64_t)hq * kHeadDim + lane * 4) = res;
    if (lse != nullptr && lane == 0) {
      lse[2 * hq] = M / kLog2e;  // natural-log units
      lse[2 * hq + 1] = L;
    }
  }
}

}  // namespace adamas_dev

namespace adamas_dev {

// ----------------------------------------------------------------- sequence-sharded decode
// Distributed top-k. Every rank holds a contiguous token range
// of the sequence and contributes its local top-k keys (dist << 23 | global
// index, the (score, index) order of top_k, estimator.cpp:75-90). A member of
// the global top-k has fewer than k predecessors in its own shard, so it is
// among that shard's keys: the selection rebuilt from the gathered keys is
// exactly the single-device one. One CTA per q-head rebuilds it, attends over
// this rank's survivors (rows of the local cache) and emits the partial
// (m, l, o[128]) for the log-sum-exp merge (attention.cpp:8-38 semantics).
#ifndef ADAMAS_SEL_STOP
#define ADAMAS_SEL_STOP 0  // diagnostics builds only: stop seq_select_attend after phase N (timing only)
#endif
constexpr int kSelThreads = 512;
constexpr int kSelMaxKeys = 8192;   // n_ranks * budget per q-head
constexpr int kSelMaxSurv = 2048;   // budget
constexpr int kSelBins = 512;
constexpr int kPartialStride = 132;  // m (natural-log units), l, pad, pad, o[128]

// One warp: out[0..128) = sum_r e^{m_r - M} o_r / sum_r e^{m_r - M} l_r over
// the n_ranks partials (m in natural-log units, l, pad, pad, o[128]) at
// base + r * stride. Every load is independent of the others: lane r reads
// rank r's (m, l) header, then every lane issues its o-quads of up to 8 ranks
// at once — two round trips to the mailbox instead of one per rank and field.
__device__ __forceinline__ void merge_partials_warp(const float* base, int64_t stride, int n_ranks, float* out_row) {
  const int lane = threadIdx.x & 31;
  float M = -INFINITY;
  for (int r0 = 0; r0 < n_ranks; r0 += 32) {
    const int r = r0 + lane;
    const float2 ml = r < n_ranks ? ld_mailbox2(base + r * stride) : make_float2(-INFINITY, 0.f);
    M = fmaxf(M, ml.y > 0.f ? ml.x : -INFINITY);
  }
#pragma unroll
  for (int m2 = 16; m2 > 0; m2 >>= 1) M = fmaxf(M, __shfl_xor_sync(kFull, M, m2));
  float L = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int r0 = 0; r0 < n_ranks; r0 += 32) {
    const int r = r0 + lane;
    const float2 ml = r < n_ranks ? ld_mailbox2(base + r * stride) : make_float2(-INFINITY, 0.f);
    const float c = ml.y > 0.f ? __expf(ml.x - M) : 0.f;  // this lane's rank weight
    L += warp_sum(ml.y * c);
    const int nr = min(32, n_ranks - r0);
    for (int q0 = 0; q0 < nr; q0 += 8) {
      float4 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        v[i] = q0 + i < nr ? ld_mailbox4(base + (r0 + q0 + i) * stride + 4 + lane * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float ci = __shfl_sync(kFull, c, (q0 + i) & 31);
        if (q0 + i < nr) {
          acc[0] += v[i].x * ci; acc[1] += v[i].y * ci; acc[2] += v[i].z * ci; acc[3] += v[i].w * ci;
        }
      }
    }
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  *reinterpret_cast<float4*>(out_row + lane * 4) = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
}



__device__ __forceinline__ void sel_block_excl_scan(int v, int& excl, int& total, int* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    const int o = __shfl_up_sync(kFull, incl, m);
    if (lane >= m) incl += o;
  }
  if (lane == 31) scratch[warp] = incl;
  __syncthreads();
  // the 16 warp totals: a 4-step shuffle scan (not a serial walk) in every warp
  constexpr int NW = kSelThreads / 32;
  int wt = lane < NW ? scratch[lane] : 0;
#pragma unroll
  for (int m = 1; m < NW; m <<= 1) {
    const int o = __shfl_up_sync(kFull, wt, m);
    if (lane >= m) wt += o;
  }
  const int before = __shfl_sync(kFull, wt, (warp + 31) & 31);  // inclusive total of warps < warp
  excl = (warp > 0 ? before : 0) + incl - v;
  total = __shfl_sync(kFull, wt, NW - 1);
  __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(kSelThreads)
seq_select_attend_kernel(const T* __restrict__ K, const T* __restrict__ V, int64_t cap, int group,
                         const T* __restrict__ q, const uint32_t* keys, int n_ranks, int n_q,
                         int64_t budget, int k_eff, int64_t rank_base, int64_t rank_len, float* __restrict__ partial,
                         int32_t* __restrict__ gidx, const __grid_constant__ PeerPush push,
                         const uint32_t* wait_flags, int* __restrict__ status,
                         const float* merge_parts, const uint32_t* merge_flags,
                         float* __restrict__ merge_out) {
  extern __shared__ uint32_t skeys[];  // the n_ranks * budget keys of this q-head, read once
  __shared__ int hist[kSelBins];
  __shared__ int scratch[32];
  __shared__ int s_T, s_below, s_bad;
  __shared__ int s_lo_cnt, s_in_cnt;  // packed (lt | eq << 16) counts below / inside the local range
  __shared__ int rows[kSelMaxSurv];  // this rank's survivors (local rows), ascending
  __shared__ float wm[kSelThreads / 32], wl[kSelThreads / 32];
  __shared__ __align__(16) float wo[kSelThreads / 32][kHeadDim];
  __shared__ __align__(16) float pre_s[8][kPartialStride];  // local fused merge: every rank's partial
  const int h = blockIdx.x, hk = h / group;
  // Fused merge whose other partials are already in place (no peer epochs to
  // wait for): they are read at the start, behind the selection, and merged
  // from shared memory with this rank's partial at the end.
  const bool merge_local = merge_out != nullptr && merge_flags == nullptr && partial != nullptr && n_ranks <= 8;
  const int my_slot = merge_local ? (int)((partial - merge_parts) / ((int64_t)n_q * kPartialStride)) : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = n_ranks * (int)budget;
  constexpr uint32_t kEmpty = 0xffffffffu;
  // programmatic dependent launch: keys / the appended row come from the
  // preceding kernel; the next launch may begin its own prologue now
  grid_dependency_wait();
  // With the peer-epoch merge (merge_flags) every CTA waits for the other
  // ranks' partials, so all must be resident: the next launch is not let in
  // early (it could take the SMs of CTAs not yet placed).
  if (tid == 0 && (merge_out == nullptr || merge_flags == nullptr)) grid_launch_dependents();
  if (ADAMAS_SEL_STOP == 9) return;  // diagnostics (timing only)
  for (int b = tid; b < kSelBins; b += kSelThreads) hist[b] = 0;
  if (tid == 0) {
    s_T = -1; s_below = 0; s_bad = 0;
    if (push.n) peer_wait(wait_flags, n_ranks, push.epoch, status);  // every rank's keys of this step have landed
  }
  // the q-head's query, consumed by the attention at the end: its load
  // latency hides behind the selection
  const typename Raw4<T>::V q_raw = Raw4<T>::load(q + (int64_t)h * kHeadDim + lane * 4);
  const T* Kh = K + (int64_t)hk * cap * kHeadDim;
  const T* Vh = V + (int64_t)hk * cap * kHeadDim;
  __syncthreads();
  constexpr int kQuads = kPartialStride / 4;
  const int pr_r = tid / kQuads, pr_c = tid - pr_r * kQuads;
  const bool pre_mine = merge_local && pr_r < n_ranks && pr_r != my_slot;
  float4 pre_v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (pre_mine) pre_v = ld_mailbox4(merge_parts + ((int64_t)pr_r * n_q + h) * kPartialStride + pr_c * 4);
  {
    int r = tid / (int)budget, i = tid - r * (int)budget;  // j = r * budget + i, advanced without a division
    for (int j = tid; j < n; j += kSelThreads) {
      const uint32_t key = ld_mailbox(keys + ((int64_t)r * n_q + h) * budget + i);
      skeys[j] = key;
      if (key != kEmpty) {
        atomicAdd(&hist[key >> 23], 1);
        // a local candidate: its K / V rows may be gathered below; warm L2
        // now so the attention after the selection does not wait on HBM
        const int64_t t = (int64_t)(key & 0x7fffffu) - rank_base;
        if (t >= 0 && t < rank_len) {
#pragma unroll
          for (int c = 0; c < (int)(kHeadDim * sizeof(T)); c += 128) {
            prefetch_l2(reinterpret_cast<const char*>(Kh + t * kHeadDim) + c);
            prefetch_l2(reinterpret_cast<const char*>(Vh + t * kHeadDim) + c);
          }
        }
      }
      for (i += kSelThreads; i >= (int)budget; i -= (int)budget) ++r;
    }
  }
  if (pre_mine) *reinterpret_cast<float4*>(&pre_s[pr_r][pr_c * 4]) = pre_v;
  __syncthreads();
  if (ADAMAS_SEL_STOP == 1) return;  // diagnostics (timing only)
  // Input contract (adamas_seq_local_candidates): each rank's keys ascending
  // in the index field, empty keys last; ranks in sequence order. The array
  // is then ascending in index, so an order-preserving compaction emits the
  // selection in top_k's output order without a sort.
  {
    int i = tid % (int)budget;  // position within the rank's keys
    for (int j = tid; j + 1 < n; j += kSelThreads) {
      if (i + 1 != (int)budget) {  // (the next key belongs to the next rank otherwise)
        const uint32_t a = skeys[j], b = skeys[j + 1];
        if ((a == kEmpty && b != kEmpty) || (a != kEmpty && b != kEmpty && (a & 0x7fffffu) >= (b & 0x7fffffu)))
          s_bad = 1;
      }
      for (i += kSelThreads; i >= (int)budget;) i -= (int)budget;
    }
  }
  {  // T = smallest distance whose cumulative count reaches k_eff (one bin per thread)
    const int v = hist[tid];
    int excl, total;
    sel_block_excl_scan(v, excl, total, scratch);
    if (excl < k_eff && excl + v >= k_eff) { s_T = tid; s_below = excl; }
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) atomicOr(status, kStatusBadSelection);
    return;  // (the peer-exchange launch's waiters time out on the missing partial and latch it too)
  }
  if (ADAMAS_SEL_STOP == 2) return;  // diagnostics (timing only)
  // Keys are unique (dist << 23 | global index) and the array ascends in the
  // index field, so the selection -- the k_eff smallest keys in top_k's
  // (score, index) order -- is every key at distance < T plus the first
  // rem = k_eff - below keys at distance T in array order: ONE
  // order-preserving compaction (a packed (lt, eq) block scan), no radix
  // select over the index bits. The selection lands in `rows` in ascending
  // index order; this rank's survivors are the contiguous part of it inside
  // [rank_base, rank_base + rank_len), located from two block counts.
  const int Tthr = s_T;
  const int rem = k_eff - s_below;
  if (tid == 0) { s_lo_cnt = 0; s_in_cnt = 0; }
  __syncthreads();
  const int per = (n + kSelThreads - 1) / kSelThreads;
  const int j0 = min(n, tid * per), j1 = min(n, j0 + per);
  int my_lt = 0, my_eq = 0, lt_lo = 0, eq_lo = 0, lt_in = 0, eq_in = 0;
  for (int j = j0; j < j1; ++j) {
    const uint32_t key = skeys[j];
    if (key == kEmpty) continue;
    const int d = (int)(key >> 23);
    const int64_t idx = key & 0x7fffffu;
    const bool lt = d < Tthr, eq = d == Tthr;
    my_lt += lt;
    my_eq += eq;
    if (idx < rank_base) { lt_lo += lt; eq_lo += eq; }
    else if (idx < rank_base + rank_len) { lt_in += lt; eq_in += eq; }
  }
  // block totals of the range counts (no prefix needed): keys below the
  // local range that are selected = lt_lo + min(rem, eq_lo), likewise inside
  lt_lo = __reduce_add_sync(kFull, lt_lo | (eq_lo << 16));
  lt_in = __reduce_add_sync(kFull, lt_in | (eq_in << 16));
  if (lane == 0) {
    if (lt_lo) atomicAdd(&s_lo_cnt, lt_lo);
    if (lt_in) atomicAdd(&s_in_cnt, lt_in);
  }
  int packed_before, packed_total;  // counts < 2^13 (n <= kSelMaxKeys): lt | eq << 16 in one scan
  sel_block_excl_scan(my_lt | (my_eq << 16), packed_before, packed_total, scratch);
  int lt_before = packed_before & 0xffff, eq_seen = packed_before >> 16;
  int pos = lt_before + min(eq_seen, rem);
  for (int j = j0; j < j1; ++j) {
    const uint32_t key = skeys[j];
    if (key == kEmpty) continue;
    const int d = (int)(key >> 23);
    if (d > Tthr || (d == Tthr && eq_seen++ >= rem)) continue;
    const int idx = (int)(key & 0x7fffffu);
    if (gidx != nullptr) gidx[(int64_t)h * budget + pos] = idx;  // the global selection, ascending
    rows[pos++] = idx;
  }
  if (gidx != nullptr)
    for (int i = k_eff + tid; i < budget; i += kSelThreads) gidx[(int64_t)h * budget + i] = -1;
  __syncthreads();
  const int lo_cnt = s_lo_cnt, in_cnt = s_in_cnt;
  const int sel_lo = (lo_cnt & 0xffff) + min(rem, lo_cnt >> 16);  // selected below the local range
  const int nl = (in_cnt & 0xffff) + min(max(0, rem - (lo_cnt >> 16)), in_cnt >> 16);  // ... inside it
  const int* lrows = rows + sel_lo;
  if (ADAMAS_SEL_STOP == 3) return;  // diagnostics (timing only)
  // attention over this rank's survivors: per-warp online softmax, log2 units
  float qf[4];
  Raw4<T>::to_float(q_raw, qf);
  const float scale = 0.088388347648318440f * kLog2e;
#pragma unroll
  for (int j = 0; j < 4; ++j) qf[j] *= scale;
  Kh += lane * 4;
  Vh += lane * 4;
  float m = -INFINITY, l = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
  constexpr int NW = kSelThreads / 32, B = 4;  // rows in flight per warp (all survivors may be local)
  for (int r0 = warp; r0 < nl; r0 += NW * B) {
    typename Raw4<T>::V kb[B], vb[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int r = r0 + b * NW;
      if (r < nl && ADAMAS_SEL_STOP != 5) {
        const int64_t t = lrows[r] - rank_base;
        kb[b] = Raw4<T>::load(Kh + t * kHeadDim);
        vb[b] = Raw4<T>::load(Vh + t * kHeadDim);
      } else {
        kb[b] = typename Raw4<T>::V{};
        vb[b] = typename Raw4<T>::V{};
      }
    }
    float sd[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      float kf[4];
      Raw4<T>::to_float(kb[b], kf);
      sd[b] = r0 + b * NW < nl ? qf[0] * kf[0] + qf[1] * kf[1] + qf[2] * kf[2] + qf[3] * kf[3] : 0.f;
    }
#pragma unroll
    for (int m2 = 16; m2 > 0; m2 >>= 1)
#pragma unroll
      for (int b = 0; b < B; ++b) sd[b] += __shfl_xor_sync(kFull, sd[b], m2);
    float mx = m;
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (r0 + b * NW < nl) mx = fmaxf(mx, sd[b]);
    const float corr = exp2f(m - mx);
    l *= corr;
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] *= corr;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (r0 + b * NW < nl) {
        float vf[4];
        Raw4<T>::to_float(vb[b], vf);
        const float pr = exp2f(sd[b] - mx);
        l += pr;
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] += pr * vf[j];
      }
    }
    m = mx;
  }
  if (ADAMAS_SEL_STOP == 6) {  // diagnostics (timing only): attention done, no combine
    if (lane == 0 && m == 12345.f) partial[0] = l;
    return;
  }
  if (lane == 0) { wm[warp] = m; wl[warp] = l; }
#pragma unroll
  for (int j = 0; j < 4; ++j) wo[warp][lane * 4 + j] = o[j];
  __syncthreads();
  if (warp == 0) {  // combine the NW warp partials: lane-parallel weights, all quads in flight
    const float mw = lane < NW ? wm[lane] : -INFINITY, lw = lane < NW ? wl[lane] : 0.f;
    float M = lw > 0.f ? mw : -INFINITY;
#pragma unroll
    for (int m2 = 16; m2 > 0; m2 >>= 1) M = fmaxf(M, __shfl_xor_sync(kFull, M, m2));
    const float cw = lw > 0.f ? exp2f(mw - M) : 0.f;
    const float L = warp_sum(lw * cw);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float c = __shfl_sync(kFull, cw, w);
      const float4 v4 = *reinterpret_cast<const float4*>(&wo[w][lane * 4]);
      acc[0] += v4.x * c; acc[1] += v4.y * c; acc[2] += v4.z * c; acc[3] += v4.w * c;
    }
    const float4 hdr = make_float4(L > 0.f ? M / kLog2e : -INFINITY, L, 0.f, 0.f);  // natural-log units
    const float4 body = make_float4(acc[0], acc[1], acc[2], acc[3]);
    const int nd = push.n ? push.n : 1;
    for (int r = 0; r < nd; ++r) {  // peer exchange: this rank's partial into every mailbox
      float* pp = (push.n ? push.part[r] : partial) + (int64_t)h * kPartialStride;
      if (lane == 0) *reinterpret_cast<float4*>(pp) = hdr;
      *reinterpret_cast<float4*>(pp + 4 + lane * 4) = body;
    }
    if (merge_local) {  // this rank's partial joins the preloaded ones; merge from shared memory
      if (lane == 0) *reinterpret_cast<float4*>(&pre_s[my_slot][0]) = hdr;
      *reinterpret_cast<float4*>(&pre_s[my_slot][4 + lane * 4]) = body;
      __syncwarp();
      const float2 ml = lane < n_ranks ? make_float2(pre_s[lane][0], pre_s[lane][1]) : make_float2(-INFINITY, 0.f);
      float Mx = ml.y > 0.f ? ml.x : -INFINITY;
#pragma unroll
      for (int m2 = 16; m2 > 0; m2 >>= 1) Mx = fmaxf(Mx, __shfl_xor_sync(kFull, Mx, m2));
      const float cr = ml.y > 0.f ? __expf(ml.x - Mx) : 0.f;
      const float Ls = warp_sum(ml.y * cr);
      float a2[4] = {0.f, 0.f, 0.f, 0.f};
      for (int r = 0; r < n_ranks; ++r) {
        const float c = __shfl_sync(kFull, cr, r);
        const float4 v = *reinterpret_cast<const float4*>(&pre_s[r][4 + lane * 4]);
        a2[0] += v.x * c; a2[1] += v.y * c; a2[2] += v.z * c; a2[3] += v.w * c;
      }
      const float inv = Ls > 0.f ? 1.f / Ls : 0.f;
      *reinterpret_cast<float4*>(merge_out + (int64_t)h * kHeadDim + lane * 4) =
          make_float4(a2[0] * inv, a2[1] * inv, a2[2] * inv, a2[3] * inv);
    }
  }
  if (push.n) {
    __syncthreads();
    if (tid == 0) peer_signal(push);
  }
  if (ADAMAS_SEL_STOP == 4) return;  // diagnostics (timing only)
  if (merge_out && !merge_local) {  // fused log-sum-exp merge of this q-head (with merge_flags: every CTA
                                   // of the launch is resident; without: the other ranks' partials are in place)
    if (tid == 0 && merge_flags) peer_wait(merge_flags, n_ranks, push.epoch, status);
    __syncthreads();
    if (warp == 0)
      merge_partials_warp(merge_parts + (int64_t)h * kPartialStride, (int64_t)n_q * kPartialStride, n_ranks,
                          merge_out + (int64_t)h * kHeadDim);
  }
}

// out[h] = sum_r e^{m_r - M} o_r / sum_r e^{m_r - M} l_r over the ranks' partials.
// With wait_flags, first acquires every rank's partial epoch (peer exchange).
__global__ void lse_merge_kernel(const float* partials, int n_ranks, int n_q, float* __restrict__ out,
                                 const uint32_t* wait_flags, const uint32_t* epoch, int* __restrict__ status) {
  const int h = blockIdx.x, lane = threadIdx.x;
  grid_dependency_wait();  // partials come from the preceding kernel (PDL launch)
  if (lane == 0) grid_launch_dependents();
  if (wait_flags) {
    if (lane == 0) peer_wait(wait_flags, n_ranks, epoch, status);
    __syncwarp();
  }
  merge_partials_warp(partials + (int64_t)h * kPartialStride, (int64_t)n_q * kPartialStride, n_ranks,
                      out + (int64_t)h * kHeadDim);
}

// An empty shard's candidates: all-empty keys into every mailbox, then the
// arrival / epoch publication of a one-CTA launch.
__global__ void peer_empty_keys_kernel(const __grid_constant__ PeerPush push, int64_t n_keys) {
  for (int r = 0; r < push.n; ++r)
    for (int64_t i = threadIdx.x; i < n_keys; i += blockDim.x) push.keys[r][i] = 0xffffffffu;
  __syncthreads();
  if (threadIdx.x == 0) peer_signal(push);
}

}  // namespace adamas_dev
