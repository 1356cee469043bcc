// common.cuh — device building blocks shared by every Adamas kernel (sm_100a).
//
// Code layout in HBM ("bit-plane", 32 B per token per kv-head at d = 128):
//   two plane arrays per kv-head, each [capacity] x 16 B:
//     lo plane of token t of kv-head h at planes[(2h + 0) * capacity + t]
//     x  plane                         at planes[(2h + 1) * capacity + t]
//   Element e (0..127) of the transformed key sits at bit (e / 4) of word
//   e % 4: the lo plane holds the code's low bit, the x plane holds
//   low XOR high bit. Separate planes make every per-lane 16-byte access
//   (global or the bulk-copied shared-memory stage) contiguous across a warp.
// This is the reference PackedCodes (quantizer.hpp:44-50: element i at bits
// [2(i%8), 2(i%8)+2) of u16 word i/8) with the bits transposed into planes, so
// the Manhattan distance becomes 2 LOP3 + ~1.25 POPC per 32 elements instead
// of the reference's nibble SWAR (kernels_scalar.cpp:41-70). Layout is an
// implementation freedom; the integer results are identical.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace adamas_dev {

constexpr int kHeadDim = 128;
constexpr uint32_t kFull = 0xffffffffu;
// k_inv_sqrt2 (reference kernels_impl.hpp:10) and kQ28 (quantizer.cpp:13).
constexpr double kInvSqrt2 = 0.70710678118654752440;
constexpr double kQ28 = 0.6744897501960817432;

// Sticky status bits (C-ABI ADAMAS_STATUS_*).
constexpr int kStatusDegenerate = 1;  // zero or non-finite vector (quantizer.cpp:46-47)
constexpr int kStatusSyncTimeout = 4;  // a multi-cluster unit barrier gave up (results invalid)
constexpr int kStatusPeerTimeout = 8;  // a peer-memory exchange wait gave up (results invalid)
constexpr int kStatusBadSelection = 16;  // gather indices not strictly increasing / out of range, or empty (kv_cache.cpp:90-91, attention.cpp:42)

// ---------------------------------------------------------------- peer-memory exchange
// Sequence-sharded decode exchanges its two small messages (the
// local candidate keys, the attention partials) by storing straight into every
// rank's mailbox over NVLink (CUDA IPC mappings) instead of NCCL all-gathers.
// Each launch's CTAs count themselves in on a local arrival counter; the last
// one publishes this rank's epoch to every mailbox with a system-scope release;
// the consumer kernel acquires every rank's epoch before reading.
constexpr int kMaxPeers = 8;

struct PeerPush {
  int n;                         // ranks (0: exchange off)
  uint32_t* keys[kMaxPeers];     // keys mode: this rank's slot in every rank's mailbox
  float* part[kMaxPeers];        // partials mode: this rank's slot in every rank's mailbox
  uint32_t* flag[kMaxPeers];     // this rank's flag in every rank's mailbox
  unsigned int* arrive;          // own mailbox: CTA arrival counter of this launch
  uint32_t* epoch;               // own mailbox: this rank's step counter (device-side: graph replays advance it)
  int bump;                      // 1: this launch starts a new step (keys phase)
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Loads of mailbox memory that other GPUs (or other kernels still running)
// write: coherent system-scope relaxed loads, never the read-only (.nc /
// LDG.CONSTANT) path. Ordered after peer_wait's acquire by the CTA barrier
// that follows it.
__device__ __forceinline__ uint32_t ld_mailbox(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float ld_mailbox(const float* p) {
  float v;
  asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float2 ld_mailbox2(const float* p) {
  float2 v;
  asm volatile("ld.relaxed.sys.global.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float4 ld_mailbox4(const float* p) {
  float4 v;
  asm volatile("ld.relaxed.sys.global.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
  return v;
}

// One thread per CTA, after a barrier covering all of the CTA's peer stores.
__device__ __forceinline__ void peer_signal(const PeerPush& pp) {
  __threadfence_system();
  const unsigned old = atomicAdd(pp.arrive, 1u);
  if (old == gridDim.x * gridDim.y * gridDim.z - 1) {
    atomicExch(pp.arrive, 0u);  // every CTA of this launch has arrived: reset for the next one
    const uint32_t e = *(volatile uint32_t*)pp.epoch + (pp.bump ? 1u : 0u);
    if (pp.bump) *(volatile uint32_t*)pp.epoch = e;
    __threadfence_system();
    for (int r = 0; r < pp.n; ++r) st_release_sys(pp.flag[r], e);
  }
}

// One thread: wait until flags[0..n) all reached this rank's current step
// (*epoch_ctr, bumped by the step's keys launch; wrap-safe compare); gives up
// after ~4 s and latches kStatusPeerTimeout.
__device__ __forceinline__ void peer_wait(const uint32_t* flags, int n, const uint32_t* epoch_ctr, int* status) {
  const uint32_t epoch = *(const volatile uint32_t*)epoch_ctr;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int r = 0; r < n; ++r) {
    while ((int32_t)(ld_acquire_sys(flags + r) - epoch) < 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 4000000000ull) {
        atomicOr(status, kStatusPeerTimeout);
        return;
      }
      __nanosleep(64);
    }
  }
}

struct __align__(32) Code {
  uint32_t lo[4];
  uint32_t hi[4];
};

// Query-side precomputation for the distance: X = lo ^ hi.
struct QCode {
  uint32_t lo[4], x[4], hi[4];
};

__device__ __forceinline__ QCode make_qcode(const Code& c) {
  QCode q;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    q.lo[w] = c.lo[w];
    q.x[w] = c.lo[w] ^ c.hi[w];
    q.hi[w] = c.hi[w];
  }
  return q;
}

// One LOP3 with an explicit truth table (the compiler's own fusion of the
// A term below took 5 instructions per word instead of 3).
template <uint32_t LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return d;
}

// Carry-save adder: a + b + c = s + 2 cy, bitwise.
__device__ __forceinline__ void csa3(uint32_t a, uint32_t b, uint32_t c, uint32_t& s, uint32_t& cy) {
  s = a ^ b ^ c;
  cy = (a & b) | (c & (a ^ b));
}

// Sum over the 128 elements of |q_e - k_e| for 2-bit codes, key given as its
// stored (lo, x = lo ^ hi) planes. Per element with a = 2ah + al, b = 2bh + bl:
// |a - b| = L + 2A where L = al ^ bl and A = (ah ^ bh) & ~(L & (al ^ ah)), and
// ah ^ bh = X ^ kx ^ L with X = al ^ ah, kx = bl ^ bh, so A is ONE 3-input
// LOP3 of (X, kx, L). Checked exhaustively over all 16 (a, b) pairs in
// tests/test_abi.py. The 4 weight-1 words L and 4 weight-2 words A are folded
// by carry-save adders into fewer popcounts (trading ALU LOP3s against the
// quarter-rate POPC pipe; see below and tools/scan_bench.cu).
// Three carry-save foldings of the same sum, picked per kernel instance by
// measurement (tools/ab.sh, profiles/r02h_ab_distance_fold.txt): FOLD 6 —
// 6 POPC, 12 LOP3 (the default: best at one q-head per scan, config 1 9.93 ->
// 9.89 us, config 2 16.80 -> 16.41); FOLD 7 — 7 POPC, 10 LOP3 (best for
// ALU-bound multi-head scans, config 3 4.20 -> 4.07); FOLD 5 — 5 POPC, 16
// LOP3 (the round-1 balance). All return the identical integer.
template <int FOLD = 6>
__device__ __forceinline__ uint32_t l1_distance(const QCode& q, const uint32_t klo[4], const uint32_t kx[4]) {
  uint32_t L[4], A[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    L[w] = q.lo[w] ^ klo[w];
    if constexpr (FOLD == 7) {
      // ah ^ bh = qh ^ kl ^ kx: one 3-input XOR independent of L; then
      // A = H & ~(L & X) is one more LOP3 (truth table 0xF0 & ~(0xCC & 0xAA)).
      // Measured: multi-head scans 4.07 -> 3.97 us (config 3); at one q-head
      // per scan the compiler's own form is faster (kept for FOLD 6).
      const uint32_t H = lop3<0x96>(q.hi[w], klo[w], kx[w]);
      A[w] = lop3<0x70>(H, L[w], q.x[w]);
    } else {
      A[w] = (q.x[w] ^ kx[w] ^ L[w]) & ~(L[w] & q.x[w]);
    }
  }
  if constexpr (FOLD == 7) {
    uint32_t s1, c1;
    csa3(L[0], L[1], L[2], s1, c1);  // weight 1: s1, weight 2: c1
    return __popc(s1) + __popc(L[3]) + 2u * (__popc(c1) + __popc(A[0]) + __popc(A[1]) + __popc(A[2]) + __popc(A[3]));
  } else if constexpr (FOLD == 6) {
    uint32_t s1, c1, s2, c2;
    csa3(L[0], L[1], L[2], s1, c1);  // weight 1: s1, weight 2: c1
    csa3(A[0], A[1], A[2], s2, c2);  // weight 2: s2, weight 4: c2
    return __popc(s1) + __popc(L[3]) + 2u * (__popc(c1) + __popc(s2) + __popc(A[3])) + 4u * __popc(c2);
  } else {
    uint32_t s1, c1, s2, c2, s3, c3;
    csa3(L[0], L[1], L[2], s1, c1);                    // weight 1: s1, weight 2: c1
    const uint32_t s1b = s1 ^ L[3], c1b = s1 & L[3];   // weight 1: s1b, weight 2: c1b
    csa3(A[0], A[1], A[2], s2, c2);                    // weight 2: s2, weight 4: c2
    csa3(A[3], c1, c1b, s3, c3);                       // weight 2: s3, weight 4: c3
    return __popc(s1b) + 2u * (__popc(s2) + __popc(s3)) + 4u * (__popc(c2) + __popc(c3));
  }
}

// Streaming 128-bit load (no L1 allocation).
__device__ __forceinline__ void ld_plane_nc(const uint4* p, uint32_t w[4]) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
               : "l"(p));
}

// ---------------------------------------------------------------------------
// Element loads: lane l owns elements 4l .. 4l+3 of a 128-vector.
template <typename T>
struct Elem;
template <>
struct Elem<float> {
  __device__ static __forceinline__ void load4(const float* p, float v[4]) {
    const float4 x = *reinterpret_cast<const float4*>(p);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  }
  __device__ static __forceinline__ void store4(float* p, const float v[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <>
struct Elem<__nv_bfloat16> {
  __device__ static __forceinline__ void load4(const __nv_bfloat16* p, float v[4]) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    v[0] = __uint_as_float(u.x << 16);
    v[1] = __uint_as_float(u.x & 0xffff0000u);
    v[2] = __uint_as_float(u.y << 16);
    v[3] = __uint_as_float(u.y & 0xffff0000u);
  }
  __device__ static __forceinline__ void load4_raw(const __nv_bfloat16* p, uint2& u) {
    u = *reinterpret_cast<const uint2*>(p);
  }
};

// ---------------------------------------------------------------------------
// Encoder: normalized FWHT (kernels_scalar.cpp:11-22), RMS thresholds
// (quantizer.cpp:40-64), strict-'>' bucketize (quantizer.cpp:74-85) and the
// bit-plane pack, for one 128-vector held 4 elements per lane across a warp.
// All arithmetic is fp64 with explicit _rn intrinsics (no FMA contraction),
// the butterflies in the reference's stage order and the sum of squares in
// index order, so the codes are bit-identical to the reference's.
// `sq` is a 128-double per-warp scratch in shared memory. fast = true takes a
// provably equivalent low-latency route for sigma (see below) with the exact
// sequential sum as its fallback.
// Returns false (and zero codes) for a zero / non-finite vector.
__device__ __forceinline__ bool encode128_warp(const float in[4], double* sq, Code& out, bool fast = false) {
  const int lane = threadIdx.x & 31;
  double x[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) x[j] = (double)in[j];
  // stage h = 1: (0,1), (2,3) within the lane
  {
    const double a0 = x[0], b0 = x[1], a1 = x[2], b1 = x[3];
    x[0] = __dmul_rn(__dadd_rn(a0, b0), kInvSqrt2);
    x[1] = __dmul_rn(__dsub_rn(a0, b0), kInvSqrt2);
    x[2] = __dmul_rn(__dadd_rn(a1, b1), kInvSqrt2);
    x[3] = __dmul_rn(__dsub_rn(a1, b1), kInvSqrt2);
  }
  // stage h = 2: (0,2), (1,3) within the lane
  {
    const double a0 = x[0], b0 = x[2], a1 = x[1], b1 = x[3];
    x[0] = __dmul_rn(__dadd_rn(a0, b0), kInvSqrt2);
    x[2] = __dmul_rn(__dsub_rn(a0, b0), kInvSqrt2);
    x[1] = __dmul_rn(__dadd_rn(a1, b1), kInvSqrt2);
    x[3] = __dmul_rn(__dsub_rn(a1, b1), kInvSqrt2);
  }
  // stages h = 4 .. 64: partner lane at distance h / 4
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    const bool upper = (lane & m) != 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double p = __shfl_xor_sync(kFull, x[j], m);
      // lower element j: (a + b) c with a = mine; upper: (a - b) c with a = partner
      x[j] = upper ? __dmul_rn(__dsub_rn(p, x[j]), kInvSqrt2)
                   : __dmul_rn(__dadd_rn(x[j], p), kInvSqrt2);
    }
  }
  double sq4[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) sq4[j] = __dmul_rn(x[j], x[j]);
  double sigma;
  bool exact = !fast;
  if (fast) {
    // Latency path: a shuffle-tree sum of the same 128 exact products. Any
    // two summation orders of n = 128 non-negative terms agree to within
    // 2 (n-1) u ~= 2.9e-14 relative, so sigma and the +/-kQ28 sigma thresholds
    // to within ~2e-14 relative. Codes can only differ for an element within
    // that distance of a threshold (the 0 threshold does not depend on sigma);
    // if any element is within 1e-12 of one, or the sum is near the fp64
    // range ends where relative bounds fail, take the exact sequential path.
    double s4 = __dadd_rn(__dadd_rn(sq4[0], sq4[1]), __dadd_rn(sq4[2], sq4[3]));
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) s4 = __dadd_rn(s4, __shfl_xor_sync(kFull, s4, m));
    sigma = __dsqrt_rn(__ddiv_rn(s4, (double)kHeadDim));
    const double t = __dmul_rn(kQ28, sigma);
    bool near = !(s4 > 1e-290 && s4 < 1e300);
#pragma unroll
    for (int j = 0; j < 4; ++j) near |= fabs(fabs(x[j]) - t) <= 1e-12 * t;
    exact = __any_sync(kFull, near);
  }
  if (exact) {
    // sum of squares in index order 0..127 (quantizer.cpp:43-44)
#pragma unroll
    for (int j = 0; j < 4; ++j) sq[lane * 4 + j] = sq4[j];
    __syncwarp();
    double sumsq = 0.0;
#pragma unroll 16
    for (int e = 0; e < kHeadDim; ++e) sumsq = __dadd_rn(sumsq, sq[e]);
    __syncwarp();
    sigma = __dsqrt_rn(__ddiv_rn(sumsq, (double)kHeadDim));
  }
  const bool ok = isfinite(sigma) && sigma != 0.0;
  const double t_hi = __dmul_rn(kQ28, sigma);
  const double t_lo = __dmul_rn(-kQ28, sigma);
  uint32_t code[4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    code[j] = ok ? (uint32_t)(x[j] > t_lo) + (uint32_t)(x[j] > 0.0) + (uint32_t)(x[j] > t_hi) : 0u;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    out.lo[j] = __ballot_sync(kFull, code[j] & 1u);
    out.hi[j] = __ballot_sync(kFull, code[j] >> 1);
  }
  return ok;
}

// fp32 route with a certified margin. The reference decides every code by
// comparing fp64 values (y against -t, 0, +t, t = kQ28 sigma). Here y is the
// same butterfly network in fp32 and sigma comes from the fp32 sum of x^2
// (Parseval: sum y^2 = sum x^2 for the orthonormal transform). Rounding
// bounds (7 stages of add + multiply, 128-term sums, u = 2^-24): every fp32 y
// is within 14 u sqrt(128) sigma of the exact real value and the fp32
// threshold within ~65 u sigma of the exact one; the reference's fp64 values
// are within ~1e-14 sigma of the exact ones. A code is certain when y is
// farther than E = 2^-15 sigma (~3.05e-5 sigma, > 2x the sum of those bounds)
// from every threshold; otherwise (about 0.3 % of Gaussian vectors) — or for
// scales where fp32 squares leave the normal range — the warp takes the exact
// fp64 path above. Returns 1 certain / 0 degenerate (as encode128_warp) /
// -1 not certified (out untouched).
template <int N>
__device__ __forceinline__ void encode128_warp_f32n(const float (&in)[N][4], Code (&out)[N], int (&res)[N]) {
  const int lane = threadIdx.x & 31;
  constexpr float c = 0.70710678118654752440f;
  float x[N][4], sq[N];
#pragma unroll
  for (int n = 0; n < N; ++n) {
#pragma unroll
    for (int j = 0; j < 4; ++j) x[n][j] = in[n][j];
    sq[n] = __fmul_rn(x[n][0], x[n][0]);
    sq[n] = __fadd_rn(sq[n], __fmul_rn(x[n][1], x[n][1]));
    sq[n] = __fadd_rn(sq[n], __fmul_rn(x[n][2], x[n][2]));
    sq[n] = __fadd_rn(sq[n], __fmul_rn(x[n][3], x[n][3]));
    const float a0 = x[n][0], b0 = x[n][1], a1 = x[n][2], b1 = x[n][3];
    x[n][0] = __fmul_rn(__fadd_rn(a0, b0), c);
    x[n][1] = __fmul_rn(__fsub_rn(a0, b0), c);
    x[n][2] = __fmul_rn(__fadd_rn(a1, b1), c);
    x[n][3] = __fmul_rn(__fsub_rn(a1, b1), c);
    const float a2 = x[n][0], b2 = x[n][2], a3 = x[n][1], b3 = x[n][3];
    x[n][0] = __fmul_rn(__fadd_rn(a2, b2), c);
    x[n][2] = __fmul_rn(__fsub_rn(a2, b2), c);
    x[n][1] = __fmul_rn(__fadd_rn(a3, b3), c);
    x[n][3] = __fmul_rn(__fsub_rn(a3, b3), c);
  }
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    const bool upper = (lane & m) != 0;
#pragma unroll
    for (int n = 0; n < N; ++n) {
      sq[n] = __fadd_rn(sq[n], __shfl_xor_sync(kFull, sq[n], m));
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float pj = __shfl_xor_sync(kFull, x[n][j], m);
        x[n][j] = upper ? __fmul_rn(__fsub_rn(pj, x[n][j]), c) : __fmul_rn(__fadd_rn(x[n][j], pj), c);
      }
    }
  }
#pragma unroll
  for (int n = 0; n < N; ++n) {
    // sq (warp-uniform) = sum x^2; usable range keeps every bound relative
    if (!(sq[n] > 1e-30f && sq[n] < 1e37f)) { res[n] = -1; continue; }
    const float sigma = __fsqrt_rn(__fdiv_rn(sq[n], 128.f));
    const float t = __fmul_rn(0.6744897501960817432f, sigma);
    const float E = sigma * 3.0517578125e-5f;  // 2^-15 sigma
    bool unsure = false;
    uint32_t code[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float y = x[n][j], ay = fabsf(y);
      unsure |= ay <= E || fabsf(ay - t) <= E;
      code[j] = (uint32_t)(y > -t) + (uint32_t)(y > 0.f) + (uint32_t)(y > t);
    }
    if (__any_sync(kFull, unsure)) { res[n] = -1; continue; }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      out[n].lo[j] = __ballot_sync(kFull, code[j] & 1u);
      out[n].hi[j] = __ballot_sync(kFull, code[j] >> 1);
    }
    res[n] = 1;
  }
}
__device__ __forceinline__ int encode128_warp_f32(const float in[4], Code& out) {
  float v[1][4] = {{in[0], in[1], in[2], in[3]}};
  Code o[1];
  int r[1];
  encode128_warp_f32n<1>(v, o, r);
  if (r[0] == 1) out = o[0];
  return r[0];
}

// Throughput form of the certified fp32 route, for bulk encodes (prefill):
// a warp encodes FOUR vectors at once, lanes 8g .. 8g+7 holding vector g,
// lane L of a group the 16 consecutive elements 16L .. 16L+15. The first
// four butterfly stages are in-register, only three cross lanes (instead of
// five at 4 elements per lane), and the network is left unnormalized:
// Y = sqrt(128) y exactly in real arithmetic, and y > t  <=>  Y > kQ28 ||x||,
// so no per-stage multiply is needed. Rounding bound (u = 2^-24, first
// order): the 2^(7-s) stage-s ancestors of an output are signed sums over a
// partition of the inputs into sets of 2^s, so sum_j v_j^2 <= 2^s ||x||^2 and
// (Cauchy-Schwarz) sum_j |v_j| <= sqrt(128) ||x||; each carries one rounding
// <= u |v_j| into the output with weight +-1, so |Y - Y_exact| <=
// 7 sqrt(128) u ||x||, i.e. 7 u ||x|| = 4.7e-6 sigma in y units (the
// normalized 32-lane route's bound is 14 u ||x||: it also rounds a multiply
// per stage). The fp32 sum of squares (19 additions of non-negative terms) and
// the square root put the threshold within ~11 u t = 4.4e-7 sigma; the
// reference's fp64 values are within ~1e-14 sigma. A code is certain when Y is
// farther than E = 2^-15 ||x|| (= 3.05e-5 sigma in y units, ~6x the total)
// from every threshold. Out (uniform within a group): res 1 certain / -1 not certified
// (also for sums of squares outside [1e-30, 1e37]: the exact path decides,
// including degenerate vectors); `out` = the group's code in every lane.
__device__ __forceinline__ int encode128_g8_f32(const float (&in)[16], Code& out) {
  const int lane = threadIdx.x & 31, L = lane & 7;
  float v[16];
  float sq = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    v[i] = in[i];
    sq = __fmaf_rn(v[i], v[i], sq);
  }
#pragma unroll
  for (int h = 1; h < 16; h <<= 1) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i & h) continue;
      const float a = v[i], b = v[i + h];
      v[i] = __fadd_rn(a, b);
      v[i + h] = __fsub_rn(a, b);
    }
  }
#pragma unroll
  for (int m = 1; m < 8; m <<= 1) {
    const float sgn = (L & m) ? -1.f : 1.f;  // lower: a + b; upper: a - b (a = the partner's)
    sq = __fadd_rn(sq, __shfl_xor_sync(kFull, sq, m));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __fmaf_rn(sgn, v[i], __shfl_xor_sync(kFull, v[i], m));
  }
  const float S = __fsqrt_rn(sq);  // ||x||
  const float Tq = __fmul_rn(0.6744897501960817432f, S);
  const float E = S * 3.0517578125e-5f;
  bool unsure = !(sq > 1e-30f && sq < 1e37f);
  uint32_t lo[4] = {0u, 0u, 0u, 0u}, hi[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float y = v[i], ay = fabsf(y);
    unsure |= ay <= E || fabsf(ay - Tq) <= E;
    const uint32_t c = (uint32_t)(y > -Tq) + (uint32_t)(y > 0.f) + (uint32_t)(y > Tq);
    // element 16 L + i: word i % 4, bit 4 L + i / 4
    lo[i & 3] |= (c & 1u) << (i >> 2);
    hi[i & 3] |= (c >> 1) << (i >> 2);
  }
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    lo[w] <<= 4 * L;
    hi[w] <<= 4 * L;
  }
#pragma unroll
  for (int m = 1; m < 8; m <<= 1) {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      lo[w] |= __shfl_xor_sync(kFull, lo[w], m);
      hi[w] |= __shfl_xor_sync(kFull, hi[w], m);
    }
  }
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    out.lo[w] = lo[w];
    out.hi[w] = hi[w];
  }
  const unsigned grp = 0xffu << (lane & 24);
  return (__ballot_sync(kFull, unsure) & grp) ? -1 : 1;
}

// The encoder used on the hot paths: certified fp32, exact fp64 fallback.
// exact = true forces the fp64 path (diagnostics / tests).
__device__ __forceinline__ bool encode128(const float in[4], double* sq, Code& out, bool exact = false) {
  if (!exact) {
    const int r = encode128_warp_f32(in, out);
    if (r >= 0) return r == 1;
  }
  return encode128_warp(in, sq, out, !exact);
}

// ---------------------------------------------------------------------------
// mbarrier + bulk-copy (TMA engine, non-tensor) helpers.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
// Adds `bytes` to the pending transaction count without arriving.
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// Waiting loop with nanosleep back-off, for a thread whose spinning would
// steal issue slots from compute warps of the same SM sub-partition (the
// warp arbiter favours the highest warp id, i.e. the producer warp).
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) __nanosleep(64);
}
// Bulk L2 prefetch (TMA engine, no shared-memory destination).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// ---------------------------------------------------------------------------
// Cluster / DSMEM primitives. Remote shared-memory traffic uses st.async with
// mbarrier transaction counting on the receiving CTA, so no cluster-wide
// barrier (and no GPU-scope fence) sits on the data path.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_v4(uint32_t remote_addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                            uint32_t remote_bar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
          remote_addr),
      "r"(a), "r"(b), "r"(c), "r"(d), "r"(remote_bar)
      : "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait;" ::: "memory"); }
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// Orders this thread's prior generic-proxy shared-memory accesses before
// subsequent async-proxy (bulk copy) accesses.
__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 16-byte global -> shared asynchronous copy (LDGSTS, per-lane addresses) and
// the mbarrier arrival that fires once this thread's prior cp.async complete.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// Programmatic dependent launch (PDL): wait for the predecessor grid's
// completion + memory visibility / allow the dependent grid to launch.
__device__ __forceinline__ void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Per-thread L2 prefetch of one 128-byte line. (The bulk TMA prefetch takes
// warp-uniform operands, so divergent per-lane use serializes; this does not.)
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}

__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(kFull, v, m);
  return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(kFull, v, m);
  return v;
}

}  // namespace adamas_dev
