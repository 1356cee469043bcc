// Scan-phase compute cost per token (cycles/token/SM), data already in shared
// memory: isolates the ALU/XU/LSU cost of the distance formulations and of the
// per-token bookkeeping (distance store, histogram atomics) from HBM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/scan_bench tools/scan_bench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

constexpr int kThreads = 512;
constexpr int kTok = 1024;  // one stage: 2 tokens per thread

struct Q { uint32_t lo[4], hi[4], x[4]; };

__device__ __forceinline__ uint32_t dist_popc(const Q& q, const uint32_t* lo, const uint32_t* hi) {
  uint32_t d = 0;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const uint32_t L = q.lo[w] ^ lo[w];
    const uint32_t A = (q.hi[w] ^ hi[w]) & ~(L & q.x[w]);
    d += __popc(L) + 2u * __popc(A);
  }
  return d;
}

// carry-save reduction of the 4 weight-1 words (L) and 4 weight-2 words (A)
// to 4 popcounts (weights 1, 2, 4, 8)
__device__ __forceinline__ void csa(uint32_t a, uint32_t b, uint32_t c, uint32_t& s, uint32_t& cy) {
  s = a ^ b ^ c;
  cy = (a & b) | (c & (a ^ b));
}
__device__ __forceinline__ uint32_t dist_csa(const Q& q, const uint32_t* lo, const uint32_t* hi) {
  uint32_t L[4], A[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    L[w] = q.lo[w] ^ lo[w];
    A[w] = (q.hi[w] ^ hi[w]) & ~(L[w] & q.x[w]);
  }
  uint32_t s1, c1, s2, c2, s3, c3, s4, c4, s5, c5;
  csa(L[0], L[1], L[2], s1, c1);       // w1: s1, w2: c1
  const uint32_t s1b = s1 ^ L[3], c1b = s1 & L[3];  // w1: s1b, w2: c1b
  csa(A[0], A[1], A[2], s2, c2);       // w2: s2, w4: c2
  csa(A[3], c1, c1b, s3, c3);          // w2: s3, w4: c3
  const uint32_t s4b = s2 ^ s3, c4b = s2 & s3;       // w2: s4b, w4: c4b
  csa(c2, c3, c4b, s5, c5);            // w4: s5, w8: c5
  (void)s4; (void)c4;
  return __popc(s1b) + 2u * __popc(s4b) + 4u * __popc(s5) + 8u * __popc(c5);
}

__device__ __forceinline__ uint32_t dist_bal(const Q& q, const uint32_t* lo, const uint32_t* hi) {
  uint32_t L[4], A[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    L[w] = q.lo[w] ^ lo[w];
    A[w] = (q.hi[w] ^ hi[w]) & ~(L[w] & q.x[w]);
  }
  uint32_t s1, c1, s2, c2, s3, c3;
  csa(L[0], L[1], L[2], s1, c1);
  const uint32_t s1b = s1 ^ L[3], c1b = s1 & L[3];
  csa(A[0], A[1], A[2], s2, c2);
  csa(A[3], c1, c1b, s3, c3);
  return __popc(s1b) + 2u * (__popc(s2) + __popc(s3)) + 4u * (__popc(c2) + __popc(c3));
}

template <int G, int MODE>
__global__ void __launch_bounds__(kThreads, 1) bench(const uint4* __restrict__ src, int iters, uint32_t lim,
                                                      long long* cyc, uint32_t* sink) {
  __shared__ uint4 stage[2 * kTok];
  __shared__ uint16_t dist[G > 4 ? 4 : G][kTok];
  __shared__ int hist[G > 4 ? 4 : G][512];
  for (int i = threadIdx.x; i < 2 * kTok; i += kThreads) stage[i] = src[i];
  for (int i = threadIdx.x; i < (G > 4 ? 4 : G) * 512; i += kThreads) hist[i / 512][i % 512] = 0;
  Q q[G];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      q[g].lo[w] = 0x9e3779b9u * (g * 8 + w + 1);
      q[g].hi[w] = 0x7f4a7c15u * (g * 8 + w + 3);
      q[g].x[w] = q[g].lo[w] ^ q[g].hi[w];
    }
  __syncthreads();
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int base = 0;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = threadIdx.x + u * kThreads;
      const int jj = (j + it * 64) & (kTok - 1);  // varies per iteration: nothing to hoist
      const uint4 a = stage[jj], b = stage[kTok + jj];
      const uint32_t lo[4] = {a.x, a.y, a.z, a.w}, hi[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint32_t d = (MODE & 32) ? dist_bal(q[g], lo, hi) : (MODE & 1) ? dist_csa(q[g], lo, hi) : dist_popc(q[g], lo, hi);
        if (MODE & 2) dist[g & 3][base + j] = (uint16_t)d;
        if (MODE & 4) atomicAdd(&hist[g & 3][d], 1);
        if (MODE & 8) { if (d <= lim) atomicAdd(&hist[g & 3][d], 1); }
        acc += d;
      }
    }
    if (MODE & 16) __syncthreads();
  }
  const long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 0x12345u) sink[0] = hist[0][threadIdx.x & 511] + dist[0][threadIdx.x];
}

template <int G, int MODE>
void run(const char* name, const uint4* src, long long* cyc, uint32_t* sink, uint32_t lim = 140) {
  const int iters = 256;
  bench<G, MODE><<<148, kThreads>>>(src, iters, lim, cyc, sink);
  bench<G, MODE><<<148, kThreads>>>(src, iters, lim, cyc, sink);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 148; ++i) m += h[i] / 148.0;
  printf("G=%d %-34s %.3f cycles/kv-token/SM  (%.3f per q-head)\n", G, name, m / (iters * (double)kTok),
         m / (iters * (double)kTok * G));
}

int main() {
  uint4 h[2 * kTok];
  uint64_t z = 88172645463325252ull;
  for (int i = 0; i < 2 * kTok; ++i) {
    uint32_t w[4];
    for (int k = 0; k < 4; ++k) { z ^= z << 13; z ^= z >> 7; z ^= z << 17; w[k] = (uint32_t)z; }
    h[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  uint4* src; long long* cyc; uint32_t* sink;
  cudaMalloc(&src, sizeof(h)); cudaMalloc(&cyc, 148 * 8); cudaMalloc(&sink, 64);
  cudaMemcpy(src, h, sizeof(h), cudaMemcpyHostToDevice);
  run<1, 0>("popc", src, cyc, sink);
  run<1, 1>("csa", src, cyc, sink);
  run<1, 2>("popc + dist store", src, cyc, sink);
  run<1, 6>("popc + dist store + hist atomic", src, cyc, sink);
  run<1, 10>("popc + dist store + hist if d<=lim", src, cyc, sink);
  run<1, 11>("csa + dist store + hist if d<=lim", src, cyc, sink);
  run<1, 27>("csa + store + lim-hist + sync", src, cyc, sink);
  run<1, 26>("popc + store + lim-hist + sync", src, cyc, sink);
  run<4, 0>("popc", src, cyc, sink);
  run<4, 1>("csa", src, cyc, sink);
  run<4, 10>("popc + dist store + hist if d<=lim", src, cyc, sink);
  run<4, 11>("csa + dist store + hist if d<=lim", src, cyc, sink);
  run<4, 14>("popc + store + hist atomic", src, cyc, sink);
  run<4, 26>("popc + store + lim-hist + sync", src, cyc, sink);
  run<1, 32>("balanced csa (5 popc)", src, cyc, sink);
  run<1, 38>("balanced + store + hist atomic", src, cyc, sink);
  run<4, 32>("balanced csa (5 popc)", src, cyc, sink);
  run<4, 38>("balanced + store + hist atomic", src, cyc, sink);
  run<8, 38>("balanced + store + hist atomic", src, cyc, sink);
  run<8, 10>("popc + dist store + hist if d<=lim", src, cyc, sink);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
