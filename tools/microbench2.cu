// Latency microbenchmarks for the post-scan phases (one 512-thread CTA/SM).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ long long clk() { return clock64(); }

__global__ void __launch_bounds__(512, 1) lat_kernel(const uint32_t* __restrict__ g, uint32_t* out, long long* res) {
  __shared__ uint32_t sm[4096];
  __shared__ volatile int sink;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 4096; i += 512) sm[i] = (i * 7 + 1) & 4095;
  __syncthreads();
  long long t0, t1;
  uint32_t acc = 0;
  // 1. dependent LDS chain (pointer chase), 64 hops, warp 0
  if (warp == 0) {
    uint32_t p = lane;
    t0 = clk();
    for (int i = 0; i < 64; ++i) p = sm[p];
    t1 = clk();
    acc += p;
    if (tid == 0) res[blockIdx.x * 16 + 0] = (t1 - t0) / 64;
  }
  __syncthreads();
  // 2. 100 back-to-back __syncthreads with 16 warps
  t0 = clk();
  for (int i = 0; i < 100; ++i) { __syncthreads(); acc += sink; }
  t1 = clk();
  if (tid == 0) res[blockIdx.x * 16 + 1] = (t1 - t0) / 100;
  // 3. dependent IADD chain (ALU latency), 256 ops
  {
    uint32_t x = tid;
    t0 = clk();
#pragma unroll 1
    for (int i = 0; i < 256; ++i) x = x * 3u + 1u;
    t1 = clk();
    acc += x;
    if (tid == 0) res[blockIdx.x * 16 + 2] = (t1 - t0) / 256;
  }
  __syncthreads();
  // 4. ballot + popc dependent chain, 64 iterations
  {
    uint32_t x = lane;
    t0 = clk();
    for (int i = 0; i < 64; ++i) x += __popc(__ballot_sync(0xffffffffu, (x & 1) != 0));
    t1 = clk();
    acc += x;
    if (tid == 0) res[blockIdx.x * 16 + 3] = (t1 - t0) / 64;
  }
  __syncthreads();
  // 5. shfl chain
  {
    uint32_t x = lane;
    t0 = clk();
    for (int i = 0; i < 64; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1;
    t1 = clk();
    acc += x;
    if (tid == 0) res[blockIdx.x * 16 + 4] = (t1 - t0) / 64;
  }
  __syncthreads();
  // 6. issue cost of 32 prefetch.global.L2 per lane (warp 0 only), then barrier
  if (warp == 0) {
    t0 = clk();
    for (int i = 0; i < 32; ++i) {
      const uint32_t* a = g + ((size_t)blockIdx.x * 65536 + (size_t)(lane * 32 + i) * 32);
      asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(a));
    }
    t1 = clk();
    if (tid == 0) res[blockIdx.x * 16 + 5] = (t1 - t0);
  }
  __syncthreads();
  // 7. global load latency (cold, HBM), warp 0: dependent chain of 8
  if (warp == 0) {
    uint32_t p = (blockIdx.x * 1000003u + lane * 7919u) & ((1u << 24) - 1);
    t0 = clk();
    for (int i = 0; i < 8; ++i) p = (g[p] + p * 2654435761u) & ((1u << 24) - 1);
    t1 = clk();
    acc += p;
    if (tid == 0) res[blockIdx.x * 16 + 6] = (t1 - t0) / 8;
  }
  // 8. work of 400 independent-ish instructions in 1 warp vs 16 warps
  __syncthreads();
  {
    t0 = clk();
    if (warp == 0) {
      uint32_t a[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = sm[lane * 16 + i];
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = a[i] * 3u + (a[(i + 1) & 15] >> 3);
      uint32_t s = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) s += a[i];
      acc += s;
    }
    __syncthreads();
    t1 = clk();
    if (tid == 0) res[blockIdx.x * 16 + 7] = (t1 - t0);
  }
  {
    t0 = clk();
    {
      uint32_t a[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = sm[lane * 16 + i];
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = a[i] * 3u + (a[(i + 1) & 15] >> 3);
      uint32_t s = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) s += a[i];
      acc += s;
    }
    __syncthreads();
    t1 = clk();
    if (tid == 0) res[blockIdx.x * 16 + 8] = (t1 - t0);
  }
  if (acc == 0x12345u) out[0] = acc;
}

int main() {
  uint32_t* g; uint32_t* out; long long* res;
  cudaMalloc(&g, (size_t)256 << 20); cudaMemset(g, 0, (size_t)256 << 20);
  cudaMalloc(&out, 64); cudaMalloc(&res, 148 * 16 * 8); cudaMemset(res, 0, 148 * 16 * 8);
  for (int it = 0; it < 2; ++it) {
    lat_kernel<<<128, 512>>>(g, out, res);
    cudaDeviceSynchronize();
  }
  long long h[128 * 16];
  cudaMemcpy(h, res, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"LDS dep latency (cyc)", "__syncthreads x16 warps (cyc)", "IMAD dep latency (cyc)",
                         "ballot+popc dep (cyc)", "shfl dep (cyc)", "32 L2 prefetch issue (cyc)",
                         "global dep load HBM (cyc)", "1 warp 400-instr + bar (cyc)", "16 warps 400-instr + bar (cyc)"};
  for (int k = 0; k < 9; ++k) {
    double m = 0; long long mx = 0;
    for (int b = 0; b < 128; ++b) { m += h[b * 16 + k] / 128.0; if (h[b * 16 + k] > mx) mx = h[b * 16 + k]; }
    printf("%-34s mean %8.1f max %lld\n", names[k], m, mx);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
