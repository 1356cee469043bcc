// Latency of the warp encoder (encode128_warp) inside different CTA contexts:
// alone, with the other warps parked at a named barrier, and with a bulk-copy
// stream in flight into shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2510_18413_b200/csrc -o tools/encode_bench tools/encode_bench.cu
#include <cuda_runtime.h>
#include <cstdio>

#include "common.cuh"

using namespace adamas_dev;

template <int MODE>
__global__ void __launch_bounds__(544, 1) enc(const float* q, const uint4* src, long long* cyc, uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ double sq[128];
  __shared__ uint64_t bar;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 512) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    if (MODE & 1) {
      mbar_expect_tx(&bar, 5 * 32768);
      for (int s = 0; s < 5; ++s) bulk_g2s(smem + s * 32768, src + (size_t)blockIdx.x * 10240 + s * 2048, 32768, &bar);
    }
  }
  float f[4];
  for (int j = 0; j < 4; ++j) f[j] = q[(blockIdx.x * 128 + lane * 4 + j) & 4095];
  __syncthreads();
  if (MODE & 8) cluster_arrive_relaxed();
  if (warp == 0) {
    Code c;
    if ((MODE & 16) && lane == 0) sink[8 + blockIdx.x] = (uint32_t)clock64();
    if ((MODE & 32)) sink[16 + blockIdx.x * 32 + lane] = __float_as_uint(f[0]);
    const long long t0 = clock64();
    const bool ok = encode128_warp(f, sq, c, (MODE & 2) == 0);
    const long long t1 = clock64() + (c.lo[0] & 0);
    if (lane == 0) {
      cyc[blockIdx.x] = t1 - t0;
      if (!ok) sink[0] = c.hi[1];
    }
  }
  if ((MODE & 4) && warp < 16) asm volatile("bar.sync 1, 512;" ::: "memory");
  if ((MODE & 1) && threadIdx.x == 0) mbar_wait(&bar, 0);
  if (MODE & 8) cluster_wait();
}

template <int MODE>
void run(const char* name, const float* q, const uint4* src, long long* cyc, uint32_t* sink, int smem) {
  cudaFuncSetAttribute(enc<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int r = 0; r < 3; ++r) {
    if (MODE & 8) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(128);
      cfg.blockDim = dim3(544);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 4;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, enc<MODE>, q, src, cyc, sink);
    } else {
      enc<MODE><<<128, 544, smem>>>(q, src, cyc, sink);
    }
  }
  cudaDeviceSynchronize();
  long long h[128];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0, mx = 0;
  for (int i = 0; i < 128; ++i) { m += h[i] / 128.0; mx = h[i] > mx ? h[i] : mx; }
  printf("%-40s encode128_warp: mean %.0f cycles (%.2f us @1.965GHz), max %.0f  [%s]\n", name, m, m / 1965.0, mx,
         cudaGetErrorString(cudaGetLastError()));
}

#include <unistd.h>
template <int MODE>
void run_idle(const char* name, const float* q, const uint4* src, long long* cyc, uint32_t* sink, int gap_us) {
  for (int r = 0; r < 4; ++r) {
    usleep(gap_us);
    enc<MODE><<<128, 544, 0>>>(q, src, cyc, sink);
    cudaDeviceSynchronize();
    long long h[128];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 128; ++i) m += h[i] / 128.0;
    printf("%-30s gap %6d us, launch %d: encode128_warp %.0f cycles (%.2f us)\n", name, gap_us, r, m, m / 1965.0);
  }
}

int main() {
  float* q; uint4* src; long long* cyc; uint32_t* sink;
  cudaMalloc(&q, 4096 * 4); cudaMalloc(&src, (size_t)128 * 10240 * 16); cudaMalloc(&cyc, 128 * 8); cudaMalloc(&sink, 1 << 20);
  float hq[4096];
  for (int i = 0; i < 4096; ++i) hq[i] = (float)((i * 7919) % 1000) / 333.0f - 1.5f;
  cudaMemcpy(q, hq, sizeof(hq), cudaMemcpyHostToDevice);
  cudaMemset(src, 1, (size_t)128 * 10240 * 16);
  run<0>("fast, alone", q, src, cyc, sink, 0);
  run<2>("exact, alone", q, src, cyc, sink, 0);
  run<4>("fast, others at named barrier", q, src, cyc, sink, 0);
  run<1>("fast, 160 KB bulk copy in flight", q, src, cyc, sink, 200 * 1024);
  run<5>("fast, bulk copy + named barrier", q, src, cyc, sink, 200 * 1024);
  run<7>("exact, bulk copy + named barrier", q, src, cyc, sink, 200 * 1024);
  run<8>("fast, cluster 4 + arrive before", q, src, cyc, sink, 0);
  run<13>("fast, cluster + bulk + named barrier", q, src, cyc, sink, 200 * 1024);
  run<16>("fast, lane-0 STG right before", q, src, cyc, sink, 0);
  run<32>("fast, warp STG right before", q, src, cyc, sink, 0);
  run_idle<0>("fast", q, src, cyc, sink, 0);
  run_idle<0>("fast", q, src, cyc, sink, 20);
  run_idle<0>("fast", q, src, cyc, sink, 200);
  run_idle<0>("fast", q, src, cyc, sink, 2000);
  return 0;
}
