// Dependent-chain latency of warp primitives on sm_100a (cycles per op), one
// warp per SM and 16 warps per SM (all doing the same chain).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_bench tools/lat_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

template <int OP>
__global__ void chain(int n, long long* cyc, int* sink) {
  __shared__ int sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7 + 3) & 1023;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int x = lane;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (OP == 0) x = __shfl_sync(0xffffffffu, x, (x + 1) & 31);           // SHFL.IDX, data-dependent lane
    if (OP == 1) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1;             // SHFL.BFLY
    if (OP == 2) x = (int)__ballot_sync(0xffffffffu, (x & 1) != 0) ^ x;  // VOTE
    if (OP == 3) x = sm[x & 1023];                                       // LDS chain
    if (OP == 4) x = x * 3 + 1;                                          // IMAD chain
    if (OP == 5) x = __popc(x) + x;                                      // POPC chain
    if (OP == 6) x = (int)__reduce_add_sync(0xffffffffu, (unsigned)x) & 1023;  // REDUX
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (x == 0x7fffffff) sink[0] = x;
}

template <int OP>
void run(const char* name, long long* cyc, int* sink) {
  const int n = 1000;
  for (int threads : {32, 512}) {
    chain<OP><<<148, threads>>>(n, cyc, sink);
    chain<OP><<<148, threads>>>(n, cyc, sink);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 148; ++i) m += h[i] / 148.0;
    printf("%-28s %3d threads: %6.1f cycles per dependent op\n", name, threads, m / n);
  }
}

int main() {
  long long* cyc; int* sink;
  cudaMalloc(&cyc, 148 * 8); cudaMalloc(&sink, 64);
  run<0>("shfl.idx (dynamic lane)", cyc, sink);
  run<1>("shfl.bfly + add", cyc, sink);
  run<2>("ballot + xor", cyc, sink);
  run<3>("lds", cyc, sink);
  run<4>("imad", cyc, sink);
  run<5>("popc + add", cyc, sink);
  run<6>("redux.add + and", cyc, sink);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
