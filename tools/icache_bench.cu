// Instruction-fetch cost of straight-line code executed once per CTA
// (design question: does a large single-pass kernel pay for I-cache misses?).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define OP(k) x = (x ^ (k * 0x9e3779b9u)) + (y >> (k & 7)); y = y * 3u + (x ^ k);
#define OP8(k) OP(k) OP(k+1) OP(k+2) OP(k+3) OP(k+4) OP(k+5) OP(k+6) OP(k+7)
#define OP64(k) OP8(k) OP8(k+8) OP8(k+16) OP8(k+24) OP8(k+32) OP8(k+40) OP8(k+48) OP8(k+56)
#define OP512(k) OP64(k) OP64(k+64) OP64(k+128) OP64(k+192) OP64(k+256) OP64(k+320) OP64(k+384) OP64(k+448)

__global__ void __launch_bounds__(512) straight(uint32_t* out, long long* cyc, int reps) {
  uint32_t x = threadIdx.x, y = blockIdx.x;
  long long t[5];
  for (int r = 0; r < reps; ++r) {
    t[r] = clock64();
    OP512(0) OP512(512) OP512(1024) OP512(1536)
  }
  t[reps] = clock64();
  if (threadIdx.x == 0) for (int r = 0; r < reps; ++r) cyc[blockIdx.x * 4 + r] = t[r + 1] - t[r];
  if (x == 12345u) out[0] = y;
}

int main() {
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, 64); cudaMalloc(&cyc, 148 * 4 * 8);
  for (int launch = 0; launch < 3; ++launch) {
    straight<<<128, 512>>>(out, cyc, 4);
    cudaDeviceSynchronize();
    long long h[128 * 4];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double m[4] = {0, 0, 0, 0};
    for (int b = 0; b < 128; ++b) for (int r = 0; r < 4; ++r) m[r] += h[b * 4 + r] / 128.0;
    printf("launch %d: cycles per pass (4096 ops x2 per thread, 16 warps): rep0 %.0f rep1 %.0f rep2 %.0f rep3 %.0f\n",
           launch, m[0], m[1], m[2], m[3]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
