// Instruction-fetch cost of straight-line code executed once per CTA
// (design question: does a large single-pass kernel pay for I-cache misses?).
// Straight-line blocks of NB x OP64 (~300 instructions, ~4.8 KB each); one CTA
// of 16 warps per SM (128 CTAs), the code run `reps` times back to back inside
// the kernel. rep0 pays the fetch from L2 (or from the SM's instruction cache
// when the previous launch left it there); later reps show whether the code
// fits the SM's instruction cache. Dependent ALU chain: ~4 cycles/op ideal.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define OP(k) x = (x ^ (k * 0x9e3779b9u)) + (y >> (k & 7)); y = y * 3u + (x ^ k);
#define OP8(k) OP(k) OP(k+1) OP(k+2) OP(k+3) OP(k+4) OP(k+5) OP(k+6) OP(k+7)
#define OP64(k) OP8(k) OP8(k+8) OP8(k+16) OP8(k+24) OP8(k+32) OP8(k+40) OP8(k+48) OP8(k+56)

template <int NB>
__global__ void __launch_bounds__(512) straight(uint32_t* out, long long* cyc, int reps) {
  uint32_t x = threadIdx.x, y = blockIdx.x;
  long long t[5];
  for (int r = 0; r < reps; ++r) {
    t[r] = clock64();
#pragma unroll
    for (int b = 0; b < NB; ++b) { OP64(b * 64) }
  }
  t[reps] = clock64();
  if (threadIdx.x == 0) for (int r = 0; r < reps; ++r) cyc[blockIdx.x * 4 + r] = t[r + 1] - t[r];
  if (x == 12345u) out[0] = y;
}

template <int NB>
void run(uint32_t* out, long long* cyc) {
  for (int launch = 0; launch < 3; ++launch) {
    straight<NB><<<128, 512>>>(out, cyc, 4);
    cudaDeviceSynchronize();
    long long h[128 * 4];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double m[4] = {0, 0, 0, 0};
    for (int b = 0; b < 128; ++b) for (int r = 0; r < 4; ++r) m[r] += h[b * 4 + r] / 128.0;
    printf("NB %2d (%5d ops) launch %d: cycles per pass rep0 %6.0f rep1 %6.0f rep2 %6.0f rep3 %6.0f  (%.2f cyc/op warm)\n",
           NB, NB * 64, launch, m[0], m[1], m[2], m[3], m[3] / (NB * 64));
  }
}

int main() {
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, 64); cudaMalloc(&cyc, 148 * 4 * 8);
  run<1>(out, cyc);
  run<4>(out, cyc);
  run<8>(out, cyc);
  run<16>(out, cyc);
  run<32>(out, cyc);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
