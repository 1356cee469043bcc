// How many thread-block clusters of C CTAs (544 threads, `smem` KB dynamic
// shared memory each, one CTA per SM) co-reside on this GPU, C = 1..16.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void dummy(int* p) { extern __shared__ int s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main(int argc, char** argv) {
  int kb = argc > 1 ? atoi(argv[1]) : 200;
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, kb * 1024);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int c = 1; c <= 16; c *= 2) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(c * 64);
    cfg.blockDim = dim3(544);
    cfg.dynamicSmemBytes = kb * 1024;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = c; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
    printf("smem %d KB cluster %2d: max active clusters %d (%d CTAs) %s\n", kb, c, n, n * c, cudaGetErrorString(e));
  }
  return 0;
}
