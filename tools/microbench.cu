// Design-settling microbenchmarks for the Adamas decode hot path on B200.
// Not product code: measures the hardware constants the kernel design depends
// on (streaming read bandwidth, shared-memory histogram cost, bit-plane
// distance ALU rate, launch gaps, cluster / global barrier latency).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void flush_kernel(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(i, i, i, i);
}

template <int UNROLL>
__global__ void ldg_stream(const uint4* __restrict__ p, size_t n, uint32_t* out) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (UNROLL - 1) * stride < n; i += UNROLL * stride) {
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint4* a = p + i + u * stride;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(a));
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n; i += stride) { uint4 v = p[i]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Each CTA streams a contiguous range via a STAGES-deep ring of bulk copies.
template <int STAGES, int STAGE_BYTES>
__global__ void __launch_bounds__(256) bulk_stream(const uint8_t* __restrict__ p, size_t bytes_per_cta, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[STAGES];
  const uint8_t* base = p + blockIdx.x * bytes_per_cta;
  const int nstage = (int)(bytes_per_cta / STAGE_BYTES);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES && s < nstage; ++s) {
      mbar_expect_tx(&full[s], STAGE_BYTES);
      bulk_g2s(smem + s * STAGE_BYTES, base + (size_t)s * STAGE_BYTES, STAGE_BYTES, &full[s]);
    }
  }
  uint32_t acc = 0;
  for (int it = 0; it < nstage; ++it) {
    const int s = it % STAGES;
    mbar_wait(&full[s], (it / STAGES) & 1);
    const uint4* sp = reinterpret_cast<const uint4*>(smem + s * STAGE_BYTES);
    for (int j = threadIdx.x; j < STAGE_BYTES / 16; j += blockDim.x) { uint4 v = sp[j]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
    __syncthreads();
    if (threadIdx.x == 0 && it + STAGES < nstage) {
      mbar_expect_tx(&full[s], STAGE_BYTES);
      bulk_g2s(smem + s * STAGE_BYTES, base + (size_t)(it + STAGES) * STAGE_BYTES, STAGE_BYTES, &full[s]);
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// Shared-memory histogram of 8192 distances (concentrated 100..200) with atomics.
__global__ void atoms_hist(uint32_t* out, long long* cycles) {
  __shared__ uint32_t hist[400];
  __shared__ uint16_t vals[8192];
  for (int i = threadIdx.x; i < 400; i += blockDim.x) hist[i] = 0;
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) {
    uint32_t h = (i * 2654435761u + blockIdx.x) >> 7;
    vals[i] = 100 + (h % 50) + ((h >> 8) % 50);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) atomicAdd(&hist[vals[i]], 1u);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) { cycles[blockIdx.x] = t1 - t0; out[blockIdx.x] = hist[150]; }
}

// Bit-plane L1 distance over tokens resident in smem; G query heads.
template <int G>
__global__ void __launch_bounds__(256) bitplane_alu(const uint4* __restrict__ codes, int reps, uint32_t* out, long long* cycles) {
  __shared__ uint4 sc[1024 * 2];  // 1024 tokens x 32 B
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sc[i] = codes[i];
  uint32_t ql[G][4], qh[G][4], qx[G][4];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      ql[g][w] = 0x9e3779b9u * (g + 1) + w; qh[g][w] = 0x7f4a7c15u * (g + 3) + w; qx[g][w] = ql[g][w] ^ qh[g][w];
    }
  __syncthreads();
  long long t0 = clock64();
  uint32_t best = 0xffffffffu;
  for (int r = 0; r < reps; ++r) {
    for (int t = threadIdx.x; t < 1024; t += blockDim.x) {
      uint4 lo = sc[2 * t], hi = sc[2 * t + 1];
      uint32_t kl[4] = {lo.x, lo.y, lo.z, lo.w}, kh[4] = {hi.x, hi.y, hi.z, hi.w};
#pragma unroll
      for (int g = 0; g < G; ++g) {
        uint32_t d = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          uint32_t L = ql[g][w] ^ kl[w];
          uint32_t A = (qh[g][w] ^ kh[w]) & ~(L & qx[g][w]);
          d += __popc(L) + 2 * __popc(A);
        }
        best = min(best, (d << 16) | (t ^ r));
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (best == 7) out[0] = best;
}

__global__ void empty_kernel() {}

__global__ void __cluster_dims__(4, 1, 1) cluster_barrier_kernel(int iters, long long* cycles) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) cycles[blockIdx.x / 4] = t1 - t0;
}

// Global spin barrier across groups of `members` CTAs (generation counter).
__global__ void global_barrier_kernel(int iters, int members, unsigned* counters, long long* cycles) {
  const int group = blockIdx.x / members;
  unsigned* ctr = counters + group * 32;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned target = (unsigned)(i + 1) * members;
      __threadfence();
      atomicAdd(ctr, 1u);
      unsigned v;
      do { asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr)); } while (v < target);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x % members == 0) cycles[group] = t1 - t0;
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) { float ms; CK(cudaEventElapsedTime(&ms, a, b)); return ms; }

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s SMs=%d clock=%d kHz l2=%d MB smem/blk optin=%zu\n", prop.name, prop.multiProcessorCount,
         prop.clockRate, prop.l2CacheSize >> 20, prop.sharedMemPerBlockOptin);
  const int nsm = prop.multiProcessorCount;
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  size_t big = 1ull << 30;  // 1 GiB
  uint8_t* buf; CK(cudaMalloc(&buf, big));
  uint4* flushbuf; size_t flushn = (512ull << 20) / 16; CK(cudaMalloc(&flushbuf, flushn * 16));
  uint32_t* out; CK(cudaMalloc(&out, 1 << 20));
  long long* cyc; CK(cudaMalloc(&cyc, 1 << 20));
  CK(cudaMemset(buf, 1, big));
  auto flush = [&]() { flush_kernel<<<nsm * 4, 512>>>(flushbuf, flushn); };

  // A. streaming read bandwidth
  for (size_t sz : {32ull << 20, 1ull << 30}) {
    for (int grid : {nsm, 2 * nsm, 4 * nsm, 8 * nsm, 128}) {
      float best = 1e9;
      for (int r = 0; r < 5; ++r) {
        flush(); CK(cudaEventRecord(e0));
        ldg_stream<8><<<grid, 256>>>((const uint4*)buf, sz / 16, out);
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        best = std::min(best, time_ms(e0, e1));
      }
      printf("ldg_stream size=%zuMB grid=%d: %.2f us  %.1f GB/s\n", sz >> 20, grid, best * 1e3, sz / best / 1e6);
    }
  }
  {
    constexpr int ST = 4, SB = 16384;
    auto k = bulk_stream<ST, SB>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * SB));
    for (size_t sz : {32ull << 20, 1ull << 30}) {
      for (int grid : {128, nsm, 2 * nsm, 256}) {
        size_t per = (sz / grid) / SB * SB;
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
          flush(); CK(cudaEventRecord(e0));
          k<<<grid, 256, ST * SB>>>(buf, per, out);
          CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
          best = std::min(best, time_ms(e0, e1));
        }
        printf("bulk_stream ST=%d SB=%d size=%zuMB grid=%d: %.2f us  %.1f GB/s\n", ST, SB, sz >> 20, grid, best * 1e3,
               per * grid / best / 1e6);
      }
    }
    constexpr int ST2 = 6, SB2 = 32768;
    auto k2 = bulk_stream<ST2, SB2>;
    CK(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, ST2 * SB2));
    for (int grid : {128, nsm}) {
      size_t sz = 32ull << 20; size_t per = (sz / grid) / SB2 * SB2;
      float best = 1e9;
      for (int r = 0; r < 5; ++r) {
        flush(); CK(cudaEventRecord(e0));
        k2<<<grid, 256, ST2 * SB2>>>(buf, per, out);
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        best = std::min(best, time_ms(e0, e1));
      }
      printf("bulk_stream ST=%d SB=%d size=32MB grid=%d: %.2f us  %.1f GB/s\n", ST2, SB2, grid, best * 1e3, per * grid / best / 1e6);
    }
  }
  CK(cudaGetLastError());

  // B. smem atomics histogram
  {
    atoms_hist<<<nsm, 256>>>(out, cyc); CK(cudaDeviceSynchronize());
    std::vector<long long> h(nsm); CK(cudaMemcpy(h.data(), cyc, nsm * 8, cudaMemcpyDeviceToHost));
    long long mx = 0; for (auto v : h) mx = std::max(mx, v);
    printf("atoms_hist 8192 vals/CTA, 256 thr: max %lld cycles (%.2f cyc/val)\n", mx, mx / 8192.0);
  }
  // C. bit-plane ALU
  {
    uint4* codes; CK(cudaMalloc(&codes, 8192 * 16)); CK(cudaMemset(codes, 0x5a, 8192 * 16));
    int reps = 64;
    bitplane_alu<1><<<nsm, 256>>>(codes, reps, out, cyc); CK(cudaDeviceSynchronize());
    std::vector<long long> h(nsm); CK(cudaMemcpy(h.data(), cyc, nsm * 8, cudaMemcpyDeviceToHost));
    long long mx = 0; for (auto v : h) mx = std::max(mx, v);
    printf("bitplane G=1: %.3f cycles/token/SM (1 CTA/SM)\n", (double)mx / (1024.0 * reps));
    CK(cudaEventRecord(e0));
    bitplane_alu<1><<<nsm * 4, 256>>>(codes, reps, out, cyc);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    printf("bitplane G=1 grid 4x: %.1f Gtok/s\n", 1024.0 * reps * nsm * 4 / time_ms(e0, e1) / 1e6);
    CK(cudaEventRecord(e0));
    bitplane_alu<4><<<nsm * 4, 256>>>(codes, reps, out, cyc);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    printf("bitplane G=4 grid 4x: %.1f Gtok/s (token = 4 q-heads)\n", 1024.0 * reps * nsm * 4 / time_ms(e0, e1) / 1e6);
  }
  // D. launch gaps
  {
    for (int i = 0; i < 10; ++i) empty_kernel<<<1, 32>>>();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int i = 0; i < 200; ++i) empty_kernel<<<nsm, 256>>>();
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    printf("empty kernel stream: %.2f us/launch\n", time_ms(e0, e1) * 1e3 / 200);
    cudaStream_t s; CK(cudaStreamCreate(&s));
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < 200; ++i) empty_kernel<<<nsm, 256, 0, s>>>();
    CK(cudaStreamEndCapture(s, &g)); CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, s)); CK(cudaStreamSynchronize(s));
    CK(cudaEventRecord(e0, s)); CK(cudaGraphLaunch(ge, s)); CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
    printf("empty kernel graph: %.2f us/launch\n", time_ms(e0, e1) * 1e3 / 200);
  }
  // E. barriers
  {
    int iters = 1000;
    cluster_barrier_kernel<<<128, 256>>>(iters, cyc); CK(cudaDeviceSynchronize());
    long long h; CK(cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost));
    printf("cluster(4) barrier: %.1f cycles\n", (double)h / iters);
    unsigned* ctr; CK(cudaMalloc(&ctr, 64 * 32 * 4)); CK(cudaMemset(ctr, 0, 64 * 32 * 4));
    iters = 200;
    global_barrier_kernel<<<128, 256>>>(iters, 4, ctr, cyc); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost));
    printf("global spin barrier (4 CTAs/group, 32 groups): %.1f cycles\n", (double)h / iters);
    CK(cudaMemset(ctr, 0, 64 * 32 * 4));
    global_barrier_kernel<<<128, 256>>>(iters, 16, ctr, cyc); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost));
    printf("global spin barrier (16 CTAs/group): %.1f cycles\n", (double)h / iters);
  }
  CK(cudaGetLastError());
  printf("done\n");
  return 0;
}
