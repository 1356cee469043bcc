// fused_decode.cuh — one Adamas decode step of one layer in ONE launch.
//
// Work unit = (sequence, kv-head) with its G = n_q / n_kv query heads. A
// thread-block cluster of C CTAs owns a unit; CTA rank r owns the contiguous
// token range [r * chunk, min(S, (r + 1) * chunk)) where S includes the token
// appended by this very step (Alg. 1: update before estimate).
// Each CTA = 16 consumer warps + 1 producer warp.
//
//   producer  one lane streams the rank's lo/x code planes through a ring of
//             32 KB shared-memory stages with bulk copies (TMA engine), full /
//             empty mbarriers per slot: no CTA-wide barrier in the scan
//   prologue  consumer warps 0..G-1 encode the G query heads (certified fp32
//             FWHT + RMS thresholds, exact fp64 fallback: bit-exact) while the
//             ring fills; in the rank owning position S-1, warp G encodes the
//             new key and appends (k, v, code) (kv_cache.cpp:62-71)
//   scan      each consumer thread turns two tokens per stage into G exact
//             distances (estimator.cpp:45-59), stored as u16 in shared memory
//             and counted in a per-CTA histogram per q-head
//   select    histograms pushed to every rank of the cluster (st.async +
//             mbarrier transaction counts); a block-parallel prefix over the
//             bins gives the threshold T (k-th smallest distance), how many
//             ties at T earlier ranks take and this rank's output offset; an
//             order-preserving compaction over per-thread token spans emits
//             top_k's (score, index) order (estimator.cpp:75-90) with no sort
//   attend    each rank gathers its own selected K/V rows, fp32 online
//             softmax per warp, combines the warps, pushes (m, l, o[128]) to
//             the merging rank over DSMEM; log-sum-exp merge -> out
//             (attention.cpp:8-45 semantics)
//
// Indices are bit-exact by construction: the selection is computed from the
// exact integer distances with the reference's total order, no approximation.
#pragma once
#include "ops.cuh"

namespace adamas_dev {

#ifndef ADAMAS_DIAG
#define ADAMAS_DIAG 0  // 1: phase stamps and timing-only switches (ADAMAS_DBG) compiled in (build.py --diag)
#endif
#ifndef ADAMAS_QPF
#define ADAMAS_QPF 1  // L2-prefetch q / k_new / v_new before the grid-dependency wait
#endif
#ifndef ADAMAS_GATHER_PREFETCH
#define ADAMAS_GATHER_PREFETCH 2  // L2-prefetch the gather rows: 1 all rows <= T in the count pass, 2 survivors in the emit, 0 none
#endif
#ifndef ADAMAS_CWARPS
#define ADAMAS_CWARPS 16  // consumer warps per CTA: 16 (1 CTA/SM) or 8 (2 CTAs/SM)
#endif
constexpr int kConsumerWarps = ADAMAS_CWARPS;
constexpr int kCtasPerSm = kConsumerWarps >= 16 ? 1 : 2;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kProducerWarp = kConsumerWarps;
constexpr int kFusedThreads = kConsumers + 32;
constexpr int kStageTok = 1024;  // tokens per bulk-copy stage: 2 x 16 KB planes
constexpr int kStageBytes = kStageTok * 32;
constexpr int kMaxStages = 8;    // ring depth cap (runtime: FusedParams::stages)
constexpr int kHistBins = 512;   // 2-bit L1 distances at d = 128 are <= 384
constexpr int kMaxG = 8;
constexpr int kMaxSeqs = 64;
constexpr int kPartStride = 132;  // floats per partial: m, l, pad, pad, o[128]
constexpr int kFusedUnsupported = -100;
constexpr int kTokPerThread = 1024 / (kConsumerWarps * 32);  // tokens per consumer thread per stage
constexpr int kTraceTid = (kConsumerWarps - 1) * 32;  // diagnostics: the thread that takes phase stamps

struct FusedSeq {
  uint4* codes;  // this sequence's cache: [n_kv][2 planes][cap] x 16 B
  void* K;       // [n_kv][cap][128]
  void* V;
  int64_t cap;
  int64_t s_old;  // tokens in the cache before this step's append
  int64_t clean;  // tokens [0, clean) were not written by the preceding kernel: streamable before the PDL wait
  int* status;    // this cache's sticky status word
  // multi-cluster units (FusedParams::P > 1): global scratch of this cache
  uint32_t* xhist;  // [unit][P][G][kHistBins] cluster-combined histograms
  float* xpart;     // [unit][P][G][kPartStride] cluster partials
  int* xsync;       // [unit][4]: histogram barrier (count, generation), partial barrier (count, generation)
};

struct FusedParams {
  int n_seqs, n_kv, C, chunk, budget, stages;
  int exact_encode;  // 1: always the sequential fp64 sum (diagnostics / tests)
  int dbg;           // diagnostics only: bit1 no idx stores
  int pdl;           // launched with programmatic stream serialization
  int append;        // 1: append (k_new, v_new) first (decode step); 0: the cache as is
  uint32_t* cand;    // candidates mode: [n_seqs][n_q][budget] keys (dist << 23 | base + token), no attention
  int64_t cand_base; // global index of this cache's token 0 (sequence-sharded caches)
  PeerPush peers;    // candidates mode, peer exchange: keys go to every rank's mailbox (cand unused)
  int qsplit;        // clusters per kv-head: each scans the codes for G of its qsplit * G q-heads
  int P;             // clusters per unit (token ranges); > 1 exchanges through global memory
  const void* q;      // [n_seqs][n_q][128]
  const void* k_new;  // [n_seqs][n_kv][128]
  const void* v_new;
  float* out;    // [n_seqs][n_q][128]
  int32_t* idx;  // [n_seqs][n_q][budget] or null
  unsigned long long* trace;  // optional per-CTA phase timestamps (diagnostics)
  FusedSeq seq[kMaxSeqs];
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// BAR.SYNC on sm_100 blocks lazily (at the next access to barrier-protected
// state), so a stamp taken right after a barrier would record the barrier's
// issue, not its release: the volatile shared load forces the wait.
// Trace clock: SM cycles (clock64), or globaltimer ns with dbg bit 6.
__device__ __forceinline__ unsigned long long trace_clock(int dbg) {
  return (dbg & 64) ? globaltimer_ns() : (unsigned long long)clock64();
}
// Diagnostics (p.trace != null): stamp i is recorded only when selected by
// dbg bits 8..12 (value = (i + 1) << 8), one stamp per launch, so the trace
// does not perturb the phases it measures; stamps 14/15 (globaltimer at CTA
// start / end) are always recorded. BAR.SYNC on sm_100 blocks lazily (at the
// next access to barrier-protected state), so a stamp taken right after a
// barrier would record the barrier's issue, not its release: the volatile
// shared load forces the wait.
#define ADAMAS_TRACE(i)                                                                 \
  do {                                                                                  \
    if (ptrace != nullptr && threadIdx.x == kTraceTid && ((pdbg >> 8) & 31) == (i) + 1) {   \
      __shared__ volatile int trace_sink;                                               \
      const int sink = trace_sink;                                                      \
      ptrace[blockIdx.x * 16 + (i)] = trace_clock(pdbg) + (unsigned long long)(sink & 0);   \
    }                                                                                   \
  } while (0)

// Self-resetting barrier among the CTAs of one multi-cluster unit (one
// thread per CTA; all of them co-resident: the launcher keeps such grids to
// one wave). The generation is read before arriving; the last arriver resets
// the count and advances the generation. Writes before the arrival are made
// visible (fence); waiters give up after ~1 s and latch a status bit rather
// than hang.
__device__ __forceinline__ void unit_barrier(int* bar, int target, bool wait, int* status) {
  volatile int* gen = bar + 1;
  const int g0 = *gen;
  __threadfence();
  const int old = atomicAdd(bar, 1);
  if (old == target - 1) {
    atomicExch(bar, 0);
    __threadfence();
    atomicAdd(bar + 1, 1);
  } else if (wait) {
    for (long long spin = 0; *gen == g0; ++spin) {
      if (spin > (1LL << 24)) {
        atomicOr(status, kStatusSyncTimeout);
        break;
      }
      __nanosleep(32);
    }
  }
  __threadfence();
}

// Named barrier over the 16 consumer warps (the producer warp never joins).
// The explicit __syncwarp makes every warp converged before the aligned
// bar.sync: a warp can reach a consumer barrier diverged (after a divergent
// loop, or an mbarrier spin whose lanes exit on different polls), and an
// aligned barrier reached by part of a warp released the block early
// (measured: wrong tie counts under skewed warps).
__device__ __forceinline__ void consumer_sync() {
  __syncwarp();
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

// Dynamic shared-memory carve-up, identical on host and device.
struct FusedSmem {
  uint32_t stage, dist, hist, hist_all, sel, inbox, wpart, qf, qcode, sq, bars, total;
  __host__ __device__ static uint32_t align(uint32_t x, uint32_t a) { return (x + a - 1u) & ~(a - 1u); }
  __host__ __device__ FusedSmem(int G, int C, int chunk, int selcap, int stages, int P = 1) {
    uint32_t o = 0;
    stage = o; o += (uint32_t)stages * kStageBytes;
    dist = o;  o = align(o + (uint32_t)G * chunk * 2, 16);
    hist = o;  o += (uint32_t)G * kHistBins * 4;
    // u16 histograms received: from every rank for every head (one hop), or
    // for the heads this rank owns only (two hops, C x G > 8)
    const uint32_t owned_max = (uint32_t)((G + C - 1) / C);
    hist_all = o; o += (C * G > 8 || P > 1 ? owned_max * C : (uint32_t)C * G) * kHistBins * 2;
    sel = o;   o = align(o + (uint32_t)G * selcap * 4, 16);
    inbox = o; o += owned_max * C * kPartStride * 4;  // partials of the heads this rank merges
    wpart = o; o += kConsumerWarps * kPartStride * 4;
    qf = o;    o += (uint32_t)G * kHeadDim * 4;  // the G query heads as fp32
    o = align(o, 32);
    qcode = o; o += (uint32_t)(G + 1) * 32;
    sq = o;    o += (uint32_t)(G + 1) * kHeadDim * 8;
    bars = o;  o += (2 * kMaxStages + 3) * 8;  // full[], empty[], hist / partial / threshold exchange
    total = o;
  }
};

// Exclusive prefix of (a, b) over the consumer threads of one q-head
// (warps [g * WG, (g + 1) * WG), thread order), plus the head totals.
// scratch: 2 * kConsumerWarps ints. Contains one consumer_sync; the caller
// syncs again before scratch is reused.
template <int G>
__device__ __forceinline__ void head_scan2(int a, int b, int& ea, int& eb, int& ta, int& tb, int* scratch) {
  constexpr int WG = kConsumerWarps / G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int ia = a, ib = b;
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    const int oa = __shfl_up_sync(kFull, ia, m), ob = __shfl_up_sync(kFull, ib, m);
    if (lane >= m) { ia += oa; ib += ob; }
  }
  if (lane == 31) { scratch[warp] = ia; scratch[kConsumerWarps + warp] = ib; }
  consumer_sync();
  // cross-warp prefix: lane l < WG holds warp (w0 + l)'s total; a short warp scan
  const int w0 = (warp / WG) * WG;
  int xa = lane < WG ? scratch[w0 + lane] : 0, xb = lane < WG ? scratch[kConsumerWarps + w0 + lane] : 0;
#pragma unroll
  for (int m = 1; m < WG; m <<= 1) {
    const int oa = __shfl_up_sync(kFull, xa, m), ob = __shfl_up_sync(kFull, xb, m);
    if (lane >= m) { xa += oa; xb += ob; }
  }
  const int wi = warp - w0;
  const int pa = __shfl_sync(kFull, xa, (wi + 31) & 31), pb = __shfl_sync(kFull, xb, (wi + 31) & 31);
  ea = (wi > 0 ? pa : 0) + ia - a;
  eb = (wi > 0 ? pb : 0) + ib - b;
  ta = __shfl_sync(kFull, xa, WG - 1);
  tb = __shfl_sync(kFull, xb, WG - 1);
}

// Masks (bit i = token i of a 32-token group) of distances < thr and == thr,
// from 32 u16 distances in shared memory: SWAR on u16 pairs, (K - x) & 0x8000
// per half is set exactly where x <= K (distances < 2^15).
__device__ __forceinline__ void group_masks(const uint16_t* d32, int thr, int valid, uint32_t& ltm, uint32_t& eqm) {
  const uint32_t kle = ((uint32_t)thr * 0x00010001u) | 0x80008000u;
  const uint32_t klt = thr > 0 ? (((uint32_t)(thr - 1) * 0x00010001u) | 0x80008000u) : 0u;
  const uint4* src = reinterpret_cast<const uint4*>(d32);
  uint32_t le = 0, lt = 0;
#pragma unroll
  for (int q4 = 0; q4 < 4; ++q4) {
    const uint4 v4 = src[q4];
    const uint32_t w[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = (q4 * 4 + e) * 2;
      const uint32_t a = (kle - w[e]) & 0x80008000u;
      const uint32_t b = thr > 0 ? ((klt - w[e]) & 0x80008000u) : 0u;
      le |= ((a >> 15) & 1u) << i | (a >> 31) << (i + 1);
      lt |= ((b >> 15) & 1u) << i | (b >> 31) << (i + 1);
    }
  }
  const uint32_t vm = valid >= 32 ? 0xffffffffu : (valid <= 0 ? 0u : ((1u << valid) - 1u));
  ltm = lt & vm;
  eqm = (le & ~lt) & vm;
}

// 8-token masks (bit e = token e of a 16-B chunk of u16 distances) of
// distances <= thr and < thr, same SWAR as group_masks.
__device__ __forceinline__ void chunk_masks(const uint4 v4, int thr, uint32_t& le, uint32_t& lt) {
  const uint32_t kle = ((uint32_t)thr * 0x00010001u) | 0x80008000u;
  const uint32_t klt = thr > 0 ? (((uint32_t)(thr - 1) * 0x00010001u) | 0x80008000u) : 0u;
  const uint32_t w[4] = {v4.x, v4.y, v4.z, v4.w};
  le = 0u;
  lt = 0u;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t a = (kle - w[e]) & 0x80008000u;
    const uint32_t b = thr > 0 ? ((klt - w[e]) & 0x80008000u) : 0u;
    le |= ((a >> 15) & 1u) << (2 * e) | (a >> 31) << (2 * e + 1);
    lt |= ((b >> 15) & 1u) << (2 * e) | (b >> 31) << (2 * e + 1);
  }
}

// The same two masks in "collected" order, 2 instructions per word cheaper:
// token 2e (low half of word e) at bit e, token 2e + 1 at bit 16 + e. The
// count pass only needs popcounts, which do not care about the order; the
// (rare) emitting threads restore index order with collected_to_index.
__device__ __forceinline__ void chunk_masks_c(const uint4 v4, int thr, uint32_t& le, uint32_t& lt) {
  const uint32_t kle = ((uint32_t)thr * 0x00010001u) | 0x80008000u;
  const uint32_t klt = thr > 0 ? (((uint32_t)(thr - 1) * 0x00010001u) | 0x80008000u) : 0u;
  const uint32_t w[4] = {v4.x, v4.y, v4.z, v4.w};
  le = 0u;
  lt = 0u;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    le |= ((kle - w[e]) & 0x80008000u) >> (15 - e);
    lt |= thr > 0 ? ((klt - w[e]) & 0x80008000u) >> (15 - e) : 0u;
  }
}
// Bit spread (Morton): bit b of a 16-bit value -> bit 2 b.
__device__ __forceinline__ uint32_t spread16(uint32_t x) {
  x = (x | (x << 8)) & 0x00ff00ffu;
  x = (x | (x << 4)) & 0x0f0f0f0fu;
  x = (x | (x << 2)) & 0x33333333u;
  return (x | (x << 1)) & 0x55555555u;
}
// A 32-token span word in collected order (chunk c = 8 tokens at nibble c of
// each half) -> index order: token 8 c + 2 e + o sits at bit 16 o + 4 c + e,
// so the index-order word is the Morton interleave of the two halves.
__device__ __forceinline__ uint32_t collected_to_index(uint32_t m) {
  return spread16(m & 0xffffu) | (spread16(m >> 16) << 1);
}
// Valid-token mask (the first v tokens of a span word) in collected order.
__device__ __forceinline__ uint32_t collected_valid(int v) {
  if (v >= 32) return 0xffffffffu;
  if (v <= 0) return 0u;
  const int full = v >> 3, rem = v & 7;
  const uint32_t lo = ((1u << (4 * full)) - 1u) | (((1u << ((rem + 1) >> 1)) - 1u) << (4 * full));
  const uint32_t hi = ((1u << (4 * full)) - 1u) | (((1u << (rem >> 1)) - 1u) << (4 * full));
  return lo | (hi << 16);
}

// encode128 (certified fp32, exact fp64 fallback) with the code stored to
// *dst by lane 0; exact = true forces the fp64 path. (The fallback stays
// inline: as a noinline call it cost 0.45 µs per layer at config 1.)
__device__ __forceinline__ bool encode128_to(const float in[4], double* sq, Code* dst, bool exact) {
  Code c;
  if (!exact) {
    const int r = encode128_warp_f32(in, c);
    if (r == 1) {
      if ((threadIdx.x & 31) == 0) *dst = c;
      return true;
    }
  }
  const bool ok = encode128_warp(in, sq, c, !exact);
  if ((threadIdx.x & 31) == 0) *dst = c;
  return ok;
}

// SW: compaction form, fixed per launch from the rank length: 2 or 4 = spans
// of up to 64 or 128 tokens per thread with that many mask words (4 costs
// registers, so only where needed), 0 = 32-token groups per thread for ranks
// longer than that. Each instance carries one form only (measured: 1.6 %
// faster than choosing at run time).
// MODE 1 (FULL): the two-hop histogram exchange (C x G > 8), multi-cluster units
// (P > 1) and candidates mode are compiled in; the common one-hop decode
// launches an instance without them (measured 3.6-4.8 % faster at configs
// 1-3: fewer registers, 71 KB instead of 125 KB of code).
// CT: the cluster size when fixed at compile time (the common C = 4 decode
// launch; measured 3 % faster), 0 = from the launch parameters.
// COLL: span masks in collected order (chunk_masks_c) — for spans of 32 or
// more tokens per thread (measured: config 2 16.54 -> 16.07 us, config 3
// 3.97 -> 3.84; at 16-token spans the index-order masks stay faster, config 1
// 9.88 vs 9.97).
template <typename T, int G, int SW, int MODE, int CT, bool COLL = false>
__global__ void __launch_bounds__(kFusedThreads, kCtasPerSm) fused_decode_kernel(const __grid_constant__ FusedParams p) {
  constexpr bool FULL = MODE == 1;  // two-hop exchange, multi-cluster units and candidates mode compiled in
  constexpr bool CAND = MODE != 0;  // candidates mode compiled in (MODE 2: with the lean one-hop exchange only)
  static_assert(G >= 1 && G <= kMaxG && (kConsumerWarps % G) == 0, "G must divide the warp count");
  constexpr int WG = kConsumerWarps / G;  // consumer warps per q-head
  constexpr int NT = kConsumers / G;      // consumer threads per q-head
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ int scratch[2 * kConsumerWarps];
  __shared__ __align__(16) int sc[kMaxG][4];  // per q-head: T, below, pre_lt, pre_eq
  __shared__ int owner_sc[2];                  // two-hop exchange, owner side: T, below
  __shared__ int rank_cnt[16][2];              // two-hop exchange, owner side: per rank (< T, == T)
  __shared__ int cl_cnt[2];                    // multi-cluster unit: earlier clusters' (< T, == T)
  __shared__ int nsel[kMaxG];
  const int C = CT > 0 ? CT : p.C;
  const int rank = (int)cluster_rank();
  const int P = FULL ? p.P : 1;
  // diagnostics (phase stamps, timing-only switches) exist only in ADAMAS_DIAG builds
  const int pdbg = ADAMAS_DIAG ? p.dbg : 0;
  unsigned long long* const ptrace = ADAMAS_DIAG ? p.trace : nullptr;
  uint32_t* const pcand = CAND ? p.cand : nullptr;  // candidates mode (sequence sharding)
  const int pc = (blockIdx.x / C) % P;  // this cluster's token range within the unit
  const int gr = pc * C + rank;          // rank over the unit's P * C CTAs
  const int unit = blockIdx.x / (C * P);
  const int part = unit % p.qsplit;  // which G of the kv-head's qsplit * G q-heads
  const int si = (unit / p.qsplit) / p.n_kv, hk = (unit / p.qsplit) % p.n_kv;
  const int n_q = p.n_kv * G * p.qsplit;
  const int q0 = (hk * p.qsplit + part) * G;  // first q-head of this unit
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  const int64_t cap = p.seq[si].cap;
  const int64_t s_old = p.seq[si].s_old;
  const int64_t S = s_old + (p.append ? 1 : 0);
  const int64_t start = (int64_t)gr * p.chunk;
  const int64_t end = min(S, start + (int64_t)p.chunk);
  const int len = end > start ? (int)(end - start) : 0;
  const int mem_len = (int)max((int64_t)0, min(end, s_old) - start);  // already in HBM
  const bool has_new = p.append && (s_old >= start) && (s_old < end);
  const int selcap = min(p.budget, p.chunk);
  const int ring = p.stages;

  const FusedSmem L(G, C, p.chunk, selcap, ring, p.P);
  uint4* stage = reinterpret_cast<uint4*>(smem + L.stage);
  uint16_t* dist = reinterpret_cast<uint16_t*>(smem + L.dist);
  int* hist = reinterpret_cast<int*>(smem + L.hist);
  uint16_t* hist_all = reinterpret_cast<uint16_t*>(smem + L.hist_all);
  int* sel = reinterpret_cast<int*>(smem + L.sel);
  float* inbox = reinterpret_cast<float*>(smem + L.inbox);
  float* wpart = reinterpret_cast<float*>(smem + L.wpart);
  float* qfs = reinterpret_cast<float*>(smem + L.qf);
  Code* qcode = reinterpret_cast<Code*>(smem + L.qcode);
  double* sqs = reinterpret_cast<double*>(smem + L.sq);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty_bar = full_bar + kMaxStages;
  uint64_t* hist_bar = full_bar + 2 * kMaxStages;
  uint64_t* inbox_bar = hist_bar + 1;
  uint64_t* sc_bar = hist_bar + 2;
  const bool two_hop = FULL && (C * G > 8 || P > 1);  // histogram exchange topology (see the select phase)
  const int xunit = hk * p.qsplit + part;     // this cache's unit index (global scratch)
  const int owners = min(C, G);               // ranks of a cluster that own a head
  int n_owned = 0;  // q-heads whose final merge this rank performs
  for (int g = rank; g < G; g += C) ++n_owned;

  uint4* planes = p.seq[si].codes + (int64_t)hk * 2 * cap;  // lo plane; x plane = +cap
  const uint4* lo_g = planes + start;
  const uint4* x_g = planes + cap + start;
  const int n_stages = (mem_len + kStageTok - 1) / kStageTok;

  // ---------------------------------------------------------------- prologue
  ADAMAS_TRACE(0);
  // (taken by the producer lane: a globaltimer read stalls the reading warp's fp64 work)
  if (ptrace != nullptr && tid == kConsumers && !(pdbg & 32)) ptrace[blockIdx.x * 16 + 14] = trace_clock(pdbg);
  // Tokens >= clean_local may still be in flight from the preceding kernel
  // (its append): stages reaching them are issued after the PDL wait.
  const int clean_local = (int)max((int64_t)0, min((int64_t)mem_len, p.seq[si].clean - start));
  bool waited = !p.pdl;
  auto issue = [&](int st, int slot) {  // slot = st % ring
    const int ntok = min(kStageTok, mem_len - st * kStageTok);
    if (!waited && st * kStageTok + ntok > clean_local) {
      grid_dependency_wait();
      waited = true;
    }
    const uint32_t bytes = (uint32_t)ntok * 16u;
    uint4* dst = stage + (size_t)slot * (kStageBytes / 16);
    mbar_expect_tx(&full_bar[slot], 2u * bytes);
    bulk_g2s(dst, lo_g + (int64_t)st * kStageTok, bytes, &full_bar[slot]);
    bulk_g2s(dst + kStageTok, x_g + (int64_t)st * kStageTok, bytes, &full_bar[slot]);
  };
  if (warp == kProducerWarp && lane == 0) {  // the code stream starts before anything else
    for (int s = 0; s < ring; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kConsumerWarps);
    }
    mbar_init(hist_bar, 1);
    mbar_init(inbox_bar, 1);
    mbar_init(sc_bar, 1);
    mbar_fence_init();
    for (int st = 0; st < min(ring, n_stages); ++st) issue(st, st);
    // bytes this CTA will receive over DSMEM: every rank's u16 histograms, and
    // C partials per q-head it merges
    // (a single-CTA unit exchanges through its own shared memory: plain stores
    // and the consumer barrier, no st.async, which needs a cluster of >= 2)
    if (C > 1 && !two_hop) mbar_expect_tx(hist_bar, (uint32_t)(C * G * kHistBins * 2));
    else if (C > 1 && n_owned) mbar_expect_tx(hist_bar, (uint32_t)(n_owned * C * kHistBins * 2));
    if (two_hop) mbar_expect_tx(sc_bar, (uint32_t)(G * 16));
    if (C > 1 && n_owned && !pcand) mbar_expect_tx(inbox_bar, (uint32_t)(n_owned * C * kPartStride * 4));
  }
  // the G query heads (and the new key) are loaded before the barrier so the
  // global-load latency overlaps the barrier initialisation
  float f[4] = {0.f, 0.f, 0.f, 0.f};
  typename Raw4<T>::V kr{}, vr{};
  if (p.pdl && warp <= G) {
#if ADAMAS_QPF
    // warm L2 with this unit's q / k_new / v_new lines while the predecessor
    // runs: the reads after the wait then hit L2 (a prefetch of a line the
    // predecessor is still writing is harmless, L2 is the coherence point)
    if (lane < 2) {
      if (warp < G)
        prefetch_l2(reinterpret_cast<const char*>(reinterpret_cast<const T*>(p.q) + ((int64_t)si * n_q + q0 + warp) * kHeadDim) + lane * 128);
      else if (has_new) {
        const int64_t vrow = (int64_t)si * p.n_kv + hk;
        prefetch_l2(reinterpret_cast<const char*>(reinterpret_cast<const T*>(p.k_new) + vrow * kHeadDim) + lane * 128);
        prefetch_l2(reinterpret_cast<const char*>(reinterpret_cast<const T*>(p.v_new) + vrow * kHeadDim) + lane * 128);
      }
    }
#endif
    // q, k_new, v_new and the cache tail come from preceding kernels. Once the
    // predecessor has completed, the next launch may start its prologue.
    grid_dependency_wait();
    if (tid == 0) grid_launch_dependents();
  }
  if (warp < G) {
    const T* qp = reinterpret_cast<const T*>(p.q) + ((int64_t)si * n_q + q0 + warp) * kHeadDim;
    Raw4<T>::to_float(Raw4<T>::load(qp + lane * 4), f);
  } else if (has_new && warp == G) {
    const int64_t vrow = (int64_t)si * p.n_kv + hk;
    kr = Raw4<T>::load(reinterpret_cast<const T*>(p.k_new) + vrow * kHeadDim + lane * 4);
    vr = Raw4<T>::load(reinterpret_cast<const T*>(p.v_new) + vrow * kHeadDim + lane * 4);
  }
  for (int i = tid; i < G * kHistBins; i += kFusedThreads) hist[i] = 0;
  __syncthreads();           // mbarrier inits visible to the whole CTA
  cluster_arrive_relaxed();  // "my mbarriers are initialized"; waited on before the first DSMEM store
  ADAMAS_TRACE(1);

  if (warp == kProducerWarp) {  // keep the ring full: refill a slot once all consumer warps released it
    if (lane == 0) {
      if (pdbg & 4) __nanosleep(8000);  // diagnostics: keep the producer off the SMSP during the prologue
      int slot = 0;
      uint32_t phase = 0u;  // of the slot's previous use: ((st / ring) - 1) & 1
      for (int st = ring; st < n_stages; ++st) {
        mbar_wait_backoff(&empty_bar[slot], phase);
        // the consumers' generic-proxy reads of the slot (released through
        // the empty barrier) are ordered before the bulk copy's async-proxy
        // writes that refill it
        fence_proxy_async_shared();
        issue(st, slot);
        if (++slot == ring) {
          slot = 0;
          phase ^= 1u;
        }
      }
    }
    return;
  }

  // One encoder call site for the query heads (warps 0..G-1) and the appended
  // key (warp G): half the inline encoder code (fp32 route + exact fp64 path;
  // measured 9.98 -> 9.91 us at config 1, profiles/r02h_ab_one_encode.txt).
  if (warp < G || (has_new && warp == G)) {
    const bool is_key = warp == G;
    float e[4];
    if (is_key) {  // append (kv_cache.cpp:62-71); part 0 of a split kv-head writes
      const int64_t row = (int64_t)hk * cap + s_old;
      if (part == 0) {
        Raw4<T>::store(reinterpret_cast<T*>(p.seq[si].K) + row * kHeadDim + lane * 4, kr);
        Raw4<T>::store(reinterpret_cast<T*>(p.seq[si].V) + row * kHeadDim + lane * 4, vr);
      }
      Raw4<T>::to_float(kr, e);
    } else {  // query head hk * G + warp (sweep.cpp:92-94)
      *reinterpret_cast<float4*>(qfs + warp * kHeadDim + lane * 4) = make_float4(f[0], f[1], f[2], f[3]);
#pragma unroll
      for (int i = 0; i < 4; ++i) e[i] = f[i];
    }
    if (!encode128_to(e, sqs + warp * kHeadDim, qcode + warp, p.exact_encode != 0) && lane == 0)
      atomicOr(p.seq[si].status, kStatusDegenerate);
    if (is_key && lane == 0 && part == 0) store_code(planes, cap, s_old, qcode[G]);  // written by this lane
  }
  consumer_sync();
  QCode qc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) qc[g] = make_qcode(qcode[g]);

  // Compaction geometry, fixed before the scan because it sets the distance
  // layout: thread t of a head owns a span of 16 << sh tokens (the smallest
  // that covers the rank with the head's NT threads, up to 128), and the
  // 16-B chunks of span s are stored XOR-swizzled by swz(s), so the 8 threads
  // of a shared-memory wavefront reading chunk j of their spans hit 8
  // distinct bank groups. Longer ranks keep the plain layout (32-token groups).
  const int span_groups = (len + 31) >> 5;
  int sh = 0;
  while ((2 << sh) < 4 * SW && (NT << (4 + sh)) < span_groups * 32) ++sh;
  constexpr bool span = SW > 0;  // the launcher picks SW so that spans cover the rank
  const int nch = 2 << sh;  // 16-B chunks (8 tokens) per span
  auto swz = [&](int sp) { return nch >= 8 ? (sp & 7) : ((sp * nch) >> 3) & (nch - 1); };
  // shared-memory slot of local token x in a head's distance row; for
  // x = base + j (base a multiple of 1024) it is base + dslot(j)
  auto dslot = [&](int x) { return span ? x ^ (swz(x >> (4 + sh)) << 3) : x; };
  int jslot[kTokPerThread];
#pragma unroll
  for (int u = 0; u < kTokPerThread; ++u) jslot[u] = dslot(tid + u * kConsumers);

  // ---------------------------------------------------------------- scan
  ADAMAS_TRACE(2);
  int slot = 0;
  uint32_t phase = 0u;  // slot = st % ring, phase = (st / ring) & 1, kept incrementally
  for (int st = 0; st < n_stages; ++st) {
    mbar_wait(&full_bar[slot], phase);
    const uint4* slo = stage + (size_t)slot * (kStageBytes / 16);
    const uint4* sx = slo + kStageTok;
    const int base = st * kStageTok;
    const int ntok = min(kStageTok, mem_len - base);
    uint4 a[kTokPerThread], b[kTokPerThread];
#pragma unroll
    for (int u = 0; u < kTokPerThread; ++u) {
      const int j = tid + u * kConsumers;
      if (j < ntok) { a[u] = slo[j]; b[u] = sx[j]; }
    }
    uint32_t d[kTokPerThread][G];
#pragma unroll
    for (int u = 0; u < kTokPerThread; ++u) {
      const uint32_t lo[4] = {a[u].x, a[u].y, a[u].z, a[u].w}, x[4] = {b[u].x, b[u].y, b[u].z, b[u].w};
#pragma unroll
      for (int g = 0; g < G; ++g) d[u][g] = l1_distance<G >= 2 ? 7 : 6>(qc[g], lo, x);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[slot]);  // this warp is done reading the slot
#pragma unroll
    for (int u = 0; u < kTokPerThread; ++u) {
      const int j = tid + u * kConsumers;
      if (j < ntok) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          dist[g * p.chunk + base + jslot[u]] = (uint16_t)d[u][g];
          atomicAdd(&hist[g * kHistBins + d[u][g]], 1);
        }
      }
    }
    if (++slot == ring) {
      slot = 0;
      phase ^= 1u;
    }
  }
  if (has_new && tid < G) {  // the appended token is a candidate
    const Code nc = qcode[G];
    uint32_t nx[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) nx[w] = nc.lo[w] ^ nc.hi[w];
    const uint32_t d = l1_distance(make_qcode(qcode[tid]), nc.lo, nx);
    dist[tid * p.chunk + dslot((int)(s_old - start))] = (uint16_t)d;
    atomicAdd(&hist[tid * kHistBins + d], 1);
  }
  consumer_sync();  // local histogram final
  ADAMAS_TRACE(3);
  if (ADAMAS_DIAG && (pdbg & (1 << 16))) return;  // diagnostics (timing only): stop after the scan
  const int k_eff = (int)min((int64_t)p.budget, S);
  const int g_me = tid / NT, t_in = tid % NT;
  cluster_wait();
  if (!two_hop) {
    // One hop: every rank's histograms (u16: counts <= chunk < 2^16) go to
    // every rank (st.async; each receiver's mbarrier counts bytes); each rank
    // then derives, per head, T, the count below T and its own offsets.
    if (tid < G * (kHistBins / 8)) {
      const int g = tid / (kHistBins / 8), b0 = (tid % (kHistBins / 8)) * 8;
      const int4 h0 = *reinterpret_cast<const int4*>(hist + g * kHistBins + b0);
      const int4 h1 = *reinterpret_cast<const int4*>(hist + g * kHistBins + b0 + 4);
      const uint32_t w0 = (uint32_t)h0.x | ((uint32_t)h0.y << 16), w1 = (uint32_t)h0.z | ((uint32_t)h0.w << 16);
      const uint32_t w2 = (uint32_t)h1.x | ((uint32_t)h1.y << 16), w3 = (uint32_t)h1.z | ((uint32_t)h1.w << 16);
      const uint32_t local = smem_addr(hist_all + ((size_t)rank * G + g) * kHistBins + b0);
      for (int r = 0; r < C; ++r)
        if (C == 1) st_shared_v4(local, w0, w1, w2, w3);
        else st_async_v4(mapa_shared(local, r), w0, w1, w2, w3, mapa_shared(smem_addr(hist_bar), r));
    }
    if (C == 1) consumer_sync();
    else mbar_wait(hist_bar, 0);
    ADAMAS_TRACE(4);

    // Head g's T = smallest distance whose cumulative count over all ranks
    // reaches k. NT threads per head, G consecutive bins each; a head-segmented
    // block prefix orders the threads; the owning thread walks its bins.
    const int b0 = t_in * G;
    int tot[G], pre[G];
#pragma unroll
    for (int i = 0; i < G; ++i) { tot[i] = 0; pre[i] = 0; }
    for (int r = 0; r < C; ++r) {
      const uint16_t* h = hist_all + ((size_t)r * G + g_me) * kHistBins + b0;
#pragma unroll
      for (int i = 0; i < G; ++i) {
        const int v = h[i];
        tot[i] += v;
        pre[i] += r < rank ? v : 0;
      }
    }
    int st = 0, sp = 0;
#pragma unroll
    for (int i = 0; i < G; ++i) { st += tot[i]; sp += pre[i]; }
    int c, cp, unused0, unused1;
    head_scan2<G>(st, sp, c, cp, unused0, unused1, scratch);
    if (c < k_eff && c + st >= k_eff) {
#pragma unroll
      for (int i = 0; i < G; ++i) {
        if (c < k_eff && c + tot[i] >= k_eff) {
          sc[g_me][0] = b0 + i;  // T
          sc[g_me][1] = c;       // count of distances < T over the whole head
          sc[g_me][2] = cp;      // count of distances < T in ranks before this one
          sc[g_me][3] = pre[i];  // count of distances == T in ranks before this one
        }
        c += tot[i];
        cp += pre[i];
      }
    }
  } else {
    // Two hops (large C x G): head g's histograms go to its owner rank g % C
    // only; the owner derives T and every rank's offsets and pushes each rank
    // its (T, below, pre_lt, pre_eq).
    if (tid < G * (kHistBins / 8)) {
      const int g = tid / (kHistBins / 8), b0 = (tid % (kHistBins / 8)) * 8;
      const int4 h0 = *reinterpret_cast<const int4*>(hist + g * kHistBins + b0);
      const int4 h1 = *reinterpret_cast<const int4*>(hist + g * kHistBins + b0 + 4);
      const uint32_t w0 = (uint32_t)h0.x | ((uint32_t)h0.y << 16), w1 = (uint32_t)h0.z | ((uint32_t)h0.w << 16);
      const uint32_t w2 = (uint32_t)h1.x | ((uint32_t)h1.y << 16), w3 = (uint32_t)h1.z | ((uint32_t)h1.w << 16);
      const uint32_t owner = (uint32_t)(g % C), slot = (uint32_t)(g / C);
      const uint32_t local = smem_addr(hist_all + ((size_t)slot * C + rank) * kHistBins + b0);
      st_async_v4(mapa_shared(local, owner), w0, w1, w2, w3, mapa_shared(smem_addr(hist_bar), owner));
    }
    if (n_owned) mbar_wait(hist_bar, 0);
    ADAMAS_TRACE(4);
    if (P > 1 && n_owned) {
      // Multi-cluster unit: publish this cluster's combined histogram of each
      // owned head, then one arrival per owner CTA on the unit's barrier.
      for (int j = 0; j < n_owned; ++j) {
        const int g = rank + j * C;
        const uint16_t* hs = hist_all + (size_t)j * C * kHistBins;
        uint32_t* dst = p.seq[si].xhist + (((size_t)xunit * P + pc) * G + g) * kHistBins;
        for (int b = tid; b < kHistBins; b += kConsumers) {
          uint32_t t = 0;
          for (int r = 0; r < C; ++r) t += hs[(size_t)r * kHistBins + b];
          __stcg(dst + b, t);
        }
      }
      consumer_sync();
      if (tid == 0) unit_barrier(p.seq[si].xsync + xunit * 4, P * owners, true, p.seq[si].status);
      consumer_sync();
    }
    for (int j = 0; j < n_owned; ++j) {  // uniform within the CTA
      const int g = rank + j * C;
      const uint16_t* hs = hist_all + (size_t)j * C * kHistBins;
      const uint32_t* xh = p.seq[si].xhist + ((size_t)xunit * P * G + g) * kHistBins;  // + pc' * G * bins
      const int b = tid;  // one bin per consumer thread (kConsumers >= kHistBins)
      int tot = 0, pre = 0;  // all ranks of the unit / clusters before this one (P > 1)
      if (b < kHistBins) {
        if (P > 1) {
          for (int c2 = 0; c2 < P; ++c2) {
            const int v = (int)__ldcg(xh + (size_t)c2 * G * kHistBins + b);
            tot += v;
            pre += c2 < pc ? v : 0;
          }
        } else {
          for (int r = 0; r < C; ++r) tot += hs[(size_t)r * kHistBins + b];
        }
      }
      int c, cp, tot_all, unused1;
      head_scan2<1>(tot, pre, c, cp, tot_all, unused1, scratch);
      if (b < kHistBins && c < k_eff && c + tot >= k_eff) {
        owner_sc[0] = b;  // T
        owner_sc[1] = c;  // below T over the unit
        cl_cnt[0] = cp;   // below T in earlier clusters
        cl_cnt[1] = pre;  // == T in earlier clusters
      }
      consumer_sync();
      const int T = owner_sc[0];
      if (warp < C) {  // warp r: rank r's count below T and at T
        int lt = 0;
        for (int bb = lane; bb < T; bb += 32) lt += hs[(size_t)warp * kHistBins + bb];
        lt = warp_sum_int(lt);
        if (lane == 0) { rank_cnt[warp][0] = lt; rank_cnt[warp][1] = hs[(size_t)warp * kHistBins + T]; }
      }
      consumer_sync();
      if (tid < C) {  // push (T, below, pre_lt, pre_eq) into rank tid's sc[g]
        int pl = P > 1 ? cl_cnt[0] : 0, pe = P > 1 ? cl_cnt[1] : 0;
        for (int r = 0; r < tid; ++r) { pl += rank_cnt[r][0]; pe += rank_cnt[r][1]; }
        st_async_v4(mapa_shared(smem_addr(&sc[g][0]), (uint32_t)tid), (uint32_t)T, (uint32_t)owner_sc[1], (uint32_t)pl,
                    (uint32_t)pe, mapa_shared(smem_addr(sc_bar), (uint32_t)tid));
      }
      consumer_sync();
    }
    mbar_wait(sc_bar, 0);
  }
  consumer_sync();
  ADAMAS_TRACE(5);
  if (ADAMAS_DIAG && (pdbg & (1 << 17))) return;  // diagnostics (timing only): stop once T is known

  // ---------------------------------------------------------------- compaction
  // Thread t_in of head g owns a contiguous span of tokens: count (< T, == T)
  // -> head-segmented prefix in index order -> emit. Spans (16..128 tokens,
  // swizzled distance layout, see before the scan) keep their masks in
  // registers between the two passes; longer ranks take 32-token groups per
  // thread and recompute the masks.
  {
    const int g = g_me;
    const int ngroups = (len + 31) >> 5;
    const int gpt = (ngroups + NT - 1) / NT;
    const int grp0 = min(ngroups, t_in * gpt), grp1 = min(ngroups, grp0 + gpt);
    const int thr = sc[g][0], below = sc[g][1], pre_lt = sc[g][2], pre_eq = sc[g][3];
    const int need = k_eff - below;               // ties at T the whole head takes
    const int eq_budget = max(0, need - pre_eq);  // ... of which this rank may take
    const int out_off = pre_lt + min(pre_eq, need);
    const uint16_t* dg = dist + g * p.chunk;
    const T* Kg = reinterpret_cast<const T*>(p.seq[si].K) + ((int64_t)hk * cap + start) * kHeadDim;
    const T* Vg = reinterpret_cast<const T*>(p.seq[si].V) + ((int64_t)hk * cap + start) * kHeadDim;
    const int tok0 = t_in << (4 + sh);
    constexpr int NW = SW > 0 ? SW : 1;
    uint32_t sl[NW], se[NW];  // span masks: bit i of word w = token tok0 + 32 w + i
#pragma unroll
    for (int w = 0; w < NW; ++w) sl[w] = se[w] = 0u;
    // warm L2 for the gather, one prefetch per 128-B line: each survivor as
    // the emit places it (default), or every row at distance <= T in the
    // count pass (ADAMAS_GATHER_PREFETCH = 1)
    auto prefetch_row = [&](int t) {
      const char* kp = reinterpret_cast<const char*>(Kg + (int64_t)t * kHeadDim);
      const char* vp = reinterpret_cast<const char*>(Vg + (int64_t)t * kHeadDim);
#pragma unroll
      for (int c = 0; c < (int)(kHeadDim * sizeof(T)); c += 128) {
        prefetch_l2(kp + c);
        prefetch_l2(vp + c);
      }
    };
    int my_lt = 0, my_eq = 0;
    if (span) {
      if (tok0 < len) {
        const int z = swz(t_in);  // this span's chunk swizzle
        const uint4* src = reinterpret_cast<const uint4*>(dg + tok0);
#pragma unroll
        for (int j = 0; j < 4 * SW; ++j) {
          if (j < nch) {
            uint32_t le8, lt8;
            if constexpr (COLL) {
              chunk_masks_c(src[j ^ z], thr, le8, lt8);
              sl[j >> 2] |= lt8 << ((j & 3) * 4);
              se[j >> 2] |= (le8 & ~lt8) << ((j & 3) * 4);
            } else {
              chunk_masks(src[j ^ z], thr, le8, lt8);
              sl[j >> 2] |= lt8 << ((j & 3) * 8);
              se[j >> 2] |= (le8 & ~lt8) << ((j & 3) * 8);
            }
          }
        }
        const int v = len - tok0;  // valid tokens in the span (>= 1)
#pragma unroll
        for (int w = 0; w < SW; ++w) {
          const int vw = v - 32 * w;
          const uint32_t vm = COLL ? collected_valid(vw) : (vw >= 32 ? 0xffffffffu : (vw <= 0 ? 0u : (1u << vw) - 1u));
          sl[w] &= vm;
          se[w] &= vm;
        }
      }
#pragma unroll
      for (int w = 0; w < SW; ++w) {
        my_lt += __popc(sl[w]);
        my_eq += __popc(se[w]);
      }
#pragma unroll
      for (int w = 0; w < SW; ++w)
        for (uint32_t m = ADAMAS_GATHER_PREFETCH == 1 ? (sl[w] | se[w]) : 0u; m; m &= m - 1)
          prefetch_row(tok0 + 32 * w + __ffs(COLL ? collected_to_index(m & (0u - m)) : m) - 1);
    } else {
      for (int grp = grp0; grp < grp1; ++grp) {
        uint32_t ltm, eqm;
        group_masks(dg + grp * 32, thr, len - grp * 32, ltm, eqm);
        my_lt += __popc(ltm);
        my_eq += __popc(eqm);
        for (uint32_t m = ADAMAS_GATHER_PREFETCH == 1 ? (ltm | eqm) : 0u; m; m &= m - 1)
          prefetch_row(grp * 32 + __ffs(m) - 1);
      }
    }
    ADAMAS_TRACE(12);
    int lt_before, eq_before, lt_tot, eq_tot;
    head_scan2<G>(my_lt, my_eq, lt_before, eq_before, lt_tot, eq_tot, scratch);
    if (t_in == 0) nsel[g] = min(lt_tot + min(eq_tot, eq_budget), selcap);
    ADAMAS_TRACE(6);
    if (my_lt > 0 || (my_eq > 0 && eq_before < eq_budget)) {
      int32_t* idx_row = (p.idx && !(pdbg & 2))
                             ? p.idx + ((int64_t)si * n_q + q0 + g) * p.budget + out_off
                             : nullptr;
      int pos = lt_before + min(eq_before, eq_budget);
      int eq_seen = eq_before;
      // local token t (in index order) at distance <= T: take it unless it is
      // a tie beyond the budget
      auto emit = [&](int t, bool is_eq) {
        if (is_eq && eq_seen++ >= eq_budget) return;  // ties beyond the budget are not taken
        const int tok = (int)start + t;
        if (ADAMAS_GATHER_PREFETCH == 2 && !pcand) prefetch_row(t);
        if (pos < selcap) sel[g * selcap + pos] = tok;
        if (idx_row) idx_row[pos] = tok;
        if (pcand) {  // (distance, global index) key: the distributed top-k's order
          const int64_t off = ((int64_t)si * n_q + q0 + g) * p.budget + out_off + pos;
          const uint32_t key = ((uint32_t)dg[dslot(t)] << 23) | (uint32_t)(p.cand_base + tok);
          if (p.peers.n) {
            for (int r = 0; r < p.peers.n; ++r) p.peers.keys[r][off] = key;  // NVLink stores
          } else {
            pcand[off] = key;
          }
        }
        ++pos;
      };
      if (span) {
#pragma unroll
        for (int w = 0; w < SW; ++w) {
          const uint32_t ml = COLL ? collected_to_index(sl[w]) : sl[w];  // index order
          const uint32_t me = COLL ? collected_to_index(se[w]) : se[w];
          for (uint32_t m = ml | me; m; m &= m - 1) {
            const int i = __ffs(m) - 1;
            emit(tok0 + 32 * w + i, (me >> i) & 1u);
          }
        }
      } else {
        for (int grp = grp0; grp < grp1; ++grp) {
          uint32_t ltm, eqm;
          group_masks(dg + grp * 32, thr, len - grp * 32, ltm, eqm);
          for (uint32_t m = ltm | eqm; m; m &= m - 1) {
            const int i = __ffs(m) - 1;
            emit(grp * 32 + i, (eqm >> i) & 1u);
          }
        }
      }
    }
    ADAMAS_TRACE(13);
    if (gr == 0 && p.idx && t_in == 0) {  // estimator.cpp:80 caps the selection at S
      int32_t* row = p.idx + ((int64_t)si * n_q + q0 + g) * p.budget;
      for (int i = k_eff; i < p.budget; ++i) row[i] = -1;
    }
    if (gr == 0 && pcand && t_in == 0) {
      const int64_t row = ((int64_t)si * n_q + q0 + g) * p.budget;
      if (p.peers.n) {
        for (int r = 0; r < p.peers.n; ++r)
          for (int i = k_eff; i < p.budget; ++i) p.peers.keys[r][row + i] = 0xffffffffu;
      } else {
        for (int i = k_eff; i < p.budget; ++i) pcand[row + i] = 0xffffffffu;
      }
    }
  }
  consumer_sync();
  ADAMAS_TRACE(7);
  if (ADAMAS_DIAG && (pdbg & (1 << 19))) return;  // diagnostics (timing only): stop after the compaction
  if (pcand) {  // candidates mode: the selection is the product
    if (p.peers.n && tid == 0) peer_signal(p.peers);
    return;
  }

  // ---------------------------------------------------------------- attend
  {
    const int g = warp % G, sub = warp / G;
    const int ns = (ADAMAS_DIAG && (pdbg & (1 << 18))) ? 0 : nsel[g];  // diagnostics: no gather
    const float4 q4 = *reinterpret_cast<const float4*>(qfs + g * kHeadDim + lane * 4);
    float qf[4] = {q4.x, q4.y, q4.z, q4.w};
    const float scale = 0.088388347648318440f * kLog2e;  // 1/sqrt(128), log2 units
#pragma unroll
    for (int j = 0; j < 4; ++j) qf[j] *= scale;
    const T* Kh = reinterpret_cast<const T*>(p.seq[si].K) + (int64_t)hk * cap * kHeadDim + lane * 4;
    const T* knew_row = reinterpret_cast<const T*>(p.k_new) + ((int64_t)si * p.n_kv + hk) * kHeadDim + lane * 4;
    const T* vnew_row = reinterpret_cast<const T*>(p.v_new) + ((int64_t)si * p.n_kv + hk) * kHeadDim + lane * 4;
    const T* Vh = reinterpret_cast<const T*>(p.seq[si].V) + (int64_t)hk * cap * kHeadDim + lane * 4;
    float m = -INFINITY, l = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
    constexpr int B = 4;  // rows in flight per warp
    for (int r0 = sub; r0 < ns; r0 += WG * B) {
      typename Raw4<T>::V kb[B], vb[B];
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int r = r0 + b * WG;
        if (r < ns) {
          const int64_t t = sel[g * selcap + r];
          if (has_new && t == s_old) {  // the appended row: from the input (another CTA of a split
            kb[b] = Raw4<T>::load(knew_row);  // kv-head may be the one writing it to the cache)
            vb[b] = Raw4<T>::load(vnew_row);
          } else {
            kb[b] = Raw4<T>::load(Kh + t * kHeadDim);
            vb[b] = Raw4<T>::load(Vh + t * kHeadDim);
          }
        } else {
          kb[b] = typename Raw4<T>::V{};
          vb[b] = typename Raw4<T>::V{};
        }
      }
      // B dot products reduced together (the butterflies interleave)
      float sd[B];
#pragma unroll
      for (int b = 0; b < B; ++b) {
        float kf[4];
        Raw4<T>::to_float(kb[b], kf);
        sd[b] = r0 + b * WG < ns ? qf[0] * kf[0] + qf[1] * kf[1] + qf[2] * kf[2] + qf[3] * kf[3] : 0.f;
      }
#pragma unroll
      for (int m2 = 16; m2 > 0; m2 >>= 1)
#pragma unroll
        for (int b = 0; b < B; ++b) sd[b] += __shfl_xor_sync(kFull, sd[b], m2);
      float mx = m;
#pragma unroll
      for (int b = 0; b < B; ++b)
        if (r0 + b * WG < ns) mx = fmaxf(mx, sd[b]);
      const float corr = exp2f(m - mx);
      l *= corr;
#pragma unroll
      for (int j = 0; j < 4; ++j) o[j] *= corr;
#pragma unroll
      for (int b = 0; b < B; ++b) {
        if (r0 + b * WG < ns) {
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
    ADAMAS_TRACE(8);
    float* wp = wpart + warp * kPartStride;
    if (lane == 0) { wp[0] = m; wp[1] = l; }
#pragma unroll
    for (int j = 0; j < 4; ++j) wp[4 + lane * 4 + j] = o[j];
    consumer_sync();
    if (sub == 0) {  // combine this head's WG warp partials, push to the merging rank
      const float* mine = wpart + (lane * G + g) * kPartStride;
      const float ml = lane < WG ? mine[0] : -INFINITY, ll = lane < WG ? mine[1] : 0.f;
      float M = ll > 0.f ? ml : -INFINITY;
#pragma unroll
      for (int m2 = 16; m2 > 0; m2 >>= 1) M = fmaxf(M, __shfl_xor_sync(kFull, M, m2));
      const float cl = ll > 0.f ? exp2f(ml - M) : 0.f;
      const float Lsum = warp_sum(ll * cl);
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int s2 = 0; s2 < WG; ++s2) {
        const float c = __shfl_sync(kFull, cl, s2);
        const float4 v4 = *reinterpret_cast<const float4*>(wpart + (s2 * G + g) * kPartStride + 4 + lane * 4);
        acc[0] += v4.x * c; acc[1] += v4.y * c; acc[2] += v4.z * c; acc[3] += v4.w * c;
      }
      // push (M, L, o[128]) into the merging rank's inbox[rank][g] (528 B)
      const uint32_t local = smem_addr(inbox + ((g / C) * C + rank) * kPartStride);
      const uint32_t dst = mapa_shared(local, (uint32_t)(g % C));
      const uint32_t bar = mapa_shared(smem_addr(inbox_bar), (uint32_t)(g % C));
      if (C == 1) {  // own inbox (no st.async within a one-CTA "cluster")
        if (lane == 0) st_shared_v4(local, __float_as_uint(M), __float_as_uint(Lsum), 0u, 0u);
        st_shared_v4(local + 16 + lane * 16, __float_as_uint(acc[0]), __float_as_uint(acc[1]),
                     __float_as_uint(acc[2]), __float_as_uint(acc[3]));
      } else {
      if (lane == 0) st_async_v4(dst, __float_as_uint(M), __float_as_uint(Lsum), 0u, 0u, bar);
      st_async_v4(dst + 16 + lane * 16, __float_as_uint(acc[0]), __float_as_uint(acc[1]), __float_as_uint(acc[2]),
                  __float_as_uint(acc[3]), bar);
      }
    }
  }
  ADAMAS_TRACE(9);
  if (C == 1) consumer_sync();
  else if (n_owned) mbar_wait(inbox_bar, 0);  // all C partials of the heads this rank merges
  ADAMAS_TRACE(10);

  // ---------------------------------------------------------------- merge
  for (int g = warp; g < G; g += kConsumerWarps) {
    if (g % C != rank) continue;
    float M = -INFINITY;
    for (int r = 0; r < C; ++r) {
      const float* q2 = inbox + ((g / C) * C + r) * kPartStride;
      if (q2[1] > 0.f) M = fmaxf(M, q2[0]);
    }
    float Lsum = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int r = 0; r < C; ++r) {
      const float* q2 = inbox + ((g / C) * C + r) * kPartStride;
      if (!(q2[1] > 0.f)) continue;
      const float c = exp2f(q2[0] - M);
      Lsum += q2[1] * c;
      const float4 v4 = *reinterpret_cast<const float4*>(q2 + 4 + lane * 4);
      acc[0] += v4.x * c; acc[1] += v4.y * c; acc[2] += v4.z * c; acc[3] += v4.w * c;
    }
    if (P > 1) {  // this cluster's partial of head g -> global (merged by cluster 0 below)
      float* xp = p.seq[si].xpart + (((size_t)xunit * P + pc) * G + g) * kPartStride;
      if (lane == 0) { __stcg(xp, Lsum > 0.f ? M : -INFINITY); __stcg(xp + 1, Lsum); }
      __stcg(reinterpret_cast<float4*>(xp + 4 + lane * 4), make_float4(acc[0], acc[1], acc[2], acc[3]));
      continue;
    }
    const float inv = 1.f / Lsum;
    float* op = p.out + ((int64_t)si * n_q + q0 + g) * kHeadDim + lane * 4;
    *reinterpret_cast<float4*>(op) = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
  }
  if (P > 1 && n_owned) {
    consumer_sync();
    if (tid == 0) unit_barrier(p.seq[si].xsync + xunit * 4 + 2, P * owners, pc == 0, p.seq[si].status);
    consumer_sync();
    if (pc == 0) {
      for (int g = warp; g < G; g += kConsumerWarps) {
        if (g % C != rank) continue;
        const float* xp = p.seq[si].xpart + ((size_t)xunit * P * G + g) * kPartStride;
        float M = -INFINITY;
        for (int c2 = 0; c2 < P; ++c2) {
          const float* q2 = xp + (size_t)c2 * G * kPartStride;
          if (__ldcg(q2 + 1) > 0.f) M = fmaxf(M, __ldcg(q2));
        }
        float Lsum = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int c2 = 0; c2 < P; ++c2) {
          const float* q2 = xp + (size_t)c2 * G * kPartStride;
          const float l2 = __ldcg(q2 + 1);
          if (!(l2 > 0.f)) continue;
          const float c = exp2f(__ldcg(q2) - M);
          Lsum += l2 * c;
          const float4 v4 = __ldcg(reinterpret_cast<const float4*>(q2 + 4 + lane * 4));
          acc[0] += v4.x * c; acc[1] += v4.y * c; acc[2] += v4.z * c; acc[3] += v4.w * c;
        }
        const float inv = 1.f / Lsum;
        float* op = p.out + ((int64_t)si * n_q + q0 + g) * kHeadDim + lane * 4;
        *reinterpret_cast<float4*>(op) = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
      }
    }
  }
  ADAMAS_TRACE(11);
  if (ptrace != nullptr && tid == kTraceTid && !(pdbg & 32)) ptrace[blockIdx.x * 16 + 15] = trace_clock(pdbg);
}

}  // namespace adamas_dev
