/*
 * adamas_b200.h — C ABI of the B200-native Adamas decode hot path.
 *
 * This is the drop-in boundary for the reference's operator layer
 * (/root/reference/proj, namespace adamas). The reference binds its hot path
 * per (query, key) pair through the function table kernels::Kernels
 * (include/adamas/kernels.hpp:16-33) called S times per decode; a GPU cannot
 * plug in at that granularity, so this ABI replaces the operator level instead,
 * batched over heads and tokens with one opaque device cache per layer.
 * Every entry point names the reference interface it replaces.
 *
 * Conventions
 *   - Plain C types only. Device pointers are raw CUDA device addresses; the
 *     `stream` argument is a cudaStream_t passed as void* (NULL = legacy stream).
 *   - head_dim is 128 and bits is 2 (the north-star scope); anything else is
 *     rejected with ADAMAS_ERR_CONFIG, never silently mis-computed.
 *   - K/V/q element type: ADAMAS_F32 or ADAMAS_BF16 (fixed per cache).
 *   - Layouts: q [n_q_heads][128]; new keys/values [n_tokens][n_kv_heads][128];
 *     attention output float32 [n_q_heads][128]; indices int32
 *     [n_q_heads][budget] ascending (min(budget, seq_len) valid per head).
 *   - GQA: q-head h reads kv-head h / (n_q_heads / n_kv_heads); every q-head
 *     is encoded, scanned, selected and attended independently, exactly like
 *     independent reference heads.
 *   - Return codes mirror the reference's exception classes:
 *       ADAMAS_ERR_CONFIG  <-> adamas::ConfigError (common.hpp:19-22)
 *       ADAMAS_ERR_RUNTIME <-> std::runtime_error / CUDA failures
 *     adamas_last_error() returns the thread-local message of the last failure.
 *   - Per-vector preconditions the reference checks with exceptions (zero or
 *     non-finite vector, quantizer.cpp:46-47) are detected on the device and
 *     latched into a sticky status word: adamas_cache_status().
 */
#ifndef ADAMAS_B200_H
#define ADAMAS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADAMAS_OK 0
#define ADAMAS_ERR_CONFIG 1
#define ADAMAS_ERR_RUNTIME 2

#define ADAMAS_F32 0
#define ADAMAS_BF16 1

/* Sticky device status bits. */
#define ADAMAS_STATUS_DEGENERATE 1     /* a zero / non-finite vector was encoded (quantizer.cpp:46-47) */
#define ADAMAS_STATUS_SYNC_TIMEOUT 4   /* a multi-cluster unit barrier gave up: results invalid */
#define ADAMAS_STATUS_PEER_TIMEOUT 8   /* a peer-memory exchange wait gave up: results invalid */
#define ADAMAS_STATUS_BAD_SELECTION 16 /* sparse_attention: a row is empty, unsorted or out of range
                                          (kv_cache.cpp:90-91, attention.cpp:42); nothing was read */

typedef struct adamas_cache adamas_cache;

/* Version string of the library build. */
const char* adamas_version(void);

/* Message of the last failing call on this thread ("" if none). */
const char* adamas_last_error(void);

/* ---------------------------------------------------------------- cache
 * Replaces KvCache(head_dim, bits) (kv_cache.cpp:32-41), batched over the
 * layer's kv-heads, with device storage for `capacity` tokens per head:
 * K, V in kv_dtype and 32 B of codes per token per head. Rejects
 * head_dim != 128, bits != 2, n_kv_heads < 1 or capacity < 1. */
int adamas_cache_create(adamas_cache** out, int n_kv_heads, int head_dim, int bits,
                        int64_t capacity, int kv_dtype);
int adamas_cache_destroy(adamas_cache* cache);
/* KvCache::seq_len (kv_cache.hpp:23). */
int adamas_cache_seq_len(const adamas_cache* cache, int64_t* out);
/* Rewinds the sequence length (tokens past it are forgotten). 0 <= seq_len <= current. */
int adamas_cache_truncate(adamas_cache* cache, int64_t seq_len);
/* Device addresses of the cache arrays (for callers fusing their own kernels). */
int adamas_cache_buffers(const adamas_cache* cache, void** keys, void** values, void** codes);
/* Reads and clears the sticky device status word (synchronizes the stream). */
int adamas_cache_status(adamas_cache* cache, void* stream, int* status);

/* Fused encode + append. Replaces, for every token and kv-head,
 * KvCache::update(k, v, pack(encode(k))) (kv_cache.cpp:62-71 with
 * sweep.cpp:32-36, :44-47 — the build_cache loop, sweep.cpp:38-50).
 * keys/values: device [n_tokens][n_kv_heads][128]. Used for single-token
 * decode appends and for bulk prefill alike. */
int adamas_cache_append(adamas_cache* cache, const void* keys, const void* values, int64_t n_tokens,
                        void* stream);

/* Append with caller-supplied codes in the REFERENCE word layout
 * (PackedCodes.words, quantizer.hpp:44-50): KvCache::update(k, v, code).
 * codes_ref: device uint16 [n_tokens][n_kv_heads][16]. */
int adamas_cache_append_coded(adamas_cache* cache, const void* keys, const void* values,
                              const uint16_t* codes_ref, int64_t n_tokens, void* stream);

/* Copies codes of tokens [start, start+n) of every kv-head out in the reference
 * word layout (KvCache::code_words, kv_cache.hpp:35-37) into device uint16
 * [n_kv_heads][n][16]. */
int adamas_cache_codes_ref(const adamas_cache* cache, int64_t start, int64_t n, uint16_t* out_ref,
                           void* stream);

/* ADKV snapshot interchange (the reference's save_snapshot / load_snapshot,
 * kv_cache.cpp:111-165; one file per kv-head, as the reference cache is one
 * head): magic "ADKV", u32 version 1, u32 seq_len, u32 head_dim, u8 bits, f32
 * keys, f32 values, u16 PackedCodes words. Save writes kv-head `kv_head`'s
 * tokens [0, seq_len) (bf16 caches widen to f32 exactly); load appends the
 * n_paths == n_kv_heads snapshots (equal lengths) with their code words
 * verbatim (no re-encode; f32 values round to bf16 in a bf16 cache).
 * I/O and format errors -> ADAMAS_ERR_RUNTIME (std::runtime_error in the
 * reference); shapes this build does not hold (head_dim != 128, 1-bit) ->
 * ADAMAS_ERR_CONFIG. Both synchronize `stream`. */
int adamas_cache_save_adkv(const adamas_cache* cache, int kv_head, const char* path, void* stream);
int adamas_cache_load_adkv(adamas_cache* cache, const char* const* paths, int n_paths, void* stream);

/* ---------------------------------------------------------------- operators */

/* pack(encode(q)) per q-head (sweep.cpp:92-94): q device [n_q_heads][128] in the
 * cache's dtype -> device uint16 [n_q_heads][16] reference-layout words. */
int adamas_encode_query(const adamas_cache* cache, const void* q, int n_q_heads, uint16_t* out_ref,
                        void* stream);

/* score_all(q_code, cache, Metric::manhattan) per q-head (estimator.cpp:45-59):
 * q_ref device uint16 [n_q_heads][16] -> device int32 [n_q_heads][seq_len]. */
int adamas_score(const adamas_cache* cache, const uint16_t* q_ref, int n_q_heads, int32_t* scores,
                 void* stream);

/* Ablation metrics over the same cache (the reference's Metric, estimator.hpp:11,
 * and its 1-bit pipeline, kernels.hpp:24-32):
 *   ADAMAS_METRIC_MANHATTAN     = adamas_score
 *   ADAMAS_METRIC_EUCLIDEAN_SQ  score_all(q, cache, Metric::euclidean_sq), 2-bit codes
 *   ADAMAS_METRIC_HAMMING_1BIT  score_all over the 1-bit pipeline (pack(encode(x, 1)),
 *                               l1_1bit): the 1-bit code is the 2-bit code's high bit
 *                               (both threshold at 0), so the 2-bit cache serves it.
 * q_ref: 2-bit reference words as for adamas_score. */
#define ADAMAS_METRIC_MANHATTAN 0
#define ADAMAS_METRIC_EUCLIDEAN_SQ 1
#define ADAMAS_METRIC_HAMMING_1BIT 2
int adamas_score_metric(const adamas_cache* cache, const uint16_t* q_ref, int n_q_heads, int metric,
                        int32_t* scores, void* stream);

/* top_k(scores, k) per row (estimator.cpp:75-90): the k smallest under the
 * order (score, index), ascending indices. scores device int32 [n_rows][n]
 * (any int32 value, as the reference's DistanceScores); idx device int32
 * [n_rows][k]; entries past min(k, n) are set to -1. */
int adamas_topk(const int32_t* scores, int n_rows, int64_t n, int64_t k, int32_t* idx, void* stream);

/* sparse_attention(q, cache, sel) per q-head (attention.cpp:40-45 = gather,
 * kv_cache.cpp:84-99, + full_attention, attention.cpp:8-38) in fp32:
 * idx device int32 [n_q_heads][k] strictly increasing (-1 entries end a row).
 * The reference's gather preconditions (indices in range and strictly
 * increasing, kv_cache.cpp:90-91) and its empty-selection check
 * (attention.cpp:42) are validated on the device per row: a violating row is
 * not read, its output is NaN and ADAMAS_STATUS_BAD_SELECTION is latched in
 * the cache status (the facades raise ConfigError from it);
 * out device float32 [n_q_heads][128]; lse (optional, may be NULL) device
 * float32 [n_q_heads][2] = (row max logit, sum of exp) for log-sum-exp merges. */
int adamas_sparse_attention(const adamas_cache* cache, const void* q, int n_q_heads,
                            const int32_t* idx, int64_t k, float* out, float* lse, void* stream);

/* ---------------------------------------------------------------- decode step
 * One Adamas decode step of one layer (Algorithm 1; sweep.cpp:87-98 then
 * :225-226, with the cache update first): append the new
 * token's (k, v) with its codes, encode q, scan every key code, select the
 * top `budget` per q-head and attend over the selection.
 * q: [n_q_heads][128]; k_new, v_new: [n_kv_heads][128]; out float32
 * [n_q_heads][128]; idx (optional, may be NULL) int32 [n_q_heads][budget].
 * Runs as one fused kernel launch. */
int adamas_decode_step(adamas_cache* cache, const void* q, int n_q_heads, const void* k_new,
                       const void* v_new, int64_t budget, float* out, int32_t* idx, void* stream);


/* Same step for a batch of independent sequences (per-request caches with the
 * same shape and dtype) in one launch: caches[i], q + i*n_q_heads*128, ...
 * out + i*n_q_heads*128, idx + i*n_q_heads*budget. */
int adamas_decode_step_batched(adamas_cache* const* caches, int n_seqs, const void* q, int n_q_heads,
                               const void* k_new, const void* v_new, int64_t budget, float* out,
                               int32_t* idx, void* stream);

/* ---------------------------------------------------------------- sequence-sharded decode
 * One decode step over a sequence split in contiguous token ranges across
 * ranks (the reference's single score_all + top_k +
 * sparse_attention, estimator.cpp:45-90 and attention.cpp:8-45, over the whole
 * sequence). Per rank: local candidates -> all-gather the keys -> select and
 * attend -> all-gather the partials -> LSE merge. Bit-exact selection: a
 * member of the global (distance, index) top-k has fewer than k predecessors
 * in its own range, so it is among that range's candidates.
 *
 * Local candidates: optionally appends (k_new, v_new) with its code (the rank
 * owning the sequence tail), encodes q, scans the local cache and writes this
 * range's top-`budget` keys per q-head, cand_keys uint32 [n_q][budget]:
 * (distance << 23) | (base_index + local token); unused entries 0xFFFFFFFF.
 * Global indices must stay below 2^23. */
int adamas_seq_local_candidates(adamas_cache* cache, const void* q, int n_q_heads, const void* k_new,
                                const void* v_new, int append, int64_t base_index, int64_t budget,
                                uint32_t* cand_keys, void* stream);

/* Select + attend: gathered uint32 [n_ranks][n_q][budget] keys of every rank,
 * total_len = tokens of the whole sequence (after this step's append),
 * rank_base = global index of this cache's token 0. Writes the partial of this
 * rank's survivors, float32 [n_q][132] = (m in natural-log units, l, 0, 0,
 * o[128] unnormalised), and optionally the global selection int32
 * [n_q][budget] ascending (-1 past min(budget, total_len)).
 * n_ranks * budget <= 8192, budget <= 2048. Input contract (what
 * adamas_seq_local_candidates produces): each rank's keys ascending in the
 * index field with empty keys (0xffffffff) last, ranks in sequence order; the
 * selection is then an order-preserving compaction (no sort). Keys violating
 * it latch ADAMAS_STATUS_BAD_SELECTION in the cache status and the launch
 * writes nothing. */
int adamas_seq_select_attend(const adamas_cache* cache, const void* q, int n_q_heads, const uint32_t* gathered,
                             int n_ranks, int64_t budget, int64_t total_len, int64_t rank_base, float* partial,
                             int32_t* global_idx, void* stream);

/* Log-sum-exp merge of the ranks' partials float32 [n_ranks][n_q][132] into
 * out float32 [n_q][128]. */
int adamas_lse_merge(const float* partials, int n_ranks, int n_q_heads, float* out, void* stream);

/* adamas_seq_select_attend + adamas_lse_merge in ONE launch, for callers whose
 * other ranks' partials are already in `partials` [n_ranks][n_q][132] when it
 * runs (this rank's goes to slot my_slot, then every q-head is merged into
 * out [n_q][128]). The peer-memory step (adamas_seq_step_p2p) fuses the same
 * way, waiting on the peers' epochs instead. Same sparse_attention /
 * attention.cpp:8-45 semantics as the two calls. */
int adamas_seq_select_attend_merge(const adamas_cache* cache, const void* q, int n_q_heads, const uint32_t* gathered,
                                   int n_ranks, int64_t budget, int64_t total_len, int64_t rank_base, float* partials,
                                   int my_slot, float* out, int32_t* global_idx, void* stream);

/* ---------------------------------------------------------------- sequence sharding over peer memory
 * The same three phases as adamas_seq_local_candidates / _select_attend /
 * _lse_merge, with the two all-gathers replaced by stores into every rank's
 * mailbox over NVLink: phase 1's fused kernel writes its candidate keys
 * straight into all mailboxes and publishes an epoch (system-scope release);
 * phase 2 acquires every rank's keys epoch, selects + attends, and writes its
 * partial into all mailboxes; phase 3 acquires the partial epochs and merges.
 * No NCCL call, no host synchronisation, graph-capturable. Mailboxes are
 * cudaMalloc'd (CUDA IPC); ranks exchange the 64-byte handles once at setup
 * (any transport: torch.distributed all_gather_object, MPI, a file) and call
 * adamas_mailbox_connect. Ranks of one process (tests, one GPU) use
 * adamas_mailbox_connect_local. A wait that exceeds ~4 s latches
 * ADAMAS_STATUS_PEER_TIMEOUT (adamas_mailbox_status) instead of hanging. */
#define ADAMAS_IPC_HANDLE_BYTES 64
#define ADAMAS_STATUS_PEER_TIMEOUT 8
typedef struct adamas_mailbox adamas_mailbox;
int adamas_mailbox_create(adamas_mailbox** out, int rank, int world, int n_q_heads, int64_t budget);
int adamas_mailbox_ipc_handle(const adamas_mailbox* mailbox, void* handle);
int adamas_mailbox_connect(adamas_mailbox* mailbox, const void* handles /* world x 64 B, rank order */);
int adamas_mailbox_connect_local(adamas_mailbox* const* mailboxes, int world);
int adamas_mailbox_status(adamas_mailbox* mailbox, int* status);
int adamas_mailbox_destroy(adamas_mailbox* mailbox);
/* phase 1: append (tail rank) + local candidates, pushed to every rank; advances the epoch */
int adamas_seq_p2p_local(adamas_cache* cache, adamas_mailbox* mailbox, const void* q, int n_q_heads, const void* k_new,
                         const void* v_new, int append, int64_t base_index, void* stream);
/* phase 2: wait for every rank's keys, global select, attend this rank's survivors, push the partial */
int adamas_seq_p2p_select_attend(const adamas_cache* cache, adamas_mailbox* mailbox, const void* q, int n_q_heads,
                                 int64_t total_len, int64_t rank_base, int32_t* global_idx, void* stream);
/* phase 3: wait for every rank's partial, log-sum-exp merge -> out [n_q][128] f32 */
int adamas_seq_p2p_merge(adamas_mailbox* mailbox, float* out, void* stream);
/* phases 1-3 */
int adamas_seq_step_p2p(adamas_cache* cache, adamas_mailbox* mailbox, const void* q, int n_q_heads, const void* k_new,
                        const void* v_new, int append, int64_t base_index, int64_t total_len, float* out,
                        int32_t* global_idx, void* stream);

/* ---------------------------------------------------------------- f3: harness selection backend
 * The sweep harness's selection step on the GPU, in the
 * harness's own arithmetic: fp64 inputs, any power-of-two head_dim in
 * [2, 1024], 1/2/3-bit codes, with or without the Hadamard transform. Codes,
 * distances, dot and page scores are bit-identical to the reference's (same
 * correctly rounded fp64 operations in the same order); the selections are
 * therefore identical index sets.
 *
 * Rows and instances: the harness pairs every query with one key/value
 * instance (workload.hpp:69-80). Gaussian workloads share one instance across
 * all queries, planted-needle workloads own one per query. Inputs are stacked
 * device arrays keys/values [n_inst][seq_len][head_dim], queries
 * [n_rows][head_dim]; row r reads instance r / rows_per_inst.
 * Index outputs are int64 [n_rows][budget], ascending, -1 past the selection. */
typedef struct adamas_hsel adamas_hsel;

/* PolicySpec{adamas, bits, metric, with_hadamard} (sweep.hpp:15-33). Rejects
 * head_dim outside {2, 4, ..., 1024} and bits outside 1..3 (quantizer.cpp:17-21). */
int adamas_hsel_create(adamas_hsel** out, int head_dim, int bits, int with_hadamard);
int adamas_hsel_destroy(adamas_hsel* sel);

/* build_cache (sweep.cpp:38-50) over n_inst key matrices: encode (sweep.cpp:32-36)
 * = fwht (hadamard.cpp:36-41) + compute_thresholds + bucketize (quantizer.cpp:40-85).
 * Synchronises `stream`; a zero or non-finite key returns ADAMAS_ERR_CONFIG with
 * the reference's message (quantizer.cpp:46-47). Replaces the previous build. */
int adamas_hsel_build(adamas_hsel* sel, const double* keys, int64_t n_inst, int64_t seq_len, void* stream);

/* Codes of built vectors first..first+n-1 (instance-major) in the reference's
 * formats, device out: PackedCodes words (quantizer.cpp:87-117) for 1/2 bits
 * (ceil(head_dim / (16 / bits)) uint16 per vector), CodeVector bytes for 3. */
int adamas_hsel_codes_ref(const adamas_hsel* sel, int64_t first, int64_t n, void* out, void* stream);

/* The adamas branch of select (sweep.cpp:87-98): encode each query, score_all
 * (estimator.cpp:45-73, metric ADAMAS_METRIC_MANHATTAN or _EUCLIDEAN_SQ; the
 * 1-bit pipeline uses popcount for both, estimator.cpp:51-52), top_k
 * (estimator.cpp:75-90). Synchronises `stream` after encoding the queries
 * (degenerate query -> ADAMAS_ERR_CONFIG). At most 65535 rows per call. */
int adamas_hsel_select(adamas_hsel* sel, const double* queries, int64_t n_rows, int64_t rows_per_inst, int metric,
                       int64_t budget, int64_t* idx, void* stream);

/* The oracle policy / recall reference: top_k_by_score (baselines.cpp:21-32)
 * over dot(q, k_i) (common.hpp:65-69), largest first, ties toward the smaller
 * index. `scores` (nullable) receives the fp64 dot scores [n_rows][seq_len]. */
int adamas_dot_topk(const double* queries, const double* keys, int64_t n_rows, int64_t rows_per_inst, int64_t n_inst,
                    int64_t seq_len, int head_dim, int64_t k, int64_t* idx, double* scores, void* stream);

/* top_k_by_score (baselines.cpp:21-32) over given fp64 scores [n_rows][n]
 * (e.g. the scores adamas_dot_topk returned, reused for several budgets). */
int adamas_topk_f64(const double* scores, int64_t n_rows, int64_t n, int64_t k, int64_t* idx, void* stream);

/* The quest baseline. PageSummaries (baselines.cpp:34-54) of n_inst key
 * matrices, built once (prepare_state, sweep.cpp:68-72), then page_select
 * (baselines.cpp:71-91) per budget: counts[r] = indices written for row r (the
 * last page may be partial); budget must be a multiple of page_size unless
 * >= seq_len. adamas_page_select is the one-shot form (synchronises). */
typedef struct adamas_pages adamas_pages;
int adamas_pages_create(adamas_pages** out, int64_t page_size, int head_dim);
int adamas_pages_destroy(adamas_pages* pages);
int adamas_pages_build(adamas_pages* pages, const double* keys, int64_t n_inst, int64_t seq_len, void* stream);
int adamas_pages_select(adamas_pages* pages, const double* queries, int64_t n_rows, int64_t rows_per_inst,
                        int64_t budget, int64_t* idx, int64_t* counts, void* stream);
int adamas_page_select(const double* queries, const double* keys, int64_t n_rows, int64_t rows_per_inst,
                       int64_t n_inst, int64_t seq_len, int head_dim, int64_t page_size, int64_t budget, int64_t* idx,
                       int64_t* counts, void* stream);

/* full_attention (attention.cpp:8-38) in fp64 over all seq_len rows (idx NULL)
 * or over the selected rows idx[r][0..counts[r]) (attend_subset, sweep.cpp:120-131;
 * counts NULL = idx_stride rows each). out [n_rows][head_dim]. Same operation
 * order as the reference; exp() may differ from libm's in the last place. */
int adamas_attention_f64(const double* queries, const double* keys, const double* values, int64_t n_rows,
                         int64_t rows_per_inst, int64_t n_inst, int64_t seq_len, int head_dim, const int64_t* idx,
                         int64_t idx_stride, const int64_t* counts, double* out, void* stream);

/* ---------------------------------------------------------------- diagnostics
 * Subsequent fused decode launches write up to 16 %globaltimer stamps per CTA
 * (phase boundaries) into device_buffer[blockIdx * 16 + i]; NULL disables.
 * Effective only in a diagnostics build of the library (ADAMAS_DIAG=1,
 * `python paper_2510_18413_b200/build.py --diag`); a no-op otherwise. */
void adamas_debug_trace(unsigned long long* device_buffer);

/* Launch-plan overrides for tests and tools (the automatic plan is the
 * product default). values[i] for i < n, in order: qsplit (0 auto), cluster
 * CTAs (0 auto), clusters per unit P (1), ring stages (0 auto), shared-memory
 * cap in KB (0 auto), exact fp64 encode (0), diagnostics switches (0), no PDL
 * (0), composed operators instead of the fused launch (0), require the fused
 * launch (0). The initial values are read once from the ADAMAS_QSPLIT,
 * ADAMAS_CLUSTER, ADAMAS_P, ADAMAS_STAGES, ADAMAS_SMEM_KB, ADAMAS_EXACT_ENCODE,
 * ADAMAS_DBG, ADAMAS_NO_PDL, ADAMAS_NO_FUSED, ADAMAS_REQUIRE_FUSED environment
 * variables at first use; nothing on the launch path reads the environment. */
#define ADAMAS_TUNING_FIELDS 10
int adamas_set_tuning(const int* values, int n);
int adamas_get_tuning(int* values, int n);

/* ---------------------------------------------------------------- host converters */

/* Reference PackedCodes words <-> device bit-plane record (32 B), host memory,
 * n vectors of 128 codes: uint32 planes[8] per vector, words 0..3 the low code
 * bits (element e at bit e/4 of word e%4), words 4..7 low XOR high bit.
 * Lossless both ways. */
void adamas_codes_ref_to_planes(const uint16_t* ref, int64_t n, uint32_t* planes);
void adamas_codes_planes_to_ref(const uint32_t* planes, int64_t n, uint16_t* ref);

#ifdef __cplusplus
}
#endif
#endif
