/*
 * adamas_oracle.h — CPU restatement of the Adamas reference algorithm for the
 * decode-time sparse-attention hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product path may link, load or call
 * this library: it is the checker that tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py compare the CUDA path against.
 *
 * Parity: pinned. tests/test_oracle.py checks every function against the
 * reference library compiled from /root/reference/proj/src (oracle/_ref, see
 * oracle/Makefile) and against the committed golden vectors in tests/golden/
 * that were produced by that reference build (tests/golden/make_golden.py).
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). Build with -ffp-contract=off: the reference's double
 * arithmetic contains no fused multiply-adds and the codes are only bit-exact
 * when the restatement performs the same roundings in the same order.
 */
#ifndef ADAMAS_ORACLE_H
#define ADAMAS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: OR_CONFIG mirrors adamas::ConfigError (include/adamas/common.hpp:19-22). */
#define OR_OK 0
#define OR_CONFIG 1

/* Deterministic synthetic Gaussian-like generator shared bit-for-bit by numpy
 * (tests/synth.py), this file and the CUDA generator: splitmix64 over the
 * element index, four 16-bit lanes summed (Irwin-Hall), scaled to unit
 * variance, rounded once to float. Pure integer + one IEEE division. */
float or_synth_value(uint64_t seed, uint64_t index);
void or_synth_fill(uint64_t seed, uint64_t first_index, size_t n, float* out);

/* fwht_scalar: kernels_scalar.cpp:11-35; dimension check hadamard.cpp:10-24. */
int or_fwht(double* x, size_t n, int normalized);

/* compute_thresholds: quantizer.cpp:40-64 (constants :12-14). out holds 2^bits-1 values. */
int or_compute_thresholds(const double* x, size_t n, int bits, double* out);

/* bucketize: quantizer.cpp:74-85 — code = number of thresholds strictly below x. */
void or_bucketize(const double* x, size_t n, const double* t, int bits, uint8_t* codes);

/* pack: quantizer.cpp:87-117. Writes ceil(n / (16/bits)) words (padded with code 0). */
int or_pack(const uint8_t* codes, size_t n, int bits, uint16_t* words, size_t* nwords);

/* unpack: quantizer.cpp:119-130. */
void or_unpack(const uint16_t* words, size_t nwords, int bits, uint8_t* codes);

/* encode (sweep.cpp:32-36) followed by pack (sweep.cpp:44-47, :92-94):
 * pack(bucketize(fwht(x), compute_thresholds(fwht(x), 2))). x is not modified. */
int or_encode_pack(const double* x, size_t d, uint16_t* words);

/* l1_2bit over nwords packed words (kernels_scalar.cpp:65-82), restated lane by lane. */
uint32_t or_l1_2bit(const uint16_t* q, const uint16_t* k, size_t nwords);

/* score_all, Manhattan, 2-bit (estimator.cpp:45-59). cache_words: seq_len rows of nwords. */
void or_score_all(const uint16_t* q, const uint16_t* cache_words, size_t seq_len, size_t nwords,
                  int32_t* scores);

/* top_k (estimator.cpp:75-90): the k smallest scores under the order (score, index),
 * returned as ascending indices. Returns the number of indices written: min(k, n). */
size_t or_top_k(const int32_t* scores, size_t n, size_t k, int64_t* idx);

/* full_attention (attention.cpp:8-38): softmax(q K^T / sqrt(d)) V in double with the
 * reference's operation order. K, V: rows x d row-major. */
int or_full_attention(const double* q, const double* K, const double* V, size_t rows, size_t d,
                      double* out);

/* sparse_attention (attention.cpp:40-45) = gather (kv_cache.cpp:84-99) + full_attention.
 * Rejects empty, out-of-range or non-increasing selections like the reference. */
int or_sparse_attention(const double* q, const double* K, const double* V, size_t seq_len, size_t d,
                        const int64_t* idx, size_t nidx, double* out);

/* output_error (attention.cpp:47-57). */
double or_output_error(const double* approx, const double* exact, size_t d);

/* One decode step for one head over a prebuilt cache (sweep.cpp:87-98 then :225-226):
 * q_words = pack(encode(q)); scores = score_all; sel = top_k(scores, budget);
 * out = sparse_attention(q, cache, sel). idx receives min(budget, seq_len) indices. */
int or_decode_head(const double* q, const double* K, const double* V, const uint16_t* cache_words,
                   size_t seq_len, size_t d, size_t budget, int64_t* idx, size_t* nidx,
                   int32_t* scores_scratch, double* out);

#ifdef __cplusplus
}
#endif
#endif
