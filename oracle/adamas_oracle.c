/*
 * adamas_oracle.c — CPU restatement of the Adamas reference hot path.
 * TEST INFRASTRUCTURE ONLY (see adamas_oracle.h). Parity pinned against the
 * reference build in oracle/_ref and tests/golden/.
 * Compile with -ffp-contract=off (see oracle/Makefile).
 */
#include "adamas_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- synthetic data */

static uint64_t or_splitmix64(uint64_t z) {
  /* splitmix64 finalizer, the same mixing workload.hpp:15-21 uses for seeds. */
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

float or_synth_value(uint64_t seed, uint64_t index) {
  const uint64_t h = or_splitmix64(seed ^ (index * 0xD1B54A32D192ED03ULL));
  const int64_t s = (int64_t)(h & 0xFFFF) + (int64_t)((h >> 16) & 0xFFFF) +
                    (int64_t)((h >> 32) & 0xFFFF) + (int64_t)(h >> 48);
  /* Irwin-Hall(4) over [0, 65535]: mean 131070, sd ~= 37837.2 */
  return (float)((double)(s - 131070) / 37837.0);
}

void or_synth_fill(uint64_t seed, uint64_t first_index, size_t n, float* out) {
  for (size_t i = 0; i < n; ++i) out[i] = or_synth_value(seed, first_index + i);
}

/* ---------------------------------------------------------------- transform */

static int is_pow2(size_t n) { return n > 0 && (n & (n - 1)) == 0; }

int or_fwht(double* x, size_t n, int normalized) {
  /* HadamardSpec::validate, hadamard.cpp:10-15 */
  if (n < 2 || !is_pow2(n)) return OR_CONFIG;
  /* fwht_scalar, kernels_scalar.cpp:11-35; k_inv_sqrt2 from kernels_impl.hpp:10 */
  const double c = 0.70710678118654752440;
  for (size_t h = 1; h < n; h <<= 1) {
    for (size_t i = 0; i < n; i += 2 * h) {
      for (size_t j = i; j < i + h; ++j) {
        const double a = x[j];
        const double b = x[j + h];
        if (normalized) {
          x[j] = (a + b) * c;
          x[j + h] = (a - b) * c;
        } else {
          x[j] = a + b;
          x[j + h] = a - b;
        }
      }
    }
  }
  return OR_OK;
}

/* ---------------------------------------------------------------- quantizer */

int or_compute_thresholds(const double* x, size_t n, int bits, double* out) {
  /* quantizer.cpp:12-14 */
  const double q18 = 1.1503493803760081783;
  const double q28 = 0.6744897501960817432;
  const double q38 = 0.31863936396437516302;
  if (bits < 1 || bits > 3) return OR_CONFIG; /* check_bits :16-21 */
  if (n == 0) return OR_CONFIG;               /* :42 */
  double sumsq = 0.0;
  for (size_t i = 0; i < n; ++i) sumsq += x[i] * x[i]; /* :43-44, index order */
  const double sigma = sqrt(sumsq / (double)n);        /* :45 */
  if (!isfinite(sigma)) return OR_CONFIG;              /* :46 */
  if (sigma == 0.0) return OR_CONFIG;                  /* :47 */
  switch (bits) {                                      /* :51-62 */
    case 1:
      out[0] = 0.0;
      break;
    case 2:
      out[0] = -q28 * sigma;
      out[1] = 0.0;
      out[2] = q28 * sigma;
      break;
    default:
      out[0] = -q18 * sigma;
      out[1] = -q28 * sigma;
      out[2] = -q38 * sigma;
      out[3] = 0.0;
      out[4] = q38 * sigma;
      out[5] = q28 * sigma;
      out[6] = q18 * sigma;
      break;
  }
  return OR_OK;
}

void or_bucketize(const double* x, size_t n, const double* t, int bits, uint8_t* codes) {
  /* quantizer.cpp:74-85: strict '>' so ties go to the lower bucket */
  const size_t nt = ((size_t)1 << bits) - 1;
  for (size_t i = 0; i < n; ++i) {
    uint8_t level = 0;
    for (size_t j = 0; j < nt; ++j) level += x[i] > t[j] ? 1 : 0;
    codes[i] = level;
  }
}

int or_pack(const uint8_t* codes, size_t n, int bits, uint16_t* words, size_t* nwords) {
  /* quantizer.cpp:87-117 (pad = true) */
  if (bits != 1 && bits != 2) return OR_CONFIG;
  const size_t per_word = 16u / (unsigned)bits;
  const size_t nw = (n + per_word - 1) / per_word;
  for (size_t w = 0; w < nw; ++w) words[w] = 0;
  const unsigned max_code = 1u << bits;
  for (size_t i = 0; i < n; ++i) {
    if (codes[i] >= max_code) return OR_CONFIG;
    words[i / per_word] |= (uint16_t)((unsigned)codes[i] << (bits * (i % per_word)));
  }
  *nwords = nw;
  return OR_OK;
}

void or_unpack(const uint16_t* words, size_t nwords, int bits, uint8_t* codes) {
  /* quantizer.cpp:119-130 */
  const size_t per_word = 16u / (unsigned)bits;
  const unsigned mask = (1u << bits) - 1u;
  for (size_t i = 0; i < nwords * per_word; ++i)
    codes[i] = (uint8_t)((words[i / per_word] >> (bits * (i % per_word))) & mask);
}

int or_encode_pack(const double* x, size_t d, uint16_t* words) {
  /* sweep.cpp:32-36 with_hadamard = true, bits = 2; then pack (sweep.cpp:46, :93) */
  double* t = (double*)malloc(d * sizeof(double));
  uint8_t* codes = (uint8_t*)malloc(d);
  double th[3];
  size_t nw = 0;
  int rc;
  if (!t || !codes) {
    free(t);
    free(codes);
    return OR_CONFIG;
  }
  memcpy(t, x, d * sizeof(double));
  rc = or_fwht(t, d, 1);
  if (rc == OR_OK) rc = or_compute_thresholds(t, d, 2, th);
  if (rc == OR_OK) {
    or_bucketize(t, d, th, 2, codes);
    rc = or_pack(codes, d, 2, words, &nw);
  }
  free(t);
  free(codes);
  return rc;
}

/* ---------------------------------------------------------------- estimator */

uint32_t or_l1_2bit(const uint16_t* q, const uint16_t* k, size_t nwords) {
  /* kernels_scalar.cpp:65-82: sum over the eight 2-bit lanes of every word of
   * |q_lane - k_lane|; restated lane by lane (the SWAR is an implementation
   * detail, test_kernels.cpp:19-32 uses this same unpack-and-subtract oracle). */
  uint32_t acc = 0;
  for (size_t w = 0; w < nwords; ++w) {
    for (int lane = 0; lane < 8; ++lane) {
      const int a = (q[w] >> (2 * lane)) & 3;
      const int b = (k[w] >> (2 * lane)) & 3;
      acc += (uint32_t)(a > b ? a - b : b - a);
    }
  }
  return acc;
}

void or_score_all(const uint16_t* q, const uint16_t* cache_words, size_t seq_len, size_t nwords,
                  int32_t* scores) {
  /* estimator.cpp:53-57 */
  for (size_t i = 0; i < seq_len; ++i)
    scores[i] = (int32_t)or_l1_2bit(q, cache_words + i * nwords, nwords);
}

typedef struct {
  int32_t s;
  int64_t i;
} or_pair;

static int cmp_pair(const void* a, const void* b) {
  const or_pair* x = (const or_pair*)a;
  const or_pair* y = (const or_pair*)b;
  if (x->s != y->s) return x->s < y->s ? -1 : 1;
  return x->i < y->i ? -1 : (x->i > y->i ? 1 : 0);
}

static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

size_t or_top_k(const int32_t* scores, size_t n, size_t k, int64_t* idx) {
  /* estimator.cpp:75-90: k >= n selects everything (:80); otherwise the k
   * smallest under (score, index), then re-sorted by index (:83-88). */
  if (k >= n) {
    for (size_t i = 0; i < n; ++i) idx[i] = (int64_t)i;
    return n;
  }
  if (k == 0) return 0;
  /* Small non-negative scores (all Adamas distances): exact counting select. */
  int32_t lo = scores[0], hi = scores[0];
  for (size_t i = 1; i < n; ++i) {
    if (scores[i] < lo) lo = scores[i];
    if (scores[i] > hi) hi = scores[i];
  }
  if (lo >= 0 && hi < 65536) {
    size_t* hist = (size_t*)calloc((size_t)hi + 1, sizeof(size_t));
    size_t cum = 0, below = 0, out = 0;
    int32_t t = 0;
    for (size_t i = 0; i < n; ++i) hist[scores[i]]++;
    for (t = 0; t <= hi; ++t) {
      if (cum + hist[t] >= k) break;
      cum += hist[t];
    }
    below = cum;                   /* strictly smaller than the threshold t */
    size_t need = k - below;       /* ties at t, lowest indices first */
    for (size_t i = 0; i < n; ++i) {
      if (scores[i] < t) {
        idx[out++] = (int64_t)i;
      } else if (scores[i] == t && need > 0) {
        idx[out++] = (int64_t)i;
        --need;
      }
    }
    free(hist);
    return out;
  }
  or_pair* p = (or_pair*)malloc(n * sizeof(or_pair));
  for (size_t i = 0; i < n; ++i) {
    p[i].s = scores[i];
    p[i].i = (int64_t)i;
  }
  qsort(p, n, sizeof(or_pair), cmp_pair);
  for (size_t i = 0; i < k; ++i) idx[i] = p[i].i;
  free(p);
  qsort(idx, k, sizeof(int64_t), cmp_i64);
  return k;
}

/* ---------------------------------------------------------------- attention */

int or_full_attention(const double* q, const double* K, const double* V, size_t rows, size_t d,
                      double* out) {
  /* attention.cpp:8-38 */
  if (rows == 0) return OR_CONFIG; /* :10 */
  const double scale = 1.0 / sqrt((double)d);
  double* logits = (double*)malloc(rows * sizeof(double));
  for (size_t i = 0; i < rows; ++i) {
    double acc = 0.0; /* dot, common.hpp:65-69 */
    for (size_t j = 0; j < d; ++j) acc += q[j] * K[i * d + j];
    logits[i] = acc * scale;
  }
  double peak = logits[0];
  for (size_t i = 1; i < rows; ++i)
    if (logits[i] > peak) peak = logits[i];
  double denom = 0.0;
  for (size_t i = 0; i < rows; ++i) {
    logits[i] = exp(logits[i] - peak);
    denom += logits[i];
  }
  for (size_t j = 0; j < d; ++j) out[j] = 0.0;
  for (size_t i = 0; i < rows; ++i) {
    const double w = logits[i] / denom;
    for (size_t j = 0; j < d; ++j) out[j] += w * V[i * d + j];
  }
  free(logits);
  return OR_OK;
}

int or_sparse_attention(const double* q, const double* K, const double* V, size_t seq_len, size_t d,
                        const int64_t* idx, size_t nidx, double* out) {
  /* attention.cpp:40-45; gather checks kv_cache.cpp:90-91 */
  if (nidx == 0) return OR_CONFIG;
  double* ks = (double*)malloc(nidx * d * sizeof(double));
  double* vs = (double*)malloc(nidx * d * sizeof(double));
  int rc = OR_OK;
  for (size_t r = 0; r < nidx && rc == OR_OK; ++r) {
    if (idx[r] < 0 || (size_t)idx[r] >= seq_len) rc = OR_CONFIG;
    else if (r > 0 && idx[r] <= idx[r - 1]) rc = OR_CONFIG;
    else {
      memcpy(ks + r * d, K + (size_t)idx[r] * d, d * sizeof(double));
      memcpy(vs + r * d, V + (size_t)idx[r] * d, d * sizeof(double));
    }
  }
  if (rc == OR_OK) rc = or_full_attention(q, ks, vs, nidx, d, out);
  free(ks);
  free(vs);
  return rc;
}

double or_output_error(const double* approx, const double* exact, size_t d) {
  /* attention.cpp:47-57 */
  double diff = 0.0, ref = 0.0;
  for (size_t i = 0; i < d; ++i) {
    const double e = approx[i] - exact[i];
    diff += e * e;
  }
  for (size_t i = 0; i < d; ++i) ref += exact[i] * exact[i];
  ref = sqrt(ref);
  return sqrt(diff) / (ref > 1e-30 ? ref : 1e-30);
}

/* ---------------------------------------------------------------- decode step */

int or_decode_head(const double* q, const double* K, const double* V, const uint16_t* cache_words,
                   size_t seq_len, size_t d, size_t budget, int64_t* idx, size_t* nidx,
                   int32_t* scores_scratch, double* out) {
  const size_t nwords = (d + 7) / 8;
  uint16_t qw[128];
  if (nwords > 128) return OR_CONFIG;
  int rc = or_encode_pack(q, d, qw);                            /* sweep.cpp:92-94 */
  if (rc != OR_OK) return rc;
  or_score_all(qw, cache_words, seq_len, nwords, scores_scratch); /* :95 */
  *nidx = or_top_k(scores_scratch, seq_len, budget, idx);         /* :97 */
  return or_sparse_attention(q, K, V, seq_len, d, idx, *nidx, out); /* sweep.cpp:225-226 */
}
