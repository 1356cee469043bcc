// ref_shim.cpp — extern "C" entry points over the UNMODIFIED reference library
// (/root/reference/proj/src, compiled by oracle/Makefile into oracle/_ref/).
//
// TEST INFRASTRUCTURE ONLY: used to pin the C restatement (adamas_oracle.c),
// to generate tests/golden/ fixtures, and as the reference CPU arm of bench.py
// (cpu_baseline.kind = "reference"). Never linked into the product library.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "adamas/attention.hpp"
#include "adamas/common.hpp"
#include "adamas/estimator.hpp"
#include "adamas/hadamard.hpp"
#include "adamas/kv_cache.hpp"
#include "adamas/quantizer.hpp"
#include "adamas/simd.hpp"
#include "adamas/baselines.hpp"
#include "adamas/sweep.hpp"
#include "adamas/workload.hpp"

using namespace adamas;

namespace {

// 0 ok, 1 ConfigError, 2 any other std::exception (adamas_cli.cpp:233-243 mapping).
thread_local std::string g_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_error = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 2;
  }
}

// sweep.cpp:32-36 (encode with the Hadamard transform) — private there, so
// restated here from the public operators it composes.
CodeVector encode(std::span<const double> x, int bits) {
  const RealVector t = fwht(x, {.dim = x.size()});
  return bucketize(t, compute_thresholds(t, bits));
}

// Same integer synthetic generator as oracle/adamas_oracle.c:or_synth_value.
uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
float synth(uint64_t seed, uint64_t index) {
  const uint64_t h = mix(seed ^ (index * 0xD1B54A32D192ED03ULL));
  const int64_t s = (int64_t)(h & 0xFFFF) + (int64_t)((h >> 16) & 0xFFFF) +
                    (int64_t)((h >> 32) & 0xFFFF) + (int64_t)(h >> 48);
  return (float)((double)(s - 131070) / 37837.0);
}
float round_bf16(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);  // round to nearest even (finite inputs)
  u &= 0xFFFF0000u;
  float y;
  std::memcpy(&y, &u, 4);
  return y;
}

WorkloadSpec make_spec(uint64_t seed, size_t seq_len, size_t head_dim, size_t num_queries, int distribution,
                       double outlier_frac, double outlier_scale, size_t position, double snr) {
  WorkloadSpec w;
  w.seed = seed;
  w.seq_len = seq_len;
  w.head_dim = head_dim;
  w.num_queries = num_queries;
  w.distribution = static_cast<DistributionKind>(distribution);
  w.outlier_frac = outlier_frac;
  w.outlier_scale = outlier_scale;
  w.position = position;
  w.snr = snr;
  return w;
}

// kinds: 0 adamas, 1 window, 2 quest, 3 oracle (PolicySpec::Kind order); metric 0 l1, 1 l2.
SweepConfig make_sweep(const size_t* budgets, size_t n_budgets, const int* kinds, const int* bits,
                       const int* metrics, const int* hadamard, const size_t* sinks, const size_t* page_sizes,
                       size_t n_policies, int measure_output_error) {
  SweepConfig c;
  c.budgets.assign(budgets, budgets + n_budgets);
  for (size_t i = 0; i < n_policies; ++i) {
    PolicySpec p;
    p.kind = static_cast<PolicySpec::Kind>(kinds[i]);
    p.bits = bits[i];
    p.metric = metrics[i] == 0 ? Metric::manhattan : Metric::euclidean_sq;
    p.with_hadamard = hadamard[i] != 0;
    p.sink = sinks[i];
    p.page_size = page_sizes[i];
    c.policies.push_back(p);
  }
  c.measure_output_error = measure_output_error != 0;
  return c;
}

size_t put(const std::string& text, char* out, size_t cap) {
  if (out && cap > 0) {
    const size_t n = std::min(cap - 1, text.size());
    std::memcpy(out, text.data(), n);
    out[n] = 0;
  }
  return text.size();
}

}  // namespace

extern "C" {

// Workload::instance (workload.cpp:125-155): writes query [d], keys and values
// [seq_len][d], the instance seed and the needle position (-1 if none).
int ref_workload_instance(uint64_t seed, size_t seq_len, size_t head_dim, size_t num_queries, int distribution,
                          double outlier_frac, double outlier_scale, size_t position, double snr, size_t qi,
                          double* query, double* keys, double* values, uint64_t* inst_seed, int64_t* needle) {
  return guarded([&] {
    const Workload w(make_spec(seed, seq_len, head_dim, num_queries, distribution, outlier_frac, outlier_scale,
                               position, snr));
    const WorkloadInstance inst = w.instance(qi);
    std::copy(inst.query.begin(), inst.query.end(), query);
    std::copy(inst.keys->data().begin(), inst.keys->data().end(), keys);
    std::copy(inst.values->data().begin(), inst.values->data().end(), values);
    *inst_seed = inst.seed;
    *needle = inst.needle_position ? (int64_t)*inst.needle_position : -1;
  });
}

// run_sweep (sweep.cpp:189-253) + rows_to_csv / rows_to_json (:280-318); the
// needle summary CSV (:255-272, :320-334) when the workload plants needles.
// Each text is returned through (out, cap) with its full length; rc as guarded
// (the ConfigError text via ref_last_error).
int ref_run_sweep(uint64_t seed, size_t seq_len, size_t head_dim, size_t num_queries, int distribution,
                  double outlier_frac, double outlier_scale, size_t position, double snr, const size_t* budgets,
                  size_t n_budgets, const int* kinds, const int* bits, const int* metrics, const int* hadamard,
                  const size_t* sinks, const size_t* page_sizes, size_t n_policies, int measure_output_error,
                  char* csv, size_t csv_cap, size_t* csv_len, char* json, size_t json_cap, size_t* json_len,
                  char* needle_csv, size_t needle_cap, size_t* needle_len) {
  try {
    const auto rows = run_sweep(make_spec(seed, seq_len, head_dim, num_queries, distribution, outlier_frac,
                                          outlier_scale, position, snr),
                                make_sweep(budgets, n_budgets, kinds, bits, metrics, hadamard, sinks, page_sizes,
                                           n_policies, measure_output_error));
    *csv_len = put(rows_to_csv(rows), csv, csv_cap);
    *json_len = put(rows_to_json(rows), json, json_cap);
    *needle_len = 0;
    if (!rows.empty() && rows[0].needle_hit) *needle_len = put(needle_summary_to_csv(needle_report(rows)), needle_csv, needle_cap);
    return 0;
  } catch (const ConfigError& e) {
    g_error = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 2;
  }
}

const char* ref_last_error() { return g_error.c_str(); }

// rows_to_csv over caller-made rows (sweep.cpp:280-297): pins format_number
// (the JSON library's shortest round-trip double text) on arbitrary values.
size_t ref_rows_to_csv(const double* recall, const double* output_error, const int* has_error, size_t n, char* out,
                       size_t cap) {
  std::vector<ResultRow> rows(n);
  for (size_t i = 0; i < n; ++i) {
    rows[i].policy = "p";
    rows[i].recall = recall[i];
    if (has_error[i]) rows[i].output_error = output_error[i];
  }
  return put(rows_to_csv(rows), out, cap);
}

// top_k_by_score (baselines.cpp:21-32) and page_select over PageSummaries
// (baselines.cpp:34-91) for one query.
size_t ref_top_k_by_score(const double* scores, size_t n, size_t k, int64_t* idx) {
  const auto sel = top_k_by_score(std::span<const double>(scores, n), k);
  for (size_t i = 0; i < sel.size(); ++i) idx[i] = (int64_t)sel[i];
  return sel.size();
}

int ref_page_select(const double* q, const double* keys, size_t seq_len, size_t d, size_t page_size, size_t k,
                    int64_t* idx, size_t* n_out) {
  return guarded([&] {
    PageSummaries pages(page_size, d);
    for (size_t i = 0; i < seq_len; ++i) pages.append(std::span<const double>(keys + i * d, d));
    const auto sel = page_select(std::span<const double>(q, d), pages, k);
    for (size_t i = 0; i < sel.indices.size(); ++i) idx[i] = (int64_t)sel.indices[i];
    *n_out = sel.indices.size();
  });
}

// The adamas branch of select (sweep.cpp:87-98) for one query against keys
// [seq_len][d]: build_cache (sweep.cpp:38-50), encode, score_all, top_k.
int ref_adamas_select(const double* q, const double* keys, size_t seq_len, size_t d, int bits, int metric,
                      int hadamard, size_t k, int64_t* idx, size_t* n_out, uint8_t* key_codes, uint8_t* q_codes) {
  return guarded([&] {
    auto enc = [&](std::span<const double> x) {
      if (!hadamard) return bucketize(x, compute_thresholds(x, bits));
      const RealVector t = fwht(x, {.dim = x.size()});
      return bucketize(t, compute_thresholds(t, bits));
    };
    const Metric m = metric == 0 ? Metric::manhattan : Metric::euclidean_sq;
    KvCache cache(d, bits);
    const std::vector<double> zero(d, 0.0);
    const size_t cb = packed_bytes(d, bits);
    for (size_t i = 0; i < seq_len; ++i) {
      const std::span<const double> row(keys + i * d, d);
      const CodeVector c = enc(row);
      if (bits == 3) {
        cache.update(row, zero, c);
        if (key_codes) std::copy(c.codes.begin(), c.codes.end(), key_codes + i * cb);
      } else {
        const PackedCodes p = pack(c);
        cache.update(row, zero, p);
        if (key_codes) std::memcpy(key_codes + i * cb, p.words.data(), p.words.size() * 2);
      }
    }
    const CodeVector qc = enc(std::span<const double>(q, d));
    DistanceScores scores;
    if (bits == 3) {
      scores = score_all(qc, cache, m);
      if (q_codes) std::copy(qc.codes.begin(), qc.codes.end(), q_codes);
    } else {
      const PackedCodes qp = pack(qc);
      scores = score_all(qp, cache, m);
      if (q_codes) std::memcpy(q_codes, qp.words.data(), qp.words.size() * 2);
    }
    const auto sel = top_k(scores, k);
    for (size_t i = 0; i < sel.indices.size(); ++i) idx[i] = (int64_t)sel.indices[i];
    *n_out = sel.indices.size();
  });
}

const char* ref_simd_level() { return simd_level_name(active_simd_level()); }

int ref_fwht(double* x, size_t n, int normalized) {
  return guarded([&] {
    auto y = fwht(std::span<const double>(x, n), {.dim = n, .normalized = normalized != 0});
    std::copy(y.begin(), y.end(), x);
  });
}

int ref_compute_thresholds(const double* x, size_t n, int bits, double* out) {
  return guarded([&] {
    auto t = compute_thresholds(std::span<const double>(x, n), bits);
    std::copy(t.values.begin(), t.values.end(), out);
  });
}

int ref_bucketize(const double* x, size_t n, const double* t, int bits, uint8_t* codes) {
  return guarded([&] {
    BucketThresholds th;
    th.bits = bits;
    th.values.assign(t, t + ((size_t{1} << bits) - 1));
    auto c = bucketize(std::span<const double>(x, n), th);
    std::copy(c.codes.begin(), c.codes.end(), codes);
  });
}

int ref_pack(const uint8_t* codes, size_t n, int bits, uint16_t* words, size_t* nwords) {
  return guarded([&] {
    CodeVector c;
    c.bits = bits;
    c.codes.assign(codes, codes + n);
    auto p = pack(c);
    std::copy(p.words.begin(), p.words.end(), words);
    *nwords = p.words.size();
  });
}

int ref_encode_pack(const double* x, size_t d, uint16_t* words) {
  return guarded([&] {
    auto p = pack(encode(std::span<const double>(x, d), 2));
    std::copy(p.words.begin(), p.words.end(), words);
  });
}

uint32_t ref_manhattan_packed(const uint16_t* a, const uint16_t* b, size_t nwords) {
  PackedCodes pa, pb;
  pa.bits = pb.bits = 2;
  pa.words.assign(a, a + nwords);
  pb.words.assign(b, b + nwords);
  pa.len = pb.len = nwords * 8;
  return manhattan_packed(pa, pb);
}

void* ref_cache_new(size_t head_dim, int bits) {
  try {
    return new KvCache(head_dim, bits);
  } catch (...) {
    return nullptr;
  }
}
void ref_cache_free(void* c) { delete static_cast<KvCache*>(c); }

int ref_cache_update(void* c, const double* k, const double* v, const uint16_t* words) {
  auto* cache = static_cast<KvCache*>(c);
  return guarded([&] {
    PackedCodes p;
    p.bits = cache->bits();
    p.words.assign(words, words + cache->words_per_code());
    p.len = p.words.size() * (16u / unsigned(p.bits));
    const size_t d = cache->head_dim();
    cache->update(std::span<const double>(k, d), std::span<const double>(v, d), p);
  });
}

size_t ref_cache_seq_len(void* c) { return static_cast<KvCache*>(c)->seq_len(); }

// save_snapshot / load_snapshot (kv_cache.cpp:111-165), for the ADKV interop tests.
int ref_save_snapshot(void* c, const char* path) {
  return guarded([&] { save_snapshot(*static_cast<KvCache*>(c), path); });
}
void* ref_load_snapshot(const char* path, int* rc) {
  KvCache* out = nullptr;
  *rc = guarded([&] { out = new KvCache(load_snapshot(path)); });
  return out;
}
void ref_cache_rows(void* c, size_t i, double* key, double* value) {
  auto* cache = static_cast<KvCache*>(c);
  auto k = cache->key_row(i);
  auto v = cache->value_row(i);
  std::copy(k.begin(), k.end(), key);
  std::copy(v.begin(), v.end(), value);
}

void ref_cache_code_words(void* c, size_t i, uint16_t* out) {
  auto w = static_cast<KvCache*>(c)->code_words(i);
  std::copy(w.begin(), w.end(), out);
}

int ref_score_all(void* c, const uint16_t* qwords, int32_t* out) {
  auto* cache = static_cast<KvCache*>(c);
  return guarded([&] {
    PackedCodes q;
    q.bits = cache->bits();
    q.words.assign(qwords, qwords + cache->words_per_code());
    q.len = q.words.size() * (16u / unsigned(q.bits));
    auto s = score_all(q, *cache, Metric::manhattan);
    std::copy(s.begin(), s.end(), out);
  });
}

// score_all with any metric and the cache's own code width (1 or 2 bits).
int ref_score_all_metric(void* c, const uint16_t* qwords, int metric, int32_t* out) {
  auto* cache = static_cast<KvCache*>(c);
  return guarded([&] {
    PackedCodes q;
    q.bits = cache->bits();
    q.words.assign(qwords, qwords + cache->words_per_code());
    q.len = q.words.size() * (16u / unsigned(q.bits));
    auto s = score_all(q, *cache, metric ? Metric::euclidean_sq : Metric::manhattan);
    std::copy(s.begin(), s.end(), out);
  });
}

// pack(encode(x, bits)) (sweep.cpp:32-36) for bits 1 or 2.
int ref_encode_pack_bits(const double* x, size_t d, int bits, uint16_t* words) {
  return guarded([&] {
    const auto p = pack(encode(std::span<const double>(x, d), bits));
    std::copy(p.words.begin(), p.words.end(), words);
  });
}

size_t ref_top_k(const int32_t* scores, size_t n, size_t k, int64_t* idx) {
  DistanceScores s(scores, scores + n);
  auto sel = top_k(s, k);
  for (size_t i = 0; i < sel.indices.size(); ++i) idx[i] = (int64_t)sel.indices[i];
  return sel.indices.size();
}

int ref_sparse_attention(void* c, const double* q, const int64_t* idx, size_t nidx, double* out) {
  auto* cache = static_cast<KvCache*>(c);
  return guarded([&] {
    SelectionResult sel;
    sel.indices.assign(idx, idx + nidx);
    auto o = sparse_attention(std::span<const double>(q, cache->head_dim()), *cache, sel);
    std::copy(o.out.begin(), o.out.end(), out);
  });
}

int ref_full_attention(const double* q, const double* K, const double* V, size_t rows, size_t d,
                       double* out) {
  return guarded([&] {
    RealMatrix km(rows, d), vm(rows, d);
    std::copy(K, K + rows * d, km.data().begin());
    std::copy(V, V + rows * d, vm.data().begin());
    auto o = full_attention(std::span<const double>(q, d), km, vm);
    std::copy(o.out.begin(), o.out.end(), out);
  });
}

// The reference decode step for one head (sweep.cpp:87-98 + :225-226).
int ref_decode_head(void* c, const double* q, size_t budget, int64_t* idx, size_t* nidx,
                    double* out) {
  auto* cache = static_cast<KvCache*>(c);
  return guarded([&] {
    const std::span<const double> qs(q, cache->head_dim());
    const auto qc = pack(encode(qs, 2));
    const auto scores = score_all(qc, *cache, Metric::manhattan);
    const auto sel = top_k(scores, budget);
    const auto o = sparse_attention(qs, *cache, sel);
    for (size_t i = 0; i < sel.indices.size(); ++i) idx[i] = (int64_t)sel.indices[i];
    *nidx = sel.indices.size();
    std::copy(o.out.begin(), o.out.end(), out);
  });
}

// ---------------------------------------------------------------- CPU decode bench
//
// One "layer" = n_heads independent per-head caches of seq_len tokens (head_dim
// d) built from the synthetic generator (bf16-rounded when bf16 != 0). A timed
// decode step runs, for every head, the reference's own operators exactly as
// its pipeline composes them: encode(k_new)+update (the append, Alg. 1 line 4),
// then encode(q) -> score_all -> top_k -> sparse_attention. Heads are spread
// over `threads` std::threads (operators are pure; heads are
// independent). Returns the per-step wall times in us.
struct RefLayer {
  size_t d = 0, heads = 0, budget = 0;
  uint64_t seed = 0;
  bool bf16 = false;
  std::vector<std::unique_ptr<KvCache>> caches;
};

void* ref_layer_build(size_t n_heads, size_t seq_len, size_t d, int bf16, uint64_t seed,
                      int threads) {
  auto* L = new RefLayer;
  L->d = d;
  L->heads = n_heads;
  L->seed = seed;
  L->bf16 = bf16 != 0;
  L->caches.resize(n_heads);
  auto work = [&](size_t h0, size_t h1) {
    std::vector<double> k(d), v(d);
    for (size_t h = h0; h < h1; ++h) {
      auto c = std::make_unique<KvCache>(d, 2);
      const uint64_t ks = seed * 1000003ULL + 2 * h + 1, vs = seed * 1000003ULL + 2 * h + 2;
      for (size_t t = 0; t < seq_len; ++t) {
        for (size_t j = 0; j < d; ++j) {
          float a = synth(ks, t * d + j), b = synth(vs, t * d + j);
          if (L->bf16) {
            a = round_bf16(a);
            b = round_bf16(b);
          }
          k[j] = a;
          v[j] = b;
        }
        c->update(k, v, pack(encode(k, 2)));
      }
      L->caches[h] = std::move(c);
    }
  };
  const int T = std::max(1, threads);
  std::vector<std::thread> pool;
  const size_t per = (n_heads + T - 1) / T;
  for (int t = 0; t < T; ++t) {
    const size_t h0 = t * per, h1 = std::min(n_heads, h0 + per);
    if (h0 < h1) pool.emplace_back(work, h0, h1);
  }
  for (auto& th : pool) th.join();
  return L;
}

void ref_layer_free(void* p) { delete static_cast<RefLayer*>(p); }

// Runs `steps` decode steps; step s appends one synthetic token per head and
// then decodes one synthetic query per head. step_us[s] = wall time of step s.
int ref_layer_decode(void* p, size_t budget, int threads, int steps, double* step_us) {
  auto* L = static_cast<RefLayer*>(p);
  const size_t d = L->d;
  return guarded([&] {
    for (int s = 0; s < steps; ++s) {
      auto work = [&](size_t h0, size_t h1) {
        std::vector<double> q(d), k(d), v(d);
        for (size_t h = h0; h < h1; ++h) {
          KvCache& c = *L->caches[h];
          const uint64_t base = L->seed * 7919ULL + (uint64_t)s * 65537ULL + h;
          for (size_t j = 0; j < d; ++j) {
            float a = synth(base * 3 + 1, j), b = synth(base * 3 + 2, j), e = synth(base * 3 + 3, j);
            if (L->bf16) {
              a = round_bf16(a);
              b = round_bf16(b);
              e = round_bf16(e);
            }
            k[j] = a;
            v[j] = b;
            q[j] = e;
          }
          c.update(k, v, pack(encode(k, 2)));
          const auto qc = pack(encode(q, 2));
          const auto scores = score_all(qc, c, Metric::manhattan);
          const auto sel = top_k(scores, budget);
          const auto o = sparse_attention(q, c, sel);
          if (!std::isfinite(o.out[0])) throw std::runtime_error("non-finite output");
        }
      };
      const int T = std::max(1, threads);
      const size_t per = (L->heads + T - 1) / T;
      const auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> pool;
      for (int t = 0; t < T; ++t) {
        const size_t h0 = t * per, h1 = std::min(L->heads, h0 + per);
        if (h0 < h1) pool.emplace_back(work, h0, h1);
      }
      for (auto& th : pool) th.join();
      const auto t1 = std::chrono::steady_clock::now();
      step_us[s] = std::chrono::duration<double, std::micro>(t1 - t0).count();
    }
  });
}

}  // extern "C"
