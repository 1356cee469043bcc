// adamas_gpu.cpp — host side of the C++ facade; every operator is one or more
// C ABI calls (sm_100a kernels) plus host<->device copies of its arguments.
#include "adamas_gpu.hpp"

#include <cuda_runtime_api.h>

#include <algorithm>
#include <cmath>
#include <cstring>

namespace adamas::gpu {
namespace {

constexpr cudaMemcpyKind kH2D = cudaMemcpyHostToDevice, kD2H = cudaMemcpyDeviceToHost;

void check(int rc) {
  if (rc == ADAMAS_OK) return;
  const std::string msg = adamas_last_error();
  if (rc == ADAMAS_ERR_CONFIG) throw ConfigError(msg);
  throw std::runtime_error(msg);
}

void cuda(cudaError_t rc, const char* what) {
  if (rc != cudaSuccess) throw std::runtime_error(std::string("CUDA failure in ") + what + ": " + cudaGetErrorString(rc));
}

// Device buffer RAII.
struct Dev {
  void* p = nullptr;
  explicit Dev(size_t n) { cuda(cudaMalloc(&p, n ? n : 1), "cudaMalloc"); }
  ~Dev() { cudaFree(p); }
  Dev(Dev&& o) noexcept : p(o.p) { o.p = nullptr; }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};

uint16_t to_bf16_bits(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// Host doubles -> device elements of the cache type.
Dev upload(std::span<const double> x, Dtype dt) {
  if (dt == Dtype::f32) {
    std::vector<float> f(x.begin(), x.end());
    Dev d(f.size() * 4);
    cuda(cudaMemcpy(d.p, f.data(), f.size() * 4, kH2D), "upload");
    return d;
  }
  std::vector<uint16_t> b(x.size());
  for (size_t i = 0; i < x.size(); ++i) b[i] = to_bf16_bits(static_cast<float>(x[i]));
  Dev d(b.size() * 2);
  cuda(cudaMemcpy(d.p, b.data(), b.size() * 2, kH2D), "upload");
  return d;
}

void raise_on_status(adamas_cache* h) {
  int st = 0;
  check(adamas_cache_status(h, nullptr, &st));
  if (st & ADAMAS_STATUS_DEGENERATE)
    throw ConfigError("degenerate scale: input vector is all zeros or non-finite");
}

}  // namespace

KvCache::KvCache(std::size_t head_dim, int bits, std::size_t capacity, Dtype dtype)
    : head_dim_(head_dim), bits_(bits), dtype_(dtype) {
  check(adamas_cache_create(&h_, 1, static_cast<int>(head_dim), bits, static_cast<int64_t>(capacity),
                            static_cast<int>(dtype)));
}

KvCache::~KvCache() { adamas_cache_destroy(h_); }

KvCache::KvCache(KvCache&& o) noexcept : h_(o.h_), head_dim_(o.head_dim_), bits_(o.bits_), dtype_(o.dtype_) {
  o.h_ = nullptr;
}

std::size_t KvCache::seq_len() const {
  int64_t n = 0;
  check(adamas_cache_seq_len(h_, &n));
  return static_cast<std::size_t>(n);
}

std::size_t KvCache::update(std::span<const double> key, std::span<const double> value, const PackedCodes& code) {
  // kv_cache.cpp:65-70 checks
  if (code.bits != bits_) throw ConfigError("KvCache: code width does not match cache");
  if (code.words.size() != words_per_code()) throw ConfigError("KvCache: code length does not match head_dim");
  if (key.size() != head_dim_ || value.size() != head_dim_)
    throw ConfigError("KvCache: key/value length does not match head_dim");
  Dev k = upload(key, dtype_), v = upload(value, dtype_);
  Dev c(32);
  cuda(cudaMemcpy(c.p, code.words.data(), 32, kH2D), "upload code");
  check(adamas_cache_append_coded(h_, k.p, v.p, static_cast<const uint16_t*>(c.p), 1, nullptr));
  cuda(cudaDeviceSynchronize(), "update");
  return seq_len();
}

std::size_t KvCache::update(std::span<const double> key, std::span<const double> value) {
  return update_rows(key, value, 1);
}

std::size_t KvCache::update_rows(std::span<const double> keys, std::span<const double> values, std::size_t rows) {
  if (keys.size() != rows * head_dim_ || values.size() != rows * head_dim_)
    throw ConfigError("KvCache: key/value length does not match head_dim");
  Dev k = upload(keys, dtype_), v = upload(values, dtype_);
  check(adamas_cache_append(h_, k.p, v.p, static_cast<int64_t>(rows), nullptr));
  raise_on_status(h_);
  return seq_len();
}

std::vector<std::uint16_t> KvCache::code_words(std::size_t i) const {
  if (i >= seq_len()) throw ConfigError("KvCache: row out of range");
  Dev d(32);
  check(adamas_cache_codes_ref(h_, static_cast<int64_t>(i), 1, static_cast<uint16_t*>(d.p), nullptr));
  std::vector<std::uint16_t> w(16);
  cuda(cudaMemcpy(w.data(), d.p, 32, kD2H), "code_words");
  return w;
}

PackedCodes encode_pack(std::span<const double> x, const KvCache& like) {
  if (x.size() != like.head_dim()) throw ConfigError("encode: length does not match head_dim");
  Dev q = upload(x, like.dtype());
  Dev w(32);
  check(adamas_encode_query(like.handle(), q.p, 1, static_cast<uint16_t*>(w.p), nullptr));
  raise_on_status(like.handle());
  PackedCodes p;
  p.words.resize(16);
  p.len = 128;
  p.bits = 2;
  cuda(cudaMemcpy(p.words.data(), w.p, 32, kD2H), "encode");
  return p;
}

DistanceScores score_all(const PackedCodes& query, const KvCache& cache, Metric metric) {
  // estimator.cpp:46-49
  if (query.bits != cache.bits()) throw ConfigError("score_all: code widths differ");
  if (query.words.size() != cache.words_per_code()) throw ConfigError("score_all: code length differs");
  if (metric != Metric::manhattan) throw ConfigError("score_all: only Metric::manhattan runs on the B200 path");
  const size_t n = cache.seq_len();
  DistanceScores s(n);
  if (n == 0) return s;
  Dev q(32), d(n * 4);
  cuda(cudaMemcpy(q.p, query.words.data(), 32, kH2D), "score q");
  check(adamas_score(cache.handle(), static_cast<const uint16_t*>(q.p), 1, static_cast<int32_t*>(d.p), nullptr));
  cuda(cudaMemcpy(s.data(), d.p, n * 4, kD2H), "score out");
  return s;
}

SelectionResult top_k(const DistanceScores& scores, std::size_t k) {
  SelectionResult r;
  const size_t n = scores.size();
  const size_t keep = k < n ? k : n;
  if (keep == 0) return r;
  Dev s(n * 4), o(k * 4);
  cuda(cudaMemcpy(s.p, scores.data(), n * 4, kH2D), "top_k in");
  check(adamas_topk(static_cast<const int32_t*>(s.p), 1, static_cast<int64_t>(n), static_cast<int64_t>(k),
                    static_cast<int32_t*>(o.p), nullptr));
  std::vector<int32_t> idx(k);
  cuda(cudaMemcpy(idx.data(), o.p, k * 4, kD2H), "top_k out");
  r.indices.assign(idx.begin(), idx.begin() + static_cast<std::ptrdiff_t>(keep));
  return r;
}

AttentionOutput sparse_attention(std::span<const double> q, const KvCache& cache, const SelectionResult& sel) {
  if (sel.indices.empty()) throw ConfigError("sparse_attention: empty selection");
  if (q.size() != cache.head_dim()) throw ConfigError("full_attention: query length mismatch");
  const size_t n = cache.seq_len();
  std::vector<int32_t> idx(sel.indices.size());
  for (size_t r = 0; r < idx.size(); ++r) {  // kv_cache.cpp:90-91
    if (sel.indices[r] >= n) throw ConfigError("KvCache: gather index out of range");
    if (r > 0 && sel.indices[r] <= sel.indices[r - 1])
      throw ConfigError("KvCache: gather indices must be increasing");
    idx[r] = static_cast<int32_t>(sel.indices[r]);
  }
  Dev qd = upload(q, cache.dtype());
  Dev id(idx.size() * 4), out(128 * 4);
  cuda(cudaMemcpy(id.p, idx.data(), idx.size() * 4, kH2D), "attend idx");
  check(adamas_sparse_attention(cache.handle(), qd.p, 1, static_cast<const int32_t*>(id.p),
                                static_cast<int64_t>(idx.size()), static_cast<float*>(out.p), nullptr, nullptr));
  std::vector<float> o(128);
  cuda(cudaMemcpy(o.data(), out.p, 128 * 4, kD2H), "attend out");
  AttentionOutput a;
  a.out.assign(o.begin(), o.end());
  return a;
}

DecodeResult decode_step(KvCache& cache, std::span<const double> q, std::span<const double> k_new,
                         std::span<const double> v_new, std::size_t budget) {
  if (q.size() != cache.head_dim() || k_new.size() != cache.head_dim() || v_new.size() != cache.head_dim())
    throw ConfigError("decode_step: vector length does not match head_dim");
  if (budget == 0) throw ConfigError("sparse_attention: empty selection");
  Dev qd = upload(q, cache.dtype()), kd = upload(k_new, cache.dtype()), vd = upload(v_new, cache.dtype());
  Dev out(128 * 4), idx(budget * 4);
  check(adamas_decode_step(cache.handle(), qd.p, 1, kd.p, vd.p, static_cast<int64_t>(budget),
                           static_cast<float*>(out.p), static_cast<int32_t*>(idx.p), nullptr));
  raise_on_status(cache.handle());
  DecodeResult r;
  std::vector<float> o(128);
  std::vector<int32_t> id(budget);
  cuda(cudaMemcpy(o.data(), out.p, 128 * 4, kD2H), "decode out");
  cuda(cudaMemcpy(id.data(), idx.p, budget * 4, kD2H), "decode idx");
  r.attention.out.assign(o.begin(), o.end());
  for (int32_t i : id)
    if (i >= 0) r.selection.indices.push_back(static_cast<size_t>(i));
  return r;
}

double output_error(const AttentionOutput& approx, const AttentionOutput& exact) {
  if (approx.out.size() != exact.out.size()) throw ConfigError("output_error: dimension mismatch");
  double diff = 0.0, ref = 0.0;
  for (size_t i = 0; i < exact.out.size(); ++i) {
    const double d = approx.out[i] - exact.out[i];
    diff += d * d;
    ref += exact.out[i] * exact.out[i];
  }
  return std::sqrt(diff) / std::max(std::sqrt(ref), 1e-30);
}

// ---------------------------------------------------------------- the sweep harness (f3)
namespace {
Dev upload_f64(std::span<const double> x) {
  Dev d(x.size() * 8);
  cuda(cudaMemcpy(d.p, x.data(), x.size() * 8, kH2D), "upload f64");
  return d;
}
}  // namespace

CodeStore::CodeStore(std::size_t head_dim, int bits, bool with_hadamard) : head_dim_(head_dim), bits_(bits) {
  check(adamas_hsel_create(&h_, static_cast<int>(head_dim), bits, with_hadamard ? 1 : 0));
}

CodeStore::~CodeStore() { adamas_hsel_destroy(h_); }

void CodeStore::build(std::span<const double> keys, std::size_t rows) {
  if (keys.size() != rows * head_dim_) throw ConfigError("build_cache: keys do not match rows x head_dim");
  Dev k = upload_f64(keys);
  check(adamas_hsel_build(h_, static_cast<const double*>(k.p), 1, static_cast<int64_t>(rows), nullptr));
  rows_ = rows;
}

SelectionResult CodeStore::select(std::span<const double> query, std::size_t budget, Metric metric) const {
  if (query.size() != head_dim_) throw ConfigError("score_all: code length differs");
  SelectionResult r;
  if (budget == 0) return r;
  Dev q = upload_f64(query), idx(budget * 8);
  check(adamas_hsel_select(h_, static_cast<const double*>(q.p), 1, 1,
                           metric == Metric::manhattan ? ADAMAS_METRIC_MANHATTAN : ADAMAS_METRIC_EUCLIDEAN_SQ,
                           static_cast<int64_t>(budget), static_cast<int64_t*>(idx.p), nullptr));
  std::vector<int64_t> h(budget);
  cuda(cudaMemcpy(h.data(), idx.p, budget * 8, kD2H), "select out");
  for (int64_t i : h)
    if (i >= 0) r.indices.push_back(static_cast<std::size_t>(i));
  return r;
}

std::vector<std::uint16_t> CodeStore::codes(std::size_t i) const {
  if (i >= rows_) throw ConfigError("CodeStore: row out of range");
  const size_t n = bits_ == 3 ? head_dim_ : (head_dim_ + 16 / bits_ - 1) / (16 / bits_);
  const size_t bytes = bits_ == 3 ? n : n * 2;
  Dev d(bytes);
  check(adamas_hsel_codes_ref(h_, static_cast<int64_t>(i), 1, d.p, nullptr));
  std::vector<std::uint16_t> out(n);
  if (bits_ == 3) {
    std::vector<std::uint8_t> b(n);
    cuda(cudaMemcpy(b.data(), d.p, n, kD2H), "codes");
    std::copy(b.begin(), b.end(), out.begin());
  } else {
    cuda(cudaMemcpy(out.data(), d.p, bytes, kD2H), "codes");
  }
  return out;
}

std::vector<std::size_t> top_k_by_dot(std::span<const double> q, std::span<const double> keys, std::size_t rows,
                                      std::size_t k) {
  const size_t d = q.size();
  if (keys.size() != rows * d) throw ConfigError("top_k_by_dot: keys do not match rows x head_dim");
  std::vector<std::size_t> r;
  if (k == 0 || rows == 0) return r;
  Dev qd = upload_f64(q), kd = upload_f64(keys), idx(k * 8);
  check(adamas_dot_topk(static_cast<const double*>(qd.p), static_cast<const double*>(kd.p), 1, 1, 1,
                        static_cast<int64_t>(rows), static_cast<int>(d), static_cast<int64_t>(k),
                        static_cast<int64_t*>(idx.p), nullptr, nullptr));
  std::vector<int64_t> h(k);
  cuda(cudaMemcpy(h.data(), idx.p, k * 8, kD2H), "top_k_by_dot out");
  for (int64_t i : h)
    if (i >= 0) r.push_back(static_cast<std::size_t>(i));
  return r;
}

}  // namespace adamas::gpu
