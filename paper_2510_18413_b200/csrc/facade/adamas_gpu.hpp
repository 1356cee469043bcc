// adamas_gpu.hpp — C++ facade of the B200 hot path with the reference's
// operator signatures (namespace adamas in /root/reference/proj/include).
//
// A reference user switches `adamas::` for `adamas::gpu::` on the hot path:
// KvCache / update / score_all / top_k / sparse_attention keep their meaning,
// argument order and error classes; the work runs in the sm_100a kernels
// behind the C ABI (include/adamas_b200.h). These entry points take and
// return HOST containers (std::vector / std::span), so every call copies its
// inputs to the device and its results back; batched device-resident decoding
// uses the C ABI directly (adamas_decode_step).
//
// Precision contract: the device stores K, V (and encodes q) in the cache's
// element type (fp32 by default). Inputs that are exactly representable in
// that type (all fp32 / bf16 model activations) give codes, distances and
// indices bit-identical to the reference; attention is fp32 (within 1e-3
// relative of the double reference for fp32 K/V, 1e-2 for bf16).
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "adamas_b200.h"

namespace adamas::gpu {

using RealVector = std::vector<double>;

// common.hpp:19-22
class ConfigError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};

// quantizer.hpp:44-50
struct PackedCodes {
  std::vector<std::uint16_t> words;
  std::size_t len = 0;
  int bits = 2;
  std::size_t codes_per_word() const { return 16u / static_cast<unsigned>(bits); }
};

// estimator.hpp:11,20,26-28
enum class Metric { manhattan, euclidean_sq };
using DistanceScores = std::vector<std::int32_t>;
struct SelectionResult {
  std::vector<std::size_t> indices;  // ascending
};

// attention.hpp:11-16
struct AttentionOutput {
  RealVector out;
};

enum class Dtype { f32 = ADAMAS_F32, bf16 = ADAMAS_BF16 };

// kv_cache.hpp:19-33 — one head, device resident. `capacity` bounds the
// append-only sequence (the reference grows without bound in 2048-row chunks).
class KvCache {
 public:
  KvCache(std::size_t head_dim, int bits, std::size_t capacity = 1u << 16, Dtype dtype = Dtype::f32);
  ~KvCache();
  KvCache(const KvCache&) = delete;
  KvCache& operator=(const KvCache&) = delete;
  KvCache(KvCache&& o) noexcept;

  // KvCache::update(key, value, code) — caller-supplied packed code.
  std::size_t update(std::span<const double> key, std::span<const double> value, const PackedCodes& code);
  // update with the code computed on the device: update(k, v, pack(encode(k))).
  std::size_t update(std::span<const double> key, std::span<const double> value);
  // Bulk prefill: rows x head_dim keys/values, codes computed on the device.
  std::size_t update_rows(std::span<const double> keys, std::span<const double> values, std::size_t rows);

  std::size_t seq_len() const;
  std::size_t head_dim() const { return head_dim_; }
  int bits() const { return bits_; }
  std::size_t words_per_code() const { return 16; }
  std::vector<std::uint16_t> code_words(std::size_t i) const;

  adamas_cache* handle() const { return h_; }
  Dtype dtype() const { return dtype_; }

 private:
  adamas_cache* h_ = nullptr;
  std::size_t head_dim_;
  int bits_;
  Dtype dtype_;
};

// pack(encode(x)) computed on the device (sweep.cpp:32-36 + quantizer.cpp:87).
PackedCodes encode_pack(std::span<const double> x, const KvCache& like);

// estimator.cpp:45-59 (Metric::manhattan only; euclidean_sq is an ablation).
DistanceScores score_all(const PackedCodes& query, const KvCache& cache, Metric metric = Metric::manhattan);

// estimator.cpp:75-90
SelectionResult top_k(const DistanceScores& scores, std::size_t k);

// attention.cpp:40-45
AttentionOutput sparse_attention(std::span<const double> q, const KvCache& cache, const SelectionResult& sel);

// One Adamas decode step (sweep.cpp:87-98, :225-226 with the update first):
// appends (k_new, v_new), selects `budget` tokens for q and attends.
struct DecodeResult {
  SelectionResult selection;
  AttentionOutput attention;
};
DecodeResult decode_step(KvCache& cache, std::span<const double> q, std::span<const double> k_new,
                         std::span<const double> v_new, std::size_t budget);

// attention.cpp:47-57
double output_error(const AttentionOutput& approx, const AttentionOutput& exact);

// ---------------------------------------------------------------- the sweep harness (f3)
// The harness's fp64 selection path on the device, any power-of-two head_dim
// in [2, 1024] and 1/2/3-bit codes: one policy's code store
// (PolicySpec{adamas, bits, metric, with_hadamard}, sweep.hpp:15-33).
class CodeStore {
 public:
  CodeStore(std::size_t head_dim, int bits = 2, bool with_hadamard = true);
  ~CodeStore();
  CodeStore(const CodeStore&) = delete;
  CodeStore& operator=(const CodeStore&) = delete;

  // build_cache (sweep.cpp:38-50) over `rows` keys (row-major rows x head_dim).
  void build(std::span<const double> keys, std::size_t rows);
  // The adamas branch of select (sweep.cpp:87-98): encode, score_all, top_k.
  SelectionResult select(std::span<const double> query, std::size_t budget, Metric metric = Metric::manhattan) const;
  // Built codes of row i in the reference's formats: PackedCodes words for
  // 1/2 bits, CodeVector bytes (one per uint16 here) for 3.
  std::vector<std::uint16_t> codes(std::size_t i) const;
  std::size_t rows() const { return rows_; }

 private:
  adamas_hsel* h_ = nullptr;
  std::size_t head_dim_, rows_ = 0;
  int bits_;
};

// top_k_by_score over dot(q, k_i) (baselines.cpp:21-32): the oracle policy.
std::vector<std::size_t> top_k_by_dot(std::span<const double> q, std::span<const double> keys, std::size_t rows,
                                      std::size_t k);

}  // namespace adamas::gpu
