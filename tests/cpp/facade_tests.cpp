// facade_tests.cpp — the reference's hot-path doctest cases, re-run through the
// C++ facade (adamas::gpu, sm_100a kernels) and checked against the reference's
// known answers and the C restatement in oracle/ (test infrastructure).
// Exit code 0 = all passed. Run by tests/test_gpu_facade.py (-m gpu).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <numeric>
#include <random>
#include <vector>

#include "adamas_gpu.hpp"
#include "adamas_oracle.h"

using namespace adamas::gpu;

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                          \
  do {                                                                    \
    if (c) ++g_pass;                                                      \
    else { ++g_fail; std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); } \
  } while (0)

template <typename F>
static bool throws_config(F&& f) {
  try { f(); } catch (const ConfigError&) { return true; } catch (...) { return false; }
  return false;
}

static std::vector<double> synth_vec(uint64_t seed, size_t n) {
  std::vector<float> f(n);
  or_synth_fill(seed, 0, n, f.data());
  return {f.begin(), f.end()};
}

int main() {
  const size_t d = 128;
  // test_estimator.cpp:217-224 top_k tie-breaks
  CHECK((top_k({5, 1, 9, 1}, 2).indices == std::vector<size_t>{1, 3}));
  CHECK((top_k({1, 1, 1}, 2).indices == std::vector<size_t>{0, 1}));
  CHECK((top_k({4, 3, 2, 1}, 10).indices == std::vector<size_t>{0, 1, 2, 3}));
  CHECK((top_k({7}, 1).indices == std::vector<size_t>{0}));
  CHECK(top_k({}, 3).indices.empty());
  CHECK(top_k({3, 2, 1}, 0).indices.empty());
  {  // test_estimator.cpp:226-243 against the oracle with dense ties
    std::mt19937_64 rng(8);
    std::uniform_int_distribution<int32_t> score(0, 50);
    for (int rep = 0; rep < 20; ++rep) {
      DistanceScores s(1000);
      for (auto& x : s) x = score(rng);
      std::vector<int64_t> idx(64);
      const size_t n = or_top_k(s.data(), s.size(), 64, idx.data());
      const auto got = top_k(s, 64).indices;
      CHECK(got.size() == n);
      bool same = true;
      for (size_t i = 0; i < n && i < got.size(); ++i) same &= (int64_t)got[i] == idx[i];
      CHECK(same);
    }
  }
  // kv_cache ctor rejections (kv_cache.cpp:33-34) + specialization
  CHECK(throws_config([] { KvCache c(0, 2); }));
  CHECK(throws_config([] { KvCache c(128, 4); }));
  CHECK(throws_config([] { KvCache c(64, 2); }));
  {  // encode / update / code_words / score_all / sparse_attention vs oracle
    KvCache cache(d, 2, 4096);
    const size_t S = 1000;
    std::vector<double> K, V;
    for (size_t i = 0; i < S; ++i) {
      auto k = synth_vec(1000 + i, d), v = synth_vec(50000 + i, d);
      K.insert(K.end(), k.begin(), k.end());
      V.insert(V.end(), v.begin(), v.end());
    }
    CHECK(cache.update_rows(K, V, S) == S);
    std::vector<uint16_t> words(S * 16);
    for (size_t i = 0; i < S; ++i) or_encode_pack(K.data() + i * d, d, words.data() + i * 16);
    bool codes_ok = true;
    for (size_t i = 0; i < S; i += 37) codes_ok &= cache.code_words(i) == std::vector<uint16_t>(words.begin() + i * 16, words.begin() + i * 16 + 16);
    CHECK(codes_ok);
    auto q = synth_vec(7, d);
    const PackedCodes qc = encode_pack(q, cache);
    std::vector<uint16_t> qw(16);
    or_encode_pack(q.data(), d, qw.data());
    CHECK(qc.words == qw);
    const auto scores = score_all(qc, cache);
    std::vector<int32_t> expect(S);
    or_score_all(qw.data(), words.data(), S, 16, expect.data());
    CHECK(scores == expect);
    const auto sel = top_k(scores, 64);
    std::vector<int64_t> eidx(64);
    or_top_k(expect.data(), S, 64, eidx.data());
    bool idx_ok = sel.indices.size() == 64;
    for (size_t i = 0; i < 64 && idx_ok; ++i) idx_ok &= (int64_t)sel.indices[i] == eidx[i];
    CHECK(idx_ok);
    const auto att = sparse_attention(q, cache, sel);
    AttentionOutput exact;
    exact.out.resize(d);
    or_sparse_attention(q.data(), K.data(), V.data(), S, d, eidx.data(), 64, exact.out.data());
    CHECK(output_error(att, exact) <= 1e-5);
    // gather checks (kv_cache.cpp:90-91), empty selection (attention.cpp:42)
    CHECK(throws_config([&] { sparse_attention(q, cache, SelectionResult{{5, 3}}); }));
    CHECK(throws_config([&] { sparse_attention(q, cache, SelectionResult{{S}}); }));
    CHECK(throws_config([&] { sparse_attention(q, cache, SelectionResult{}); }));
    // score_all width checks (estimator.cpp:46-49)
    PackedCodes bad = qc;
    bad.bits = 1;
    CHECK(throws_config([&] { score_all(bad, cache); }));
    // singleton selection returns the value row (test_attention.cpp:174-179)
    const auto one = sparse_attention(q, cache, SelectionResult{{5}});
    bool row_ok = true;
    for (size_t j = 0; j < d; ++j) row_ok &= std::fabs(one.out[j] - V[5 * d + j]) < 1e-6;
    CHECK(row_ok);
    // decode step: update then select (Alg. 1), against the oracle over S+1 tokens
    auto kn = synth_vec(777, d), vn = synth_vec(778, d), q2 = synth_vec(779, d);
    const auto r = decode_step(cache, q2, kn, vn, 128);
    K.insert(K.end(), kn.begin(), kn.end());
    V.insert(V.end(), vn.begin(), vn.end());
    words.resize((S + 1) * 16);
    or_encode_pack(kn.data(), d, words.data() + S * 16);
    std::vector<int32_t> sc(S + 1);
    std::vector<int64_t> di(128);
    size_t nd = 0;
    AttentionOutput dex;
    dex.out.resize(d);
    or_decode_head(q2.data(), K.data(), V.data(), words.data(), S + 1, d, 128, di.data(), &nd, sc.data(), dex.out.data());
    bool dec_ok = r.selection.indices.size() == nd;
    for (size_t i = 0; i < nd && dec_ok; ++i) dec_ok &= (int64_t)r.selection.indices[i] == di[i];
    CHECK(dec_ok);
    CHECK(output_error(r.attention, dex) <= 1e-5);
    CHECK(cache.seq_len() == S + 1);
    // degenerate vector -> ConfigError (quantizer.cpp:47)
    std::vector<double> zeros(d, 0.0);
    CHECK(throws_config([&] { encode_pack(zeros, cache); }));
  }
  {  // the sweep harness's fp64 selection (f3): codes + select against the C restatement
    const size_t S = 700;
    std::vector<double> K;
    for (size_t i = 0; i < S; ++i) {
      auto row = synth_vec(5000 + i, d);
      K.insert(K.end(), row.begin(), row.end());
    }
    CodeStore store(d, 2, true);
    store.build(K, S);
    bool codes_ok = true;
    std::vector<uint16_t> ref_words(S * 16);
    for (size_t i = 0; i < S; ++i) {
      or_encode_pack(K.data() + i * d, d, ref_words.data() + i * 16);
      const auto got = store.codes(i);
      codes_ok &= got.size() == 16 && std::equal(got.begin(), got.end(), ref_words.begin() + i * 16);
    }
    CHECK(codes_ok);
    const auto q = synth_vec(777, d);
    std::vector<uint16_t> qw(16);
    or_encode_pack(q.data(), d, qw.data());
    std::vector<int32_t> sc(S);
    or_score_all(qw.data(), ref_words.data(), S, 16, sc.data());
    for (size_t budget : {1u, 64u, 699u, 700u, 900u}) {
      std::vector<int64_t> ei(budget);
      const size_t n = or_top_k(sc.data(), S, budget, ei.data());
      const auto got = store.select(q, budget).indices;
      bool same = got.size() == n;
      for (size_t i = 0; i < n && same; ++i) same &= (int64_t)got[i] == ei[i];
      CHECK(same);
    }
    // top_k_by_score over dot products (baselines.cpp:21-32): largest first, ties to the lower index
    std::vector<double> dots(S);
    for (size_t i = 0; i < S; ++i) {
      double acc = 0.0;
      for (size_t j = 0; j < d; ++j) acc += q[j] * K[i * d + j];
      dots[i] = acc;
    }
    std::vector<size_t> order(S);
    std::iota(order.begin(), order.end(), size_t{0});
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return dots[a] > dots[b]; });
    std::vector<size_t> exp(order.begin(), order.begin() + 32);
    std::sort(exp.begin(), exp.end());
    CHECK(top_k_by_dot(q, K, S, 32) == exp);
    CHECK(throws_config([] { CodeStore bad(48, 2, true); }));
    CHECK(throws_config([] { CodeStore bad(64, 4, true); }));
    std::vector<double> zk(3 * d, 1.0);
    std::fill(zk.begin() + d, zk.begin() + 2 * d, 0.0);
    CodeStore z(d, 2, true);
    CHECK(throws_config([&] { z.build(zk, 3); }));
  }
  std::printf("facade_tests: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
