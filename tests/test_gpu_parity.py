"""-m gpu: the CUDA path (through the C ABI) against the oracle and the
reference's golden vectors. Integer results bit-exact; attention within the
north-star tolerance (1e-3 relative for fp32 K/V, 1e-2 for bf16 K/V) against
the double oracle that consumes the same stored values."""
import numpy as np
import pytest
import torch

from tests.golden.make_golden import CASES, case_inputs
from tests.gpu_helpers import make_inputs, oracle_decode, rel_err, to_dev

pytestmark = pytest.mark.gpu
TOL = {False: 1e-3, True: 1e-2}


def fill_cache(ad, K, V, bf16, capacity=None):
    S, n_kv, _ = K.shape
    cache = ad.KvCache(n_kv, capacity or S + 8, torch.bfloat16 if bf16 else torch.float32)
    if S:
        cache.update(to_dev(K, bf16), to_dev(V, bf16))
    return cache


@pytest.mark.parametrize("bf16", [False, True])
def test_encode_append_codes_bit_exact(gpu, oracle, bf16):
    S, n_kv = 3000, 3
    K, V, _ = make_inputs(S, n_kv, n_kv, bf16, 11)
    K[7] *= 1e-30  # tiny and huge scales
    K[8] *= 1e30 if not bf16 else 1e20
    if bf16:
        from oracle.bindings import bf16_round
        K = bf16_round(K)
    cache = fill_cache(gpu, K, V, bf16)
    assert cache.seq_len == S
    words = cache.code_words().cpu().numpy().view(np.uint16)
    for h in range(n_kv):
        assert np.array_equal(words[h], oracle.encode_pack_rows(K[:, h].astype(np.float64))), h
    # K/V rows stored verbatim
    keys = cache.keys()[:, :S].float().cpu().numpy()
    assert np.array_equal(keys.transpose(1, 0, 2), K.astype(np.float32))
    assert cache.status() == 0


@pytest.mark.parametrize("bf16", [False, True])
def test_bulk_append_near_threshold_keys(gpu, oracle, bf16):
    """Bulk prefill (the 8-lane encoder, four vectors per warp): keys built to
    sit exactly on the 0 / +-kQ28 sigma thresholds after the transform, at
    scales 1e-4 .. 1e4, mixed with random keys, ragged count; the uncertain
    ones take the exact path, every code must equal the reference's."""
    from oracle.bindings import bf16_round
    rng = np.random.default_rng(23)
    H = np.array([[1.0]])
    for _ in range(7):
        H = np.block([[H, H], [H, -H]])
    H /= np.sqrt(128.0)
    n_kv, S = 2, 517
    K = rng.standard_normal((S, n_kv, 128))
    for t in range(0, S, 3):
        for h in range(n_kv):
            y = rng.standard_normal(128)
            sigma = np.sqrt(np.mean(y * y))
            j = (t + h) % 128
            y[j] = [0.0, 0.6744897501960817 * sigma, -0.6744897501960817 * sigma][(t // 3 + h) % 3]
            K[t, h] = (H @ y) * 10.0 ** ((t % 9) - 4)
    K = K.astype(np.float32)
    if bf16:
        K = bf16_round(K)
    V = rng.standard_normal((S, n_kv, 128)).astype(np.float32)
    if bf16:
        V = bf16_round(V)
    cache = fill_cache(gpu, K, V, bf16)
    words = cache.code_words().cpu().numpy().view(np.uint16)
    for h in range(n_kv):
        assert np.array_equal(words[h], oracle.encode_pack_rows(K[:, h].astype(np.float64))), h
    assert cache.status() == 0


def test_query_encode_bit_exact_many(gpu, oracle):
    n = 4096
    _, _, q = make_inputs(1, 1, n, False, 12)
    cache = gpu.KvCache(1, 16, torch.float32)
    got = cache.encode_query(to_dev(q, False)).cpu().numpy().view(np.uint16)
    exp = oracle.encode_pack_rows(q.astype(np.float64))
    assert np.array_equal(got, exp)


def test_degenerate_vector_sets_status(gpu):
    cache = gpu.KvCache(1, 16, torch.float32)
    z = torch.zeros((1, 1, 128), device="cuda")
    cache.update(z, z)
    with pytest.raises(gpu.ConfigError):
        cache.raise_on_degenerate()
    assert cache.status() == 0  # read-and-clear
    nan = torch.full((1, 128), float("nan"), device="cuda")
    cache.encode_query(nan)
    assert cache.status() == 1


def test_append_coded_roundtrip(gpu, oracle):
    S = 500
    K, V, _ = make_inputs(S, 2, 2, False, 13)
    rng = np.random.default_rng(0)
    codes = rng.integers(0, 65536, (S, 2, 16)).astype(np.uint16)
    cache = gpu.KvCache(2, S, torch.float32)
    cache.update_coded(to_dev(K, False), to_dev(V, False), torch.from_numpy(codes.view(np.int16)).cuda())
    back = cache.code_words().cpu().numpy().view(np.uint16)
    assert np.array_equal(back, codes.transpose(1, 0, 2))


@pytest.mark.parametrize("S,n_kv,G", [(1, 1, 1), (257, 2, 1), (4096, 1, 4), (10000, 2, 2)])
def test_score_all_bit_exact(gpu, oracle, S, n_kv, G):
    K, V, q = make_inputs(S, n_kv, n_kv * G, True, 14)
    cache = fill_cache(gpu, K, V, True)
    qw = cache.encode_query(to_dev(q, True))
    scores = cache.score_all(qw).cpu().numpy()
    kw, exp_scores, _, _ = oracle_decode(oracle, K, V, q, 1)
    assert np.array_equal(qw.cpu().numpy().view(np.uint16), oracle.encode_pack_rows(q.astype(np.float64)))
    assert np.array_equal(scores, exp_scores)


@pytest.mark.parametrize("n,k", [(1000, 64), (1000, 0), (1000, 1), (1000, 999), (1000, 1000), (1000, 5000),
                                 (33000, 128), (5, 2)])
def test_top_k_matches_oracle_dense_ties(gpu, oracle, n, k):
    rng = np.random.default_rng(n + k)
    rows = [rng.integers(0, 51, n), rng.integers(100, 110, n), np.full(n, 7), rng.integers(0, 385, n)]
    s = np.stack(rows).astype(np.int32)
    if k == 0:
        return
    got = gpu.top_k(torch.from_numpy(s).cuda(), k).cpu().numpy()
    for r in range(s.shape[0]):
        exp = oracle.top_k(s[r], k)
        assert np.array_equal(got[r, :len(exp)], exp), r
        assert (got[r, len(exp):] == -1).all()
    assert list(gpu.top_k(torch.tensor([5, 1, 9, 1], dtype=torch.int32).cuda(), 2)[0].cpu()) == [1, 3]
    assert list(gpu.top_k(torch.tensor([1, 1, 1], dtype=torch.int32).cuda(), 2)[0].cpu()) == [0, 1]


@pytest.mark.parametrize("bf16", [False, True])
def test_sparse_attention_tolerance(gpu, oracle, bf16):
    S, n_kv, G = 2000, 2, 2
    K, V, q = make_inputs(S, n_kv, n_kv * G, bf16, 15)
    cache = fill_cache(gpu, K, V, bf16)
    rng = np.random.default_rng(1)
    k = 100
    idx = np.stack([np.sort(rng.choice(S, k, replace=False)) for _ in range(n_kv * G)])
    out = cache.sparse_attention(to_dev(q, bf16), torch.from_numpy(idx.astype(np.int32)).cuda()).cpu().numpy()
    for h in range(n_kv * G):
        exp = oracle.sparse_attention(q[h].astype(np.float64), K[:, h // G].astype(np.float64),
                                      V[:, h // G].astype(np.float64), idx[h])
        assert rel_err(out[h], exp) <= TOL[bf16] / 10
    # singleton selection returns the value row (test_attention.cpp:174-179)
    one = cache.sparse_attention(to_dev(q, bf16), torch.full((n_kv * G, 1), 5, dtype=torch.int32).cuda())
    for h in range(n_kv * G):
        assert np.allclose(one[h].cpu().numpy(), V[5, h // G], rtol=0, atol=1e-6)


def run_decode(gpu, oracle, S, n_kv, G, budget, bf16, seed, steps=1):
    """Cache prefilled with S - steps tokens, then `steps` fused decode steps;
    each step is compared with the oracle over the tokens present after its append."""
    n_q = n_kv * G
    K, V, _ = make_inputs(S, n_kv, n_q, bf16, seed)
    pre = S - steps
    cache = fill_cache(gpu, K[:pre], V[:pre], bf16, capacity=S + 4)
    for st in range(steps):
        t = pre + st
        q = make_inputs(1, 1, n_q, bf16, seed * 1000 + st)[2]
        out, idx = cache.decode_step(to_dev(q, bf16), to_dev(K[t], bf16), to_dev(V[t], bf16), budget)
        out, idx = out.cpu().numpy(), idx.cpu().numpy()
        _, _, eidx, eout = oracle_decode(oracle, K[:t + 1], V[:t + 1], q, budget)
        keep = min(budget, t + 1)
        assert np.array_equal(idx[:, :keep], eidx), f"step {st}"
        assert (idx[:, keep:] == -1).all()
        assert rel_err(out, eout).max() <= TOL[bf16], f"step {st}"
    assert cache.seq_len == S
    assert cache.status() == 0
    return cache


@pytest.mark.parametrize("S,n_kv,G,budget,bf16", [
    (1, 1, 1, 4, False),        # empty cache: the new token is the whole selection
    (2, 1, 1, 1, True),
    (300, 2, 1, 16, False),     # ragged
    (777, 2, 4, 32, True),      # GQA
    (5000, 4, 1, 5000, True),   # budget == S
    (5000, 1, 2, 9000, False),  # budget > S
    (4097, 1, 8, 128, True),
    (32768, 1, 1, 128, False),  # config 0: 1 head, 32K, fp32, budget 128
    (32768, 2, 4, 128, True),   # Llama GQA group at 32K: C x G > 8, two-hop threshold exchange
    (20000, 1, 8, 64, True),    # G = 8 (owners hold several heads when C < G)
])
def test_fused_decode_step_matches_oracle(gpu, oracle, S, n_kv, G, budget, bf16):
    run_decode(gpu, oracle, S, n_kv, G, budget, bf16, seed=S + budget)


def test_fused_decode_multi_step(gpu, oracle):
    run_decode(gpu, oracle, 3000, 2, 2, 64, True, seed=77, steps=5)


@pytest.mark.parametrize("cluster", ["1", "2", "8", "16"])
def test_fused_decode_cluster_sizes(gpu, oracle, tune, cluster):
    tune(cluster=int(cluster))
    run_decode(gpu, oracle, 6000, 2, 1, 128, True, seed=int(cluster))


@pytest.mark.parametrize("qsplit", ["1", "2", "4"])
def test_fused_decode_qsplit(gpu, oracle, tune, qsplit):
    """a kv-head's q-heads split over several clusters (each scans the codes
    for its share); the appended row comes from the input for every part"""
    tune(qsplit=int(qsplit))
    run_decode(gpu, oracle, 9000, 2, 4, 128, True, seed=71 + int(qsplit), steps=3)


@pytest.mark.parametrize("cluster,G", [("2", 4), ("4", 4), ("2", 8)])
def test_fused_decode_exchange_topologies(gpu, oracle, tune, cluster, G):
    """one-hop (C x G <= 8) and two-hop (C x G > 8) histogram exchanges,
    including owners of several heads (G > C)"""
    tune(cluster=int(cluster))
    run_decode(gpu, oracle, 5000, 1, G, 96, True, seed=31 * G + int(cluster), steps=2)


@pytest.mark.parametrize("S,G", [(8000, 1), (16000, 1), (32000, 1), (40000, 1),
                                 (70000, 1), (2000, 4), (4000, 4), (8000, 4), (9000, 4), (20000, 4)])
def test_fused_compaction_span_sizes(gpu, oracle, tune, S, G):
    """one CTA per unit, so the rank length picks the compaction instance:
    16..64-token spans (SW 2), 128-token spans (SW 4), or 32-token groups (SW 0)"""
    tune(cluster=1)
    run_decode(gpu, oracle, S, 1, G, 128, True, seed=S + 13 * G, steps=2)


@pytest.mark.parametrize("S,G", [(16000, 1), (40000, 1), (8000, 4)])
def test_fused_compaction_span_sizes_fp32(gpu, oracle, tune, S, G):
    """the same instances (collected-order masks for 32+-token spans) with fp32 K/V"""
    tune(cluster=1)
    run_decode(gpu, oracle, S, 1, G, 128, False, seed=S + 7 * G, steps=2)


@pytest.mark.parametrize("cluster", ["1", "4"])
def test_fused_decode_heavy_ties(gpu, oracle, tune, cluster):
    """keys drawn from 6 distinct vectors: whole bins of equal distances at T,
    ties taken in index order across spans and ranks (estimator.cpp:75-90)"""
    tune(cluster=int(cluster))
    S, n_kv, G, budget = 6001, 1, 2, 100
    K, V, q = make_inputs(S, n_kv, n_kv * G, True, 4242)
    pick = np.random.default_rng(7).integers(0, 6, S)
    K = K[:6][pick]
    cache = fill_cache(gpu, K[:-1], V[:-1], True, capacity=S + 4)
    out, idx = cache.decode_step(to_dev(q, True), to_dev(K[-1], True), to_dev(V[-1], True), budget)
    _, _, eidx, eout = oracle_decode(oracle, K, V, q, budget)
    assert np.array_equal(idx.cpu().numpy(), eidx)
    assert rel_err(out.cpu().numpy(), eout).max() <= TOL[True]


def test_operator_composition_matches_fused(gpu, oracle, tune):
    tune(composed=1)
    run_decode(gpu, oracle, 2000, 2, 2, 64, False, seed=5, steps=2)


def test_batched_decode_matches_single(gpu, oracle):
    n_seqs, S, n_kv, G, budget = 5, 1500, 2, 2, 48
    caches, qs, ks, vs, exp = [], [], [], [], []
    for i in range(n_seqs):
        K, V, q = make_inputs(S + i * 100, n_kv, n_kv * G, True, 900 + i)
        caches.append(fill_cache(gpu, K[:-1], V[:-1], True, capacity=S + 1000))
        qs.append(q); ks.append(K[-1]); vs.append(V[-1])
        exp.append(oracle_decode(oracle, K, V, q, budget))
    out, idx = gpu.decode_step_batched(caches, to_dev(np.stack(qs), True), to_dev(np.stack(ks), True),
                                       to_dev(np.stack(vs), True), budget)
    out, idx = out.cpu().numpy(), idx.cpu().numpy()
    for i in range(n_seqs):
        assert np.array_equal(idx[i], exp[i][2]), i
        assert rel_err(out[i], exp[i][3]).max() <= 1e-2


@pytest.mark.parametrize("name", sorted(CASES))
def test_cuda_path_reproduces_reference_golden(gpu, golden, name):
    """Bit-exact against vectors produced by the unmodified reference build."""
    S, n_kv, n_q, budget, bf16, seed = (int(v) for v in golden[f"{name}/meta"])
    K, V, q = case_inputs(S, n_kv, n_q, bool(bf16), seed)
    cache = fill_cache(gpu, K[:-1], V[:-1], bool(bf16), capacity=S + 1)
    qd = to_dev(q, bool(bf16))
    out, idx = cache.decode_step(qd, to_dev(K[-1], bool(bf16)), to_dev(V[-1], bool(bf16)), budget)
    words = cache.code_words().cpu().numpy().view(np.uint16)
    assert np.array_equal(words, golden[f"{name}/key_words"])
    assert np.array_equal(cache.encode_query(qd).cpu().numpy().view(np.uint16), golden[f"{name}/q_words"])
    assert np.array_equal(cache.score_all(cache.encode_query(qd)).cpu().numpy(), golden[f"{name}/scores"])
    keep = min(budget, S)
    assert np.array_equal(idx.cpu().numpy()[:, :keep], golden[f"{name}/idx"])
    assert rel_err(out.cpu().numpy(), golden[f"{name}/out"]).max() <= TOL[bool(bf16)]


def test_fused_decode_exact_encode_path(gpu, oracle, tune):
    """The fused kernel's low-latency sigma (shuffle-tree sum with a near-tie
    guard) and the sequential-sum path give identical codes and selections."""
    tune(exact_encode=1)
    run_decode(gpu, oracle, 3000, 2, 4, 64, True, seed=31, steps=3)


def test_fast_encode_near_ties_and_scales(gpu, oracle):
    """Query vectors built to sit on the +/- kQ28 sigma thresholds after the
    transform, plus extreme scales, through the fused decode step."""
    from oracle.bindings import bf16_round
    rng = np.random.default_rng(5)
    S, budget = 600, 32
    K, V, _ = make_inputs(S, 1, 1, False, 41)
    cache = fill_cache(gpu, K[:-1], V[:-1], False, capacity=S + 64)
    H = np.array([[1.0]])
    for _ in range(7):
        H = np.block([[H, H], [H, -H]])
    H /= np.sqrt(128.0)
    for trial in range(24):
        y = rng.standard_normal(128)
        sigma = np.sqrt(np.mean(y * y))
        y[trial % 128] = 0.6744897501960817 * sigma * (1 if trial % 2 else -1)
        q = (H @ y).astype(np.float32) * np.float32(10.0 ** ((trial % 9) - 4))
        q = q.reshape(1, 128)
        out, idx = cache.decode_step(to_dev(q, False), to_dev(K[-1], False), to_dev(V[-1], False), budget)
        Kt = np.concatenate([K[:-1], K[-1:]])  # cache + appended token
        _, _, eidx, eout = oracle_decode(oracle, Kt, np.concatenate([V[:-1], V[-1:]]), q, budget)
        assert np.array_equal(idx.cpu().numpy(), eidx), trial
        cache.truncate(S - 1)


@pytest.mark.parametrize("cluster", ["1", "4"])
def test_uncertified_appended_key(gpu, oracle, tune, cluster):
    """Appended keys built to sit on the +/- kQ28 sigma thresholds (the fp32
    certificate fails): the fused step takes the exact code (at G = 1 from the
    helper warp, after the scan), stores it in the cache and selects with it."""
    tune(cluster=int(cluster))
    rng = np.random.default_rng(9)
    S, budget = 3000, 64
    K, V, q = make_inputs(S, 1, 1, False, 43)
    H = np.array([[1.0]])
    for _ in range(7):
        H = np.block([[H, H], [H, -H]])
    H /= np.sqrt(128.0)
    cache = fill_cache(gpu, K[:-1], V[:-1], False, capacity=S + 64)
    for trial in range(12):
        y = rng.standard_normal(128)
        sigma = np.sqrt(np.mean(y * y))
        y[(5 * trial) % 128] = 0.6744897501960817 * sigma * (1 if trial % 2 else -1)
        k = (H @ y).astype(np.float32).reshape(1, 1, 128)
        # the query close to the key, so the appended token competes for the selection
        qq = (k[0] + 0.05 * rng.standard_normal((1, 128))).astype(np.float32)
        out, idx = cache.decode_step(to_dev(qq, False), to_dev(k[0], False), to_dev(V[-1], False), budget)
        Kt = np.concatenate([K[:-1], k])
        Vt = np.concatenate([V[:-1], V[-1:]])
        _, _, eidx, eout = oracle_decode(oracle, Kt, Vt, qq, budget)
        assert np.array_equal(idx.cpu().numpy(), eidx), trial
        assert rel_err(out.cpu().numpy(), eout).max() <= TOL[False], trial
        words = cache.code_words().cpu().numpy().view(np.uint16)
        assert np.array_equal(words[0][S - 1], oracle.encode_pack_rows(k[:, 0].astype(np.float64))[0]), trial
        assert cache.status() == 0
        cache.truncate(S - 1)


@pytest.mark.parametrize("metric,bits,ref_metric", [("euclidean_sq", 2, 1), ("hamming_1bit", 1, 0)])
def test_ablation_metrics_match_reference(gpu, reference, metric, bits, ref_metric):
    """Metric::euclidean_sq over 2-bit codes and the 1-bit
    pipeline's L1, from the same device cache, bit-exact against the
    unmodified reference's score_all."""
    S, n_kv, G = 1000, 1, 2
    K, V, q = make_inputs(S, n_kv, n_kv * G, False, 23)
    cache = fill_cache(gpu, K, V, False)
    qw = cache.encode_query(to_dev(q, False))
    got = cache.score_all(qw, metric=metric).cpu().numpy()
    for h in range(n_kv * G):
        exp = reference.score_all_metric(K[:, h // G], q[h], bits, ref_metric)
        assert np.array_equal(got[h], exp), h


def test_decode_errors_mirror_the_reference(gpu):
    """ConfigError classes of the reference preconditions (common.hpp:19-22)."""
    cache = gpu.KvCache(2, 3, torch.bfloat16)
    kv = torch.randn((2, 128), device="cuda").bfloat16()
    q3 = torch.randn((3, 128), device="cuda").bfloat16()
    with pytest.raises(gpu.ConfigError):  # q-heads not a multiple of kv-heads
        cache.decode_step(q3, kv, kv, 8)
    q = torch.randn((4, 128), device="cuda").bfloat16()
    with pytest.raises(gpu.ConfigError):  # empty selection (attention.cpp:42)
        cache.decode_step(q, kv, kv, 0)
    for _ in range(3):
        cache.decode_step(q, kv, kv, 8)
    with pytest.raises(gpu.ConfigError):  # capacity exhausted
        cache.decode_step(q, kv, kv, 8)
    with pytest.raises(gpu.ConfigError):  # dtype mismatch
        gpu.KvCache(2, 8, torch.float32).decode_step(q, kv, kv, 8)


def test_degenerate_query_latches_status_in_fused_step(gpu, oracle):
    S = 300
    K, V, _ = make_inputs(S, 1, 1, True, 61)
    cache = fill_cache(gpu, K[:-1], V[:-1], True, capacity=S + 2)
    assert cache.status() == 0
    z = torch.zeros((1, 128), device="cuda").bfloat16()
    cache.decode_step(z, to_dev(K[-1], True), to_dev(V[-1], True), 16)
    with pytest.raises(gpu.ConfigError):  # quantizer.cpp:46-47: zero vector
        cache.raise_on_degenerate()


def test_seq_shard_empty_rank_and_errors(gpu, oracle):
    from paper_2510_18413_b200.seqshard import CudaSeqOps
    ops = CudaSeqOps()
    c = gpu.KvCache(1, 8, torch.bfloat16)
    q = torch.randn((2, 128), device="cuda").bfloat16()
    keys = ops.local_candidates(c, q, None, None, False, 0, 16)  # empty shard: no candidates
    assert (keys.cpu().numpy().view(np.uint32) == 0xFFFFFFFF).all()
    g = torch.stack([keys, keys])
    with pytest.raises(gpu.ConfigError):  # n_ranks * budget > 8192
        ops.select_attend(c, q, torch.stack([keys] * 2).repeat(1, 1, 300)[:, :, :4800], 4800, 10, 0)
    part, gidx = ops.select_attend(c, q, g, 16, 1, 0, want_idx=True)  # nothing selected here
    assert (gidx.cpu().numpy() == -1).all() and (part[:, 1].cpu().numpy() == 0).all()


@pytest.mark.parametrize("P,C,n_kv,G,steps", [(2, 4, 1, 1, 3), (4, 4, 2, 4, 2), (4, 2, 1, 2, 2), (8, 4, 1, 8, 1)])
def test_fused_decode_multi_cluster_units(gpu, oracle, tune, P, C, n_kv, G, steps):
    """A unit spanning P clusters: histograms and partials through global
    memory with the self-resetting barrier (reused across consecutive steps)."""
    tune(P=P, cluster=C, require_fused=1)
    cache = run_decode(gpu, oracle, 12000, n_kv, G, 128, True, seed=P * 10 + G, steps=steps)
    assert cache.status() == 0  # no barrier timeout


def test_seq_shard_candidates_multi_cluster(gpu, oracle, tune):
    tune(P=4, cluster=4)
    from tests.test_gpu_seqshard import test_seq_sharded_decode_matches_single_device as t
    t(gpu, oracle, 20000, 2, 2, 4, 128, True)
