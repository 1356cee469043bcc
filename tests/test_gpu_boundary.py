"""-m gpu: the operator boundary keeps the reference's contracts.

top_k accepts any int32 score (DistanceScores = std::vector<int32_t>,
estimator.hpp:20; top_k, estimator.cpp:75-90), and sparse_attention rejects
what KvCache::gather rejects (out-of-range or non-increasing indices,
kv_cache.cpp:90-91) and the empty selection (attention.cpp:42) with
ConfigError, reading nothing out of range."""
import numpy as np
import pytest
import torch

from tests.gpu_helpers import make_inputs, to_dev

pytestmark = pytest.mark.gpu


def _ref_top_k(s, k):
    """The k smallest under (score, index), ascending indices (estimator.cpp:78-88)."""
    order = np.lexsort((np.arange(len(s)), s))
    return np.sort(order[:min(k, len(s))])


@pytest.mark.parametrize("n,k", [(2, 1), (1000, 64), (1000, 999), (33000, 128), (70000, 2048)])
def test_top_k_any_int32(gpu, oracle, n, k):
    rng = np.random.default_rng(n * 7 + k)
    rows = [
        rng.integers(1024, 70000, n),                       # beyond the 2-bit distance range
        rng.integers(-500, 500, n),                         # negative scores
        rng.integers(-2**31, 2**31 - 1, n, dtype=np.int64),  # the whole int32 range
        rng.integers(-2**31, -2**31 + 3, n, dtype=np.int64),  # dense ties at INT32_MIN
        np.concatenate([np.full(n - 1, 2**31 - 1), [-2**31]]),  # extremes
        rng.integers(0, 1153, n),                           # euclidean_sq range (9 * 128)
    ]
    s = np.stack(rows).astype(np.int32)
    got = gpu.top_k(torch.from_numpy(s).cuda(), k).cpu().numpy()
    for r in range(s.shape[0]):
        exp = oracle.top_k(s[r], k)
        assert np.array_equal(exp, _ref_top_k(s[r], k))
        assert np.array_equal(got[r, :len(exp)], exp), r
        assert (got[r, len(exp):] == -1).all()


def test_top_k_reference_examples(gpu):
    t = lambda v, k: list(gpu.top_k(torch.tensor(v, dtype=torch.int32).cuda(), k)[0].cpu())  # noqa: E731
    assert t([2000, 1500], 1) == [1]
    assert t([-3, 5, -3, 9], 2) == [0, 2]
    assert t([70000, 65536, 65535], 2) == [1, 2]


def test_top_k_euclidean_scores(gpu, oracle):
    """score_all(q, cache, euclidean_sq) reaches 1152; its top-k near k = n."""
    S, n_kv, G = 3000, 1, 2
    K, V, q = make_inputs(S, n_kv, n_kv * G, True, 99)
    cache = gpu.KvCache(n_kv, S + 8, torch.bfloat16)
    cache.update(to_dev(K, True), to_dev(V, True))
    qw = cache.encode_query(to_dev(q, True))
    sc = cache.score_all(qw, metric="euclidean_sq")
    for k in (128, S - 3, S):
        got = gpu.top_k(sc, k).cpu().numpy()
        s = sc.cpu().numpy()
        for r in range(s.shape[0]):
            assert np.array_equal(got[r, :min(k, S)], oracle.top_k(s[r], k))


@pytest.mark.parametrize("bad", ["out_of_range", "negative", "unsorted", "duplicate", "empty", "hole"])
def test_sparse_attention_rejects_bad_gather(gpu, bad):
    S, n_kv, G = 500, 2, 2
    K, V, q = make_inputs(S, n_kv, n_kv * G, True, 5)
    cache = gpu.KvCache(n_kv, S + 8, torch.bfloat16)
    cache.update(to_dev(K, True), to_dev(V, True))
    idx = np.tile(np.arange(0, 40, 2, dtype=np.int32), (n_kv * G, 1))
    row = idx[3]
    if bad == "out_of_range":
        row[-1] = S  # == seq_len: past the cache (capacity is larger)
    elif bad == "negative":
        row[5] = -7
    elif bad == "unsorted":
        row[4], row[5] = row[5], row[4]
    elif bad == "duplicate":
        row[6] = row[5]
    elif bad == "empty":
        row[:] = -1
    elif bad == "hole":  # an index after a -1 terminator
        row[10] = -1
    with pytest.raises(gpu.ConfigError):
        cache.sparse_attention(to_dev(q, True), torch.from_numpy(idx).cuda())
    # the status was consumed: a valid call afterwards succeeds
    ok = np.tile(np.arange(0, 40, 2, dtype=np.int32), (n_kv * G, 1))
    out = cache.sparse_attention(to_dev(q, True), torch.from_numpy(ok).cuda())
    assert torch.isfinite(out).all()


def test_sparse_attention_terminated_rows_ok(gpu):
    """-1 entries after a non-empty increasing prefix end the row (budget > S)."""
    S, n_kv = 300, 1
    K, V, q = make_inputs(S, n_kv, 1, False, 8)
    cache = gpu.KvCache(n_kv, S + 8, torch.float32)
    cache.update(to_dev(K, False), to_dev(V, False))
    idx = np.full((1, 16), -1, dtype=np.int32)
    idx[0, :3] = [0, 7, S - 1]
    out = cache.sparse_attention(to_dev(q, False), torch.from_numpy(idx).cuda())
    assert torch.isfinite(out).all()
