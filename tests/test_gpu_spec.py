"""-m gpu: the speculative-threshold path of the fused decode step.

From its second step on, a cache lists only the tokens at distance <= Tg (the
q-head's previous threshold T plus a margin) during the scan; if T moved above
Tg or a list overflowed, the unit falls back to the full-row selection. Either
way the selection must equal the reference's top_k (estimator.cpp:75-90)
exactly. These tests drive hits, misses (T jumping up), T jumping down, list
overflow (dense ties) and the margin settings over many consecutive steps."""
import numpy as np
import pytest
import torch

from tests.gpu_helpers import make_inputs, oracle_decode, rel_err, to_dev

pytestmark = pytest.mark.gpu
TOL = {False: 1e-3, True: 1e-2}


def _steps(gpu, oracle, K, V, qs, budget, bf16):
    S_total, n_kv, _ = K.shape
    steps = len(qs)
    pre = S_total - steps
    cache = gpu.KvCache(n_kv, S_total + 4, torch.bfloat16 if bf16 else torch.float32)
    cache.update(to_dev(K[:pre], bf16), to_dev(V[:pre], bf16))
    for st, q in enumerate(qs):
        t = pre + st
        out, idx = cache.decode_step(to_dev(q, bf16), to_dev(K[t], bf16), to_dev(V[t], bf16), budget)
        _, _, eidx, eout = oracle_decode(oracle, K[:t + 1], V[:t + 1], q, budget)
        keep = min(budget, t + 1)
        got = idx.cpu().numpy()
        assert np.array_equal(got[:, :keep], eidx), f"step {st}: heads {np.nonzero((got[:, :keep] != eidx).any(1))[0]}"
        assert (got[:, keep:] == -1).all()
        assert rel_err(out.cpu().numpy(), eout).max() <= TOL[bf16], f"step {st}"
    cache.raise_on_status()
    return cache


def _mixed_queries(K, n_q, n_kv, steps, bf16, seed):
    """random queries, interleaved with queries close to a cached key (their
    T drops far below the previous step's) and back (T jumps above Tg)"""
    rng = np.random.default_rng(seed)
    G = n_q // n_kv
    qs = []
    for st in range(steps):
        q = make_inputs(1, 1, n_q, bf16, seed * 100 + st)[2].copy()
        if st % 3 == 1:
            for h in range(n_q):
                src = K[rng.integers(0, K.shape[0] - steps), h // G]
                q[h] = src + 0.05 * q[h]
        if bf16:
            from oracle.bindings import bf16_round
            q = bf16_round(q)
        qs.append(q.astype(np.float32))
    return qs


@pytest.mark.parametrize("margin", [-1, 0, 2, 6, 40])
@pytest.mark.parametrize("S,n_kv,G,budget,cluster", [(20000, 2, 1, 128, 4), (12000, 2, 4, 64, 2), (9000, 1, 2, 200, 1)])
def test_spec_mixed_steps(gpu, oracle, tune, margin, S, n_kv, G, budget, cluster):
    tune(spec_margin=margin, cluster=cluster)
    steps = 9
    K, V, _ = make_inputs(S + steps, n_kv, n_kv * G, True, S + margin + 3)
    qs = _mixed_queries(K, n_kv * G, n_kv, steps, True, S + G)
    cache = _steps(gpu, oracle, K, V, qs, budget, True)
    listed, fallback = cache.spec_stats()
    if margin < 0:
        assert listed == 0
    elif margin in (2, 6):
        assert listed > 0, (listed, fallback)  # random steps after random steps hit


@pytest.mark.parametrize("cluster", [1, 4])
def test_spec_list_overflow_dense_ties(gpu, oracle, tune, cluster):
    """keys from 4 distinct vectors: thousands of tokens share each distance,
    so the candidate lists overflow on every step after the first"""
    tune(cluster=cluster)
    S, n_kv, G, budget, steps = 8000, 1, 2, 100, 4
    K, V, _ = make_inputs(S + steps, n_kv, n_kv * G, False, 77)
    pick = np.random.default_rng(3).integers(0, 4, S + steps)
    K = K[:4][pick]
    qs = [make_inputs(1, 1, n_kv * G, False, 500 + st)[2] for st in range(steps)]
    _steps(gpu, oracle, K, V, qs, budget, False)


def test_spec_budget_above_length(gpu, oracle, tune):
    """budget > S: T is the largest distance, far above any guess"""
    tune(cluster=1)
    S, n_kv, G, budget, steps = 300, 1, 1, 512, 4
    K, V, _ = make_inputs(S + steps, n_kv, n_kv * G, True, 5)
    qs = [make_inputs(1, 1, n_kv * G, True, 900 + st)[2] for st in range(steps)]
    _steps(gpu, oracle, K, V, qs, budget, True)


def test_spec_repeated_query_hits(gpu, oracle, tune):
    """the same query every step: T stays put and every step after the first
    takes the listed path (margin 0: Tg == T)"""
    tune(spec_margin=0, cluster=4)
    S, n_kv, G, budget, steps = 16000, 2, 1, 128, 5
    K, V, _ = make_inputs(S + steps, n_kv, n_kv * G, True, 31)
    q = make_inputs(1, 1, n_kv * G, True, 32)[2]
    cache = _steps(gpu, oracle, K, V, [q] * steps, budget, True)
    listed, fallback = cache.spec_stats()
    assert fallback == n_kv and listed == n_kv * (steps - 1), (listed, fallback)  # only the first step falls back
