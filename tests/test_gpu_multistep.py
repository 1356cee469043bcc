"""-m gpu: many consecutive fused decode steps on one cache with queries whose
threshold jumps from step to step (random queries, queries close to a cached
key, back to random), heavy ties, budgets above the length, and the rank
lengths that need ring refills (more stages than the ring holds). Every step's
selection must equal the reference's top_k (estimator.cpp:75-90) exactly.

These cases exposed a barrier bug during development: an aligned bar.sync
reached by a diverged warp released the consumer warps early and the tie
count below T came out wrong under skewed warps (fixed by converging each warp
before the named barrier, fused_decode.cuh consumer_sync)."""
import numpy as np
import pytest
import torch

from oracle.bindings import bf16_round
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
    T drops far below the previous step's) and back (T jumps up)"""
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
            q = bf16_round(q)
        qs.append(q.astype(np.float32))
    return qs


@pytest.mark.parametrize("S,n_kv,G,budget,cluster,stages", [
    (20000, 2, 1, 128, 4, 0), (12000, 2, 4, 64, 2, 0), (9000, 1, 2, 200, 1, 0),
    (8000, 2, 1, 64, 1, 2),    # 8 stages through a 2-slot ring
    (24000, 2, 1, 64, 4, 2),
    (12000, 2, 2, 64, 1, 3),
])
def test_multistep_mixed_queries(gpu, oracle, tune, S, n_kv, G, budget, cluster, stages):
    tune(cluster=cluster, stages=stages)
    steps = 7
    K, V, _ = make_inputs(S + steps, n_kv, n_kv * G, True, S + 3)
    qs = _mixed_queries(K, n_kv * G, n_kv, steps, True, S + G)
    _steps(gpu, oracle, K, V, qs, budget, True)


@pytest.mark.parametrize("cluster", [1, 4])
def test_multistep_dense_ties(gpu, oracle, tune, cluster):
    """keys from 4 distinct vectors: thousands of tokens share each distance"""
    tune(cluster=cluster)
    S, n_kv, G, budget, steps = 8000, 1, 2, 100, 4
    K, V, _ = make_inputs(S + steps, n_kv, n_kv * G, False, 77)
    pick = np.random.default_rng(3).integers(0, 4, S + steps)
    K = K[:4][pick]
    qs = [make_inputs(1, 1, n_kv * G, False, 500 + st)[2] for st in range(steps)]
    _steps(gpu, oracle, K, V, qs, budget, False)


def test_multistep_budget_above_length(gpu, oracle, tune):
    tune(cluster=1)
    S, n_kv, G, budget, steps = 300, 1, 1, 512, 4
    K, V, _ = make_inputs(S + steps, n_kv, n_kv * G, True, 5)
    qs = [make_inputs(1, 1, n_kv * G, True, 900 + st)[2] for st in range(steps)]
    _steps(gpu, oracle, K, V, qs, budget, True)
