"""-m gpu: f3, the GPU backend for the sweep harness, against
the unmodified reference (oracle/_ref): codes, selections, dot / page top-k
bit-exact; fp64 attention to 1e-12 relative; run_sweep's CSV / JSON / needle
summary byte-identical (output_error to 1e-13 absolute), including the
reference's own needle pin (tests/test_sweep.cpp:115-155)."""
import json

import numpy as np
import pytest
import torch

from paper_2510_18413_b200 import harness as H
from paper_2510_18413_b200._lib import ConfigError

pytestmark = pytest.mark.gpu
DIMS = [2, 4, 8, 16, 32, 64, 128, 256, 1024]


def keys_for(d, S, seed, outliers=True):
    rng = np.random.default_rng(seed)
    K = rng.standard_normal((S, d))
    if outliers and d >= 8:
        K[:, rng.choice(d, max(1, d // 16), replace=False)] *= 10.0  # gaussian_with_outliers-like channels
    K[1] *= 1e-140  # scale extremes (sigma stays finite and nonzero)
    K[2] *= 1e150
    return K


def ref_instances(reference, spec):
    """Workload(spec).instance(qi) for every query, sharing key/value arrays by
    identity where the reference shares them (workload.hpp:69-80)."""
    out, shared = [], None
    for qi in range(spec.num_queries):
        seed, q, K, V, needle = reference.workload_instance(spec, qi)
        if spec.distribution != "planted_needle":
            if shared is None:
                shared = (K, V)
            K, V = shared
        out.append(H.Instance(seed, q, K, V, needle))
    return out


@pytest.mark.parametrize("bits", [1, 2, 3])
@pytest.mark.parametrize("had", [True, False])
@pytest.mark.parametrize("d", DIMS)
def test_codes_bit_exact(gpu, reference, d, bits, had):
    S = 48
    K = keys_for(d, S, d * 10 + bits)
    q = np.random.default_rng(d).standard_normal(d)
    _, kc, qc = reference.adamas_select(q, K, bits, 0, had, 8, want_codes=True)
    sel = H.HarnessSelector(d, bits, had)
    sel.build(torch.as_tensor(K, device="cuda"))
    got = sel.codes_ref().cpu().numpy()
    exp = kc if bits == 3 else kc.view(np.uint16)
    assert np.array_equal(got.view(exp.dtype).reshape(exp.shape), exp)


@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("bits", [1, 2, 3])
@pytest.mark.parametrize("had", [True, False])
@pytest.mark.parametrize("d", [2, 8, 32, 128, 512])
def test_select_bit_exact(gpu, reference, d, bits, had, metric):
    """score_all + top_k (estimator.cpp:45-90) incl. heavy ties at small d."""
    S, nq = 300, 5
    rng = np.random.default_rng(1000 + d * 7 + bits)
    K = keys_for(d, S, d + 3 * bits)
    Q = rng.standard_normal((nq, d))
    sel = H.HarnessSelector(d, bits, had)
    sel.build(torch.as_tensor(K, device="cuda"))
    for budget in [1, 7, 64, S - 1, S, S + 5]:
        got = sel.select(torch.as_tensor(Q, device="cuda"), budget, ["l1", "l2"][metric], rows_per_inst=nq)
        got = got.cpu().numpy()
        for r in range(nq):
            exp = reference.adamas_select(Q[r], K, bits, metric, had, budget)
            n = min(budget, S)
            assert np.array_equal(got[r, :n], exp), (budget, r)
            assert (got[r, n:] == -1).all()


def test_select_many_instances(gpu, reference):
    """needle-style batching: one key matrix per query row (rows_per_inst = 1)."""
    d, S, n = 32, 200, 6
    rng = np.random.default_rng(5)
    K = rng.standard_normal((n, S, d))
    Q = rng.standard_normal((n, d))
    sel = H.HarnessSelector(d, 2, True)
    sel.build(torch.as_tensor(K, device="cuda"))
    got = sel.select(torch.as_tensor(Q, device="cuda"), 16, "l1", rows_per_inst=1).cpu().numpy()
    for r in range(n):
        assert np.array_equal(got[r], reference.adamas_select(Q[r], K[r], 2, 0, True, 16))


def test_degenerate_vectors_raise(gpu):
    d = 64
    sel = H.HarnessSelector(d, 2, True)
    K = np.random.default_rng(0).standard_normal((10, d))
    K[4] = 0.0
    with pytest.raises(ConfigError, match="degenerate scale"):
        sel.build(torch.as_tensor(K, device="cuda"))
    K[4] = 1.0
    K[5, 3] = np.nan
    with pytest.raises(ConfigError, match="non-finite"):
        sel.build(torch.as_tensor(K, device="cuda"))
    K[5, 3] = 0.5
    K[6] *= 1e-170  # squares underflow: sigma == 0 in the reference too
    with pytest.raises(ConfigError, match="degenerate scale"):
        sel.build(torch.as_tensor(K, device="cuda"))
    K[6] *= 1e170
    sel.build(torch.as_tensor(K, device="cuda"))
    with pytest.raises(ConfigError, match="degenerate scale"):
        sel.select(torch.zeros((1, d), dtype=torch.float64, device="cuda"), 4, "l1", 1)
    with pytest.raises(ConfigError):
        H.HarnessSelector(48, 2, True)
    with pytest.raises(ConfigError):
        H.HarnessSelector(64, 4, True)


def test_dot_topk_bit_exact(gpu, reference):
    d, S, nq = 64, 1000, 4
    rng = np.random.default_rng(9)
    K = rng.standard_normal((S, d))
    K[100:110] = K[5]  # exact ties -> smaller index first
    Q = rng.standard_normal((nq, d))
    Q[3] = 0.0  # every score +-0.0: the first k indices
    Kd = torch.as_tensor(K[None], device="cuda")
    for k in [1, 16, 999, 1000, 1200]:
        idx, sc = H.dot_topk(torch.as_tensor(Q, device="cuda"), Kd, k, rows_per_inst=nq, want_scores=True)
        idx = idx.cpu().numpy()
        sc = sc.cpu().numpy()
        for r in range(nq):
            exp = reference.top_k_by_score(sc[r], k)
            assert np.array_equal(idx[r, :min(k, S)], exp), (k, r)
    # the dot scores themselves follow dot() (common.hpp:65-69) bit for bit
    for r in range(nq):
        acc = np.zeros(S)
        for j in range(d):
            acc = acc + Q[r, j] * K[:, j]
        assert np.array_equal(sc[r], acc)


@pytest.mark.parametrize("page", [1, 16, 24])
def test_page_select_bit_exact(gpu, reference, page):
    d, S, nq = 32, 1000, 3  # 1000 % 16 and % 24 != 0: a partial last page
    rng = np.random.default_rng(page)
    K = rng.standard_normal((S, d))
    Q = rng.standard_normal((nq, d))
    for budget in [page, 4 * page, 20 * page, S, S + 3]:
        idx, cnt = H.page_select(torch.as_tensor(Q, device="cuda"), torch.as_tensor(K[None], device="cuda"), page,
                                 budget, rows_per_inst=nq)
        idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
        for r in range(nq):
            exp = reference.page_select(Q[r], K, page, budget)
            assert cnt[r] == exp.size
            assert np.array_equal(idx[r, :cnt[r]], exp)
    with pytest.raises(ConfigError):
        H.page_select(torch.as_tensor(Q, device="cuda"), torch.as_tensor(K[None], device="cuda"), 16, 20, nq)


def test_attention_f64(gpu, reference):
    d, S, nq = 128, 700, 3
    rng = np.random.default_rng(3)
    K, V, Q = rng.standard_normal((S, d)), rng.standard_normal((S, d)), rng.standard_normal((nq, d)) * 3
    Kd, Vd = torch.as_tensor(K[None], device="cuda"), torch.as_tensor(V[None], device="cuda")
    Qd = torch.as_tensor(Q, device="cuda")
    full = H.attention_f64(Qd, Kd, Vd, rows_per_inst=nq).cpu().numpy()
    idx = torch.as_tensor(np.tile(np.arange(0, S, 3), (nq, 1)), device="cuda")
    part = H.attention_f64(Qd, Kd, Vd, nq, idx).cpu().numpy()
    # acceptance.cpp:155-205: sparse over the full set == dense (here bit for
    # bit: same kernel, same order), a singleton selection returns its value row
    every = torch.as_tensor(np.tile(np.arange(S), (nq, 1)), device="cuda")
    assert np.array_equal(H.attention_f64(Qd, Kd, Vd, nq, every).cpu().numpy(), full)
    one = torch.as_tensor(np.array([[5], [77], [699]]), device="cuda")
    assert np.array_equal(H.attention_f64(Qd, Kd, Vd, nq, one).cpu().numpy(), V[[5, 77, 699]])
    for r in range(nq):
        e = reference.full_attention(Q[r], K, V)
        assert np.abs(full[r] - e).max() <= 1e-12 * np.abs(e).max()
        e2 = reference.full_attention(Q[r], K[::3], V[::3])
        assert np.abs(part[r] - e2).max() <= 1e-12 * np.abs(e2).max()


def _err_close(a, b):
    """output_error = |approx - exact| / |exact| is a difference of two fp64
    attention outputs, each off the reference's by ~1e-16 relative (device
    exp()): the error value agrees to ~1e-15 ABSOLUTE, however small it is."""
    return abs(a - b) <= 1e-13 + 1e-9 * abs(b)


def _compare_csv(got, exp):
    g, e = got.splitlines(), exp.splitlines()
    assert len(g) == len(e) and g[0] == e[0]
    for a, b in zip(g[1:], e[1:]):
        fa, fb = a.split(","), b.split(",")
        assert fa[:4] == fb[:4] and fa[5:] == fb[5:], (a, b)
        if fa[4] != fb[4]:
            assert _err_close(float(fa[4]), float(fb[4])), (a, b)


def test_needle_pin(gpu, reference):
    """tests/test_sweep.cpp:115-155, selections on the GPU."""
    spec = H.WorkloadSpec(seed=5, seq_len=128, head_dim=32, num_queries=6, distribution="planted_needle",
                          position=60)
    sweep = H.SweepConfig(budgets=[16], policies=[H.PolicySpec("adamas"), H.PolicySpec("window", sink=4),
                                                  H.PolicySpec("oracle")])
    rows = H.run_sweep(ref_instances(reference, spec), sweep)
    assert all(r.needle_hit is not None for r in rows)
    summary = H.needle_report(rows)
    assert H.needle_summary_to_csv(summary) == ("policy,budget,needle_fraction,queries\n"
                                                "adamas-2bit-l1,16,1.0,6\n"
                                                "window-sink4,16,0.0,6\n"
                                                "oracle,16,1.0,6\n")
    csv, js, nd = reference.run_sweep(spec, sweep)
    _compare_csv(H.rows_to_csv(rows), csv)
    assert nd == H.needle_summary_to_csv(summary)


ALL_POLICIES = [H.PolicySpec("adamas"), H.PolicySpec("adamas", metric="l2"), H.PolicySpec("adamas", bits=1),
                H.PolicySpec("adamas", bits=3), H.PolicySpec("adamas", bits=3, metric="l2"),
                H.PolicySpec("adamas", with_hadamard=False), H.PolicySpec("window", sink=4),
                H.PolicySpec("quest", page_size=16), H.PolicySpec("oracle")]


@pytest.mark.parametrize("dist", ["gaussian", "gaussian_with_outliers", "planted_needle"])
@pytest.mark.parametrize("measure", [True, False])
def test_run_sweep_matches_reference(gpu, reference, dist, measure):
    spec = H.WorkloadSpec(seed=11, seq_len=500, head_dim=64, num_queries=5, distribution=dist, position=200)
    sweep = H.SweepConfig(budgets=[16, 32, 64, 512], policies=ALL_POLICIES, measure_output_error=measure)
    rows = H.run_sweep(ref_instances(reference, spec), sweep)
    csv, js, nd = reference.run_sweep(spec, sweep)
    got_csv, got_js = H.rows_to_csv(rows), H.rows_to_json(rows)
    if measure:
        _compare_csv(got_csv, csv)
        for a, b in zip(json.loads(got_js), json.loads(js)):
            ea, eb = a.pop("output_error"), b.pop("output_error")
            assert a == b and _err_close(ea, eb)
    else:
        assert got_csv == csv
        assert got_js == js
    if dist == "planted_needle":
        assert H.needle_summary_to_csv(H.needle_report(rows)) == nd


def test_acceptance_needle_criterion(gpu, reference):
    """acceptance.cpp:290-325 at 100 of its 1000 queries (the full criterion
    runs in tools/harness_bench.py): adamas needle fraction >= 0.9 at budget 64,
    window <= 0.05, adamas >= quest at 16 and 32; and the rows equal the
    reference's."""
    spec = H.WorkloadSpec(seed=2024, seq_len=8192, head_dim=128, num_queries=100, distribution="planted_needle",
                          position=4096, snr=10.0)
    sweep = H.SweepConfig(budgets=[16, 32, 64], policies=[H.PolicySpec("adamas"), H.PolicySpec("window", sink=4),
                                                          H.PolicySpec("quest", page_size=16)],
                          measure_output_error=False)
    rows = H.run_sweep(ref_instances(reference, spec), sweep)
    frac = {(c.policy, c.budget): c.needle_fraction for c in H.needle_report(rows)}
    assert frac[("adamas-2bit-l1", 64)] >= 0.9
    assert all(frac[("window-sink4", b)] <= 0.05 for b in (16, 32, 64))
    assert all(frac[("adamas-2bit-l1", b)] >= frac[("quest-p16", b)] for b in (16, 32))
    csv, _, nd = reference.run_sweep(spec, sweep)
    assert H.rows_to_csv(rows) == csv
    assert H.needle_summary_to_csv(H.needle_report(rows)) == nd


def test_select_many_rows_chunked(gpu, reference):
    """More query rows than one launch's grid holds: chunks of whole instances."""
    d, S, n_inst, rpi = 16, 40, 700, 100  # 70000 rows
    rng = np.random.default_rng(77)
    K = rng.standard_normal((n_inst, S, d))
    Q = rng.standard_normal((n_inst * rpi, d))
    sel = H.HarnessSelector(d, 2, True)
    sel.build(torch.as_tensor(K, device="cuda"))
    got = sel.select(torch.as_tensor(Q, device="cuda"), 5, "l1", rows_per_inst=rpi).cpu().numpy()
    for r in [0, 1, 32767, 32768, 32800, 69999]:
        assert np.array_equal(got[r], reference.adamas_select(Q[r], K[r // rpi], 2, 0, True, 5)), r


def test_acceptance_ablation_criterion(gpu, reference):
    """acceptance.cpp:346-413 (all 120 seeds) with every selection on the GPU:
    the Hadamard transform helps significantly, 3 >= 2 >= 1 bits up to noise,
    diminishing returns from 2 to 3 bits; rows equal the reference's."""
    seeds, z95, budgets = 120, 1.645, [16, 64, 256]
    sweep = H.SweepConfig(budgets=budgets, policies=[H.PolicySpec("adamas", bits=2),
                                                     H.PolicySpec("adamas", bits=2, with_hadamard=False),
                                                     H.PolicySpec("adamas", bits=1), H.PolicySpec("adamas", bits=3)],
                          measure_output_error=False)
    specs = [H.WorkloadSpec(seed=9000 + s, seq_len=2048, head_dim=128, num_queries=1,
                            distribution="gaussian_with_outliers", outlier_frac=0.01, outlier_scale=10.0)
             for s in range(seeds)]
    insts = [ref_instances(reference, sp)[0] for sp in specs]
    rows = H.run_sweep(insts, sweep)  # one batched sweep: instance s = seed s
    n_cells = len(sweep.policies) * len(budgets)
    assert len(rows) == n_cells * seeds
    rec = np.array([r.recall for r in rows]).reshape(len(sweep.policies), len(budgets), seeds)
    for s in range(3):  # per-seed rows equal the reference's own sweep
        csv, _, _ = reference.run_sweep(specs[s], sweep)
        mine = [rows[c * seeds + s] for c in range(n_cells)]
        assert H.rows_to_csv(mine) == csv

    def paired(a, b):
        d = a - b
        return d.mean(), np.sqrt(d.var(ddof=1) / d.size)

    for bi in range(len(budgets)):
        with2, without2, with1, with3 = rec[0, bi], rec[1, bi], rec[2, bi], rec[3, bi]
        m, se = paired(with2, without2)
        assert m > z95 * se, ("transform gain not significant", budgets[bi], m, se)
        m, se = paired(with3, with2)
        assert m > -z95 * se, ("3-bit below 2-bit", budgets[bi])
        m, se = paired(with2, with1)
        assert m > -z95 * se, ("2-bit below 1-bit", budgets[bi])
        m, se = paired((with3 - with2) - (with2 - with1), np.zeros(seeds))
        assert m < z95 * se, ("no diminishing returns", budgets[bi], m)
