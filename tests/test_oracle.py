"""CPU: the C restatement (oracle/) pinned against the reference's own known
answers (proj/tests/*.cpp) and against the reference build (oracle/_ref) and
its golden vectors (tests/golden/)."""
import hashlib

import numpy as np
import pytest

from oracle.bindings import bf16_round, synth
from tests.golden.make_golden import CASES, case_inputs


def test_synth_is_bit_identical_between_numpy_and_c(oracle):
    for seed, first, n in [(0, 0, 1000), (7, 12345, 4096), (2**63 + 5, 2**40, 257)]:
        assert np.array_equal(synth(seed, first, n), oracle.synth(seed, first, n))
    x = synth(99, 0, 1 << 16)
    assert abs(float(x.mean())) < 0.02 and 0.95 < float(x.std()) < 1.05


def test_fwht_hand_values(oracle):  # test_hadamard.cpp:25-42
    a = oracle.fwht([1.0, 0.0])
    assert a[0] == pytest.approx(0.70710678, rel=1e-8) and a[1] == pytest.approx(0.70710678, rel=1e-8)
    assert np.allclose(oracle.fwht([1.0, 1.0, 1.0, 1.0]), [2.0, 0.0, 0.0, 0.0])
    c = oracle.fwht([3.0, -1.0])
    assert c[0] == pytest.approx(1.41421356, rel=1e-8) and c[1] == pytest.approx(2.82842712, rel=1e-8)
    with pytest.raises(ValueError):
        oracle.fwht([1.0, 2.0, 3.0])


def test_thresholds_known_answers(oracle):  # test_quantizer.cpp:14-49
    t = oracle.compute_thresholds([1.0, -1.0, 1.0, -1.0], 2)
    assert t[0] == pytest.approx(-0.6745, rel=1e-4) and t[1] == 0.0 and t[2] == pytest.approx(0.6745, rel=1e-4)
    assert list(oracle.compute_thresholds([2.0, -2.0], 1)) == [0.0]
    for bad in ([0.0, 0.0, 0.0], [1.0, np.inf]):
        with pytest.raises(ValueError):
            oracle.compute_thresholds(bad, 2)


def test_bucketize_boundaries(oracle):  # test_quantizer.cpp:63-74
    t = [-0.6745, 0.0, 0.6745]
    assert list(oracle.bucketize([-1.0, -0.3, 0.3, 1.0], t)) == [0, 1, 2, 3]
    assert list(oracle.bucketize([0.6745], t)) == [2]
    assert list(oracle.bucketize([0.0], t)) == [1]
    assert list(oracle.bucketize([-0.6745], t)) == [0]


def test_pack_known_answers(oracle):  # test_quantizer.cpp:125-139, :177-187
    assert list(oracle.pack([3, 2, 1, 0, 0, 1, 2, 3])) == [58395]
    assert list(oracle.pack([0] * 8)) == [0]
    assert list(oracle.pack([3] * 8)) == [65535]
    assert list(oracle.pack([1] * 16, bits=1)) == [65535]
    assert list(oracle.pack([1, 1, 1])) == [1 | (1 << 2) | (1 << 4)]
    w = np.arange(65536, dtype=np.uint16)  # exhaustive round trip, acceptance.cpp criterion 3
    codes = np.stack([oracle.unpack(w[i:i + 1]) for i in range(0, 65536, 257)])
    assert all(oracle.pack(c)[0] == w[i * 257] for i, c in enumerate(codes))


def test_distance_known_answers(oracle):  # test_estimator.cpp:49-67, test_kernels.cpp:74-79
    a, b = oracle.pack([0, 1, 2, 3]), oracle.pack([3, 2, 1, 0])
    assert oracle.l1_2bit(a, b) == 8
    assert oracle.l1_2bit(oracle.pack([0, 3]), oracle.pack([3, 0])) == 6
    assert oracle.l1_2bit(a, a) == 0
    assert oracle.l1_2bit(np.array([0], np.uint16), np.array([0xFFFF], np.uint16)) == 24
    z = oracle.pack([0] * 128)
    t = oracle.pack([3] * 128)
    assert oracle.l1_2bit(z, t) == 384


def test_top_k_known_answers(oracle):  # test_estimator.cpp:217-243
    assert list(oracle.top_k([5, 1, 9, 1], 2)) == [1, 3]
    assert list(oracle.top_k([1, 1, 1], 2)) == [0, 1]
    assert list(oracle.top_k([4, 3, 2, 1], 10)) == [0, 1, 2, 3]
    assert list(oracle.top_k([7], 1)) == [0]
    assert list(oracle.top_k(np.array([], np.int32), 3)) == []
    assert list(oracle.top_k([3, 2, 1], 0)) == []
    rng = np.random.default_rng(8)
    for _ in range(50):
        s = rng.integers(0, 51, 1000).astype(np.int32)
        expected = np.sort(np.argsort(s, kind="stable")[:64])
        assert np.array_equal(oracle.top_k(s, 64), expected)
    s = rng.integers(-5, 1 << 20, 999).astype(np.int32)  # general (non-counting) path
    assert np.array_equal(oracle.top_k(s, 17), np.sort(np.argsort(s, kind="stable")[:17]))


def test_attention_known_answers(oracle):  # test_attention.cpp:70-98
    K = np.array([[0.3, -2.0, 5.0]])
    V = np.array([[1.5, -0.25, 1e6]])
    assert np.array_equal(oracle.full_attention([1.0, 2.0, 3.0], K, V), V[0])
    K = np.array([[0.7, -1.2], [0.7, -1.2]])
    V = np.array([[2.0, 4.0], [6.0, -2.0]])
    assert np.allclose(oracle.full_attention([0.5, 0.5], K, V), [4.0, 1.0], rtol=1e-15)
    with pytest.raises(ValueError):
        oracle.sparse_attention(np.ones(2), K, V, np.array([1, 0]))  # not increasing
    with pytest.raises(ValueError):
        oracle.sparse_attention(np.ones(2), K, V, np.array([], np.int64))


def test_oracle_matches_reference_build(oracle, reference):
    """Restatement == unmodified reference, bit for bit, on random vectors."""
    for i in range(300):
        x = synth(1000 + i, 0, 128).astype(np.float64) * (10.0 ** ((i % 7) - 3))
        assert np.array_equal(oracle.encode_pack(x), reference.encode_pack(x))
        assert np.array_equal(oracle.fwht(x), reference.fwht(x))
        assert np.array_equal(oracle.compute_thresholds(x), reference.compute_thresholds(x))
    rng = np.random.default_rng(3)
    for _ in range(200):
        a = rng.integers(0, 65536, 16).astype(np.uint16)
        b = rng.integers(0, 65536, 16).astype(np.uint16)
        assert oracle.l1_2bit(a, b) == reference.manhattan_packed(a, b)
    for _ in range(20):
        s = rng.integers(0, 40, 3000).astype(np.int32)
        for k in (0, 1, 64, 2999, 3000, 5000):
            assert np.array_equal(oracle.top_k(s, k), reference.top_k(s, k))
    S, d = 700, 128
    K = synth(5, 0, S * d).reshape(S, d).astype(np.float64)
    V = synth(6, 0, S * d).reshape(S, d).astype(np.float64)
    q = synth(7, 0, d).astype(np.float64)
    words, qw, scores, idx, out = reference.decode_head(q, K, V, 40)
    cw = oracle.encode_pack_rows(K)
    qw2, s2, i2, o2 = oracle.decode_head(q, K, V, cw, 40)
    assert np.array_equal(cw, words) and np.array_equal(qw, qw2)
    assert np.array_equal(scores, s2) and np.array_equal(idx, i2)
    assert np.array_equal(out, o2)  # same operation order: bit-identical doubles


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_reproduces_golden(oracle, golden, name):
    S, n_kv, n_q, budget, bf16, seed = (int(v) for v in golden[f"{name}/meta"])
    K, V, q = case_inputs(S, n_kv, n_q, bool(bf16), seed)
    h = hashlib.sha256()
    for a in (K, V, q):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.digest() == golden[f"{name}/input_sha256"].tobytes(), "synthetic generator drifted"
    G = n_q // n_kv
    for hq in range(n_q):
        hk = hq // G
        Kh, Vh = K[:, hk].astype(np.float64), V[:, hk].astype(np.float64)
        cw = oracle.encode_pack_rows(Kh)
        assert np.array_equal(cw, golden[f"{name}/key_words"][hk])
        qw, s, idx, out = oracle.decode_head(q[hq].astype(np.float64), Kh, Vh, cw, budget)
        assert np.array_equal(qw, golden[f"{name}/q_words"][hq])
        assert np.array_equal(s, golden[f"{name}/scores"][hq])
        assert np.array_equal(idx, golden[f"{name}/idx"][hq])
        assert np.array_equal(out, golden[f"{name}/out"][hq])


def test_bf16_round_matches_torch():
    import torch
    x = synth(17, 0, 4096) * 3.0
    assert np.array_equal(bf16_round(x), torch.from_numpy(x).to(torch.bfloat16).float().numpy())


def test_reference_snapshot_round_trip(reference, oracle, tmp_path):
    """The reference's own save_snapshot/load_snapshot through the shim (the
    checker the ADKV interop tests rely on)."""
    K = synth(91, 0, 40 * 128).reshape(40, 128)
    V = synth(92, 0, 40 * 128).reshape(40, 128)
    W = oracle.encode_pack_rows(K.astype(np.float64))
    c = reference.cache_from_rows(K, V, W)
    reference.save_snapshot(c, tmp_path / "r.adkv")
    reference.cache_free(c)
    Kr, Vr, Wr = reference.load_snapshot(tmp_path / "r.adkv")
    assert np.array_equal(Kr, K.astype(np.float64)) and np.array_equal(Vr, V.astype(np.float64))
    assert np.array_equal(Wr, W)
    raw = (tmp_path / "r.adkv").read_bytes()
    assert raw[:4] == b"ADKV" and len(raw) == 4 + 4 + 4 + 4 + 1 + 40 * 128 * 8 + 40 * 16 * 2


def test_plane_identities_for_ablation_metrics():
    """(a-b)^2 = L + 4Hd + 4(Hd&L&~X) - 4(Hd&L&X) and [ah != bh] = Hd with
    Hd = X ^ kx ^ L — the per-element identities behind adamas_score_metric."""
    for a in range(4):
        for b in range(4):
            al, ah, bl, bh = a & 1, a >> 1, b & 1, b >> 1
            L, X, kx = al ^ bl, al ^ ah, bl ^ bh
            Hd = X ^ kx ^ L
            assert Hd == ah ^ bh
            cr = Hd & L
            assert L + 4 * Hd + 4 * (cr & (1 - X)) - 4 * (cr & X) == (a - b) ** 2, (a, b)


def test_one_bit_code_is_the_two_bit_high_bit(reference):
    """The reference's 1-bit code (threshold {0}) equals the high bit of its
    2-bit code, so 1-bit distances follow from the 2-bit cache."""
    x = synth(77, 0, 64 * 128).reshape(64, 128).astype(np.float64)
    for row in x:
        w1 = reference.encode_pack_bits(row, 1)
        w2 = reference.encode_pack_bits(row, 2)
        c1 = np.array([(int(w1[i // 16]) >> (i % 16)) & 1 for i in range(128)])
        c2 = np.array([(int(w2[i // 8]) >> (2 * (i % 8))) & 3 for i in range(128)])
        assert np.array_equal(c1, c2 >> 1)
