"""-m gpu: ADKV snapshot interchange with the UNMODIFIED reference
(save_snapshot / load_snapshot, kv_cache.cpp:111-165, via oracle/_ref):
files written by the device cache are byte-identical to the reference's for
the same rows and codes, and reference snapshots load into a device cache with
the same code words and decode like the oracle."""
import os

import numpy as np
import pytest
import torch

from tests.gpu_helpers import make_inputs, oracle_decode, rel_err, to_dev

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bf16", [False, True])
def test_device_snapshot_is_byte_identical_to_reference(gpu, oracle, reference, tmp_path, bf16):
    S, n_kv = 700, 2
    K, V, _ = make_inputs(S, n_kv, n_kv, bf16, 3)
    cache = gpu.KvCache(n_kv, S, torch.bfloat16 if bf16 else torch.float32)
    cache.update(to_dev(K, bf16), to_dev(V, bf16))
    for h in range(n_kv):
        mine = tmp_path / f"dev_{h}.adkv"
        cache.save_snapshot(h, mine)
        words = oracle.encode_pack_rows(K[:, h].astype(np.float64))
        rc = reference.cache_from_rows(K[:, h], V[:, h], words)
        theirs = tmp_path / f"ref_{h}.adkv"
        reference.save_snapshot(rc, theirs)
        reference.cache_free(rc)
        assert mine.read_bytes() == theirs.read_bytes(), h
        Kr, Vr, Wr = reference.load_snapshot(mine)  # and the reference reads ours back
        assert np.array_equal(Wr, words) and np.array_equal(Kr, K[:, h].astype(np.float64))


def test_reference_snapshots_load_and_decode(gpu, oracle, reference, tmp_path):
    S, n_kv, G, budget = 1500, 2, 2, 64
    K, V, q = make_inputs(S + 1, n_kv, n_kv * G, False, 4)
    paths = []
    for h in range(n_kv):
        words = oracle.encode_pack_rows(K[:S, h].astype(np.float64))
        rc = reference.cache_from_rows(K[:S, h], V[:S, h], words)
        paths.append(tmp_path / f"ref_{h}.adkv")
        reference.save_snapshot(rc, paths[-1])
        reference.cache_free(rc)
    cache = gpu.KvCache(n_kv, S + 4, torch.float32)
    assert cache.load_snapshots(paths) == S
    got = cache.code_words().cpu().numpy().view(np.uint16)
    for h in range(n_kv):
        assert np.array_equal(got[h], oracle.encode_pack_rows(K[:S, h].astype(np.float64)))
    out, idx = cache.decode_step(to_dev(q, False), to_dev(K[S], False), to_dev(V[S], False), budget)
    _, _, eidx, eout = oracle_decode(oracle, K, V, q, budget)
    assert np.array_equal(idx.cpu().numpy(), eidx)
    assert rel_err(out.cpu().numpy(), eout).max() <= 1e-3


def test_snapshot_errors_mirror_the_reference(gpu, tmp_path):
    cache = gpu.KvCache(1, 16, torch.float32)
    bad = tmp_path / "bad.adkv"
    bad.write_bytes(b"XXXX" + bytes(20))
    with pytest.raises(gpu.AdamasRuntimeError):  # std::runtime_error: bad magic
        cache.load_snapshots([bad])
    with pytest.raises(gpu.ConfigError):  # one snapshot per kv-head
        cache.load_snapshots([bad, bad])
    with pytest.raises(gpu.AdamasRuntimeError):
        cache.load_snapshots([tmp_path / "missing.adkv"])
