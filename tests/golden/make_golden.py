"""Generates tests/golden/golden.npz from the UNMODIFIED reference library.

Run in the build container (needs /root/reference to build oracle/_ref):
    make -C oracle all ref && python tests/golden/make_golden.py

Inputs are not stored: they are regenerated bit-exactly from the integer
synthetic generator (oracle.bindings.synth) and pinned by a sha256 digest.
Per case and q-head the fixture stores what the reference computes:
the key codes (PackedCodes words of every cached token), the query code, the
int32 distances, the selected indices and the double attention output —
i.e. build_cache + select(adamas) + attend (sweep.cpp:38-50, :87-98, :225-226).
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.bindings import Reference, bf16_round, synth  # noqa: E402

# name: (S, n_kv, n_q, budget, bf16, seed)
CASES = {
    "ragged_fp32": (300, 2, 2, 16, False, 101),
    "bf16_1000": (1000, 1, 1, 64, True, 202),
    "ties_4096": (4096, 1, 1, 128, False, 303),
    "gqa_777": (777, 2, 8, 32, True, 404),
    "single_token": (1, 1, 1, 4, False, 505),
    "budget_eq_S": (5, 1, 2, 5, False, 606),
    "budget_gt_S": (100, 1, 1, 256, True, 707),
}


def case_inputs(S, n_kv, n_q, bf16, seed):
    K = synth(seed * 10 + 1, 0, S * n_kv * 128).reshape(S, n_kv, 128)
    V = synth(seed * 10 + 2, 0, S * n_kv * 128).reshape(S, n_kv, 128)
    q = synth(seed * 10 + 3, 0, n_q * 128).reshape(n_q, 128)
    if bf16:
        K, V, q = bf16_round(K), bf16_round(V), bf16_round(q)
    return K, V, q


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    ref = Reference()
    out = {}
    for name, (S, n_kv, n_q, budget, bf16, seed) in CASES.items():
        K, V, q = case_inputs(S, n_kv, n_q, bf16, seed)
        G = n_q // n_kv
        words = np.zeros((n_kv, S, 16), np.uint16)
        qw = np.zeros((n_q, 16), np.uint16)
        scores = np.zeros((n_q, S), np.int32)
        keep = min(budget, S)
        idx = np.zeros((n_q, keep), np.int64)
        att = np.zeros((n_q, 128), np.float64)
        for h in range(n_q):
            hk = h // G
            w, qwh, s, i, o = ref.decode_head(q[h].astype(np.float64), K[:, hk].astype(np.float64),
                                             V[:, hk].astype(np.float64), budget)
            if h % G == 0:
                words[hk] = w
            qw[h], scores[h], idx[h], att[h] = qwh, s, i, o
        meta = np.array([S, n_kv, n_q, budget, int(bf16), seed], np.int64)
        out[f"{name}/meta"] = meta
        out[f"{name}/input_sha256"] = np.frombuffer(bytes.fromhex(digest(K, V, q)), np.uint8)
        out[f"{name}/key_words"] = words
        out[f"{name}/q_words"] = qw
        out[f"{name}/scores"] = scores
        out[f"{name}/idx"] = idx
        out[f"{name}/out"] = att
        print(name, "S", S, "budget", budget, "selected", idx.shape, "simd", ref.simd_level())
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
