"""Shared helpers for the -m gpu parity tests (oracle = checker only)."""
import numpy as np
import torch

from oracle.bindings import bf16_round, synth


def make_inputs(S, n_kv, n_q, bf16, seed):
    """Token-major inputs as the ABI takes them: K, V [S][n_kv][128], q [n_q][128]."""
    K = synth(seed * 10 + 1, 0, S * n_kv * 128).reshape(S, n_kv, 128)
    V = synth(seed * 10 + 2, 0, S * n_kv * 128).reshape(S, n_kv, 128)
    q = synth(seed * 10 + 3, 0, n_q * 128).reshape(n_q, 128)
    if bf16:
        K, V, q = bf16_round(K), bf16_round(V), bf16_round(q)
    return K, V, q


def to_dev(x, bf16):
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t.to(torch.bfloat16) if bf16 else t


def oracle_decode(oracle, K, V, q, budget, key_words=None):
    """Per q-head reference decode over the full (S, n_kv) cache."""
    S, n_kv, _ = K.shape
    n_q = q.shape[0]
    G = n_q // n_kv
    keep = min(budget, S)
    if key_words is None:
        key_words = np.stack([oracle.encode_pack_rows(K[:, h].astype(np.float64)) for h in range(n_kv)])
    idx = np.zeros((n_q, keep), np.int64)
    out = np.zeros((n_q, 128))
    scores = np.zeros((n_q, S), np.int32)
    for h in range(n_q):
        hk = h // G
        _, s, i, o = oracle.decode_head(q[h].astype(np.float64), K[:, hk].astype(np.float64),
                                        V[:, hk].astype(np.float64), key_words[hk], budget)
        idx[h], out[h], scores[h] = i, o, s
    return key_words, scores, idx, out


def rel_err(a, e):
    a = np.asarray(a, np.float64)
    e = np.asarray(e, np.float64)
    return np.linalg.norm(a - e, axis=-1) / np.maximum(np.linalg.norm(e, axis=-1), 1e-30)
