"""Reference (CPU, double) implementation of the three sequence-sharded decode
phases' contracts (include/adamas_b200.h: adamas_seq_local_candidates,
adamas_seq_select_attend, adamas_lse_merge), built on the oracle — TEST
INFRASTRUCTURE ONLY. It lets the host protocol
(paper_2510_18413_b200/seqshard.py) run over torch.distributed/gloo on CPU
and be checked against the single-device oracle decode."""
import math

import numpy as np
import torch

from oracle.bindings import Oracle


class RefShard:
    """One rank's contiguous token range: K, V [len][n_kv][128] (values as
    stored on the device, widened to double) and the reference code words."""

    def __init__(self, oracle: Oracle, K, V):
        self.oracle = oracle
        self.K = np.asarray(K, np.float64).copy()
        self.V = np.asarray(V, np.float64).copy()
        n_kv = self.K.shape[1]
        self.words = [oracle.encode_pack_rows(self.K[:, h]) if len(self.K) else np.zeros((0, 16), np.uint16)
                      for h in range(n_kv)]

    def append(self, k, v):
        k = np.asarray(k, np.float64).reshape(1, -1, 128)
        v = np.asarray(v, np.float64).reshape(1, -1, 128)
        self.K = np.concatenate([self.K, k])
        self.V = np.concatenate([self.V, v])
        for h in range(k.shape[1]):
            self.words[h] = np.concatenate([self.words[h], self.oracle.encode_pack(k[0, h])[None]])


def _u32(t):
    return t.numpy().view(np.uint32) if isinstance(t, torch.Tensor) else np.asarray(t).view(np.uint32)


class RefSeqOps:
    def __init__(self, oracle: Oracle):
        self.o = oracle

    def local_candidates(self, shard, q, k_new, v_new, append, base, budget):
        if append:
            shard.append(k_new.numpy(), v_new.numpy())
        q = q.numpy().astype(np.float64).reshape(-1, 128)
        n_q, n_kv = q.shape[0], shard.K.shape[1]
        G = n_q // n_kv
        keys = np.full((n_q, budget), 0xFFFFFFFF, np.uint32)
        for h in range(n_q):
            if len(shard.K) == 0:
                continue
            scores = self.o.score_all(self.o.encode_pack(q[h]), shard.words[h // G])
            idx = self.o.top_k(scores, budget)  # the k smallest by (score, index), ascending
            keys[h, :len(idx)] = (scores[idx].astype(np.uint32) << 23) | (base + idx).astype(np.uint32)
        return torch.from_numpy(keys.view(np.int32))

    def select_attend(self, shard, q, gathered, budget, total_len, base, want_idx=False):
        q = q.numpy().astype(np.float64).reshape(-1, 128)
        keys = _u32(gathered)  # [world][n_q][budget]
        n_q, n_kv = q.shape[0], shard.K.shape[1]
        G = n_q // n_kv
        k_eff = min(budget, total_len)
        partial = np.zeros((n_q, 132), np.float32)
        gidx = np.full((n_q, budget), -1, np.int32)
        for h in range(n_q):
            kk = keys[:, h, :].ravel()
            kk = np.sort(kk[kk != 0xFFFFFFFF])[:k_eff]  # (distance, index) order
            sel = np.sort((kk & 0x7FFFFF).astype(np.int64))
            gidx[h, :len(sel)] = sel
            local = sel[(sel >= base) & (sel < base + len(shard.K))] - base
            if len(local) == 0:
                partial[h, 0] = -np.inf
                continue
            Kh, Vh = shard.K[local, h // G], shard.V[local, h // G]
            logits = Kh @ q[h] / math.sqrt(128.0)
            m = logits.max()
            p = np.exp(logits - m)
            partial[h, 0], partial[h, 1] = m, p.sum()
            partial[h, 4:] = p @ Vh
        return torch.from_numpy(partial), (torch.from_numpy(gidx) if want_idx else None)

    def lse_merge(self, partials):
        P = partials.numpy().astype(np.float64)
        m, l, o = P[:, :, 0], P[:, :, 1], P[:, :, 4:]
        M = np.where(l > 0, m, -np.inf).max(axis=0)
        c = np.where(l > 0, np.exp(m - M), 0.0)
        return torch.from_numpy(((c[:, :, None] * o).sum(0) / (c * l).sum(0)[:, None]).astype(np.float32))
