"""Debug: the failing speculative case (12000 tokens, 2 kv x 4 q, budget 64, C = 2, margin 40)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2510_18413_b200 as ad
from oracle.bindings import Oracle
from tests.gpu_helpers import make_inputs, oracle_decode, to_dev
from tests.test_gpu_spec import _mixed_queries
o = Oracle()
for margin, cluster, G in [(40, 2, 4), (-1, 2, 4), (40, 4, 1), (40, 1, 2), (6, 2, 4)]:
    ad.set_tuning(spec_margin=margin, cluster=cluster)
    S, n_kv, budget, steps = 12000, 2, 64, 4
    K, V, _ = make_inputs(S + steps, n_kv, n_kv * G, True, S + margin + 3)
    qs = _mixed_queries(K, n_kv * G, n_kv, steps, True, S + G)
    c = ad.KvCache(n_kv, S + steps + 4, torch.bfloat16)
    pre = S
    c.update(to_dev(K[:pre], True), to_dev(V[:pre], True))
    for st, q in enumerate(qs):
        t = pre + st
        out, idx = c.decode_step(to_dev(q, True), to_dev(K[t], True), to_dev(V[t], True), budget)
        _, sc, eidx, _ = oracle_decode(o, K[:t + 1], V[:t + 1], q, budget)
        got = idx.cpu().numpy()
        bad = np.nonzero((got != eidx).any(1))[0]
        print(f"margin {margin} C {cluster} G {G} step {st}: stats {c.spec_stats()} bad heads {bad.tolist()}")
        for h in bad[:2]:
            srt = np.sort(sc[h]); T = srt[budget - 1]
            extra = sorted(set(got[h]) - set(eidx[h])); miss = sorted(set(eidx[h]) - set(got[h]))
            print(f"   head {h}: T {T} extra {[(x, int(sc[h][x])) for x in extra][:6]} missing {[(x, int(sc[h][x])) for x in miss][:6]}")
