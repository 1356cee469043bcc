import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2510_18413_b200 as ad
from oracle.bindings import Oracle
from tests.gpu_helpers import make_inputs, oracle_decode, to_dev
o = Oracle()
margin, cluster, G, S = [int(x) for x in sys.argv[1:5]]
ad.set_tuning(spec_margin=margin, cluster=cluster)
n_kv, budget, steps = 2, 64, 3
K, V, _ = make_inputs(S + steps, n_kv, n_kv * G, True, S + 7)
c = ad.KvCache(n_kv, S + steps + 4, torch.bfloat16)
c.update(to_dev(K[:S], True), to_dev(V[:S], True))
res = []
for st in range(steps):
    t = S + st
    q = make_inputs(1, 1, n_kv * G, True, 100 + st)[2]
    out, idx = c.decode_step(to_dev(q, True), to_dev(K[t], True), to_dev(V[t], True), budget)
    _, sc, eidx, _ = oracle_decode(o, K[:t + 1], V[:t + 1], q, budget)
    res.append(np.nonzero((idx.cpu().numpy() != eidx).any(1))[0].tolist())
print(f"margin {margin} C {cluster} G {G} S {S}: stats {c.spec_stats()} bad heads per step {res}", flush=True)
