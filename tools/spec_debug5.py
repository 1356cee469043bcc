import os, sys, ctypes as C
sys.path.insert(0, os.getcwd())
os.environ["ADAMAS_LIB"] = os.path.join(os.getcwd(), "paper_2510_18413_b200", "libadamas_b200_diag.so")
import numpy as np, torch
import paper_2510_18413_b200 as ad
from paper_2510_18413_b200._lib import load
from oracle.bindings import Oracle
from tests.gpu_helpers import make_inputs, oracle_decode, to_dev
o = Oracle(); L = load()
margin, cluster, G, S = [int(x) for x in sys.argv[1:5]]
ad.set_tuning(spec_margin=margin, cluster=cluster, dbg=1 << 20, stages=2)
n_kv, budget, steps = 2, 64, 3
K, V, _ = make_inputs(S + steps, n_kv, n_kv * G, True, S + 7)
c = ad.KvCache(n_kv, S + steps + 4, torch.bfloat16)
c.update(to_dev(K[:S], True), to_dev(V[:S], True))
trace = torch.zeros(4096 * 64, dtype=torch.int64, device="cuda")
for st in range(steps):
    t = S + st
    q = make_inputs(1, 1, n_kv * G, True, 100 + st)[2]
    trace.zero_()
    L.adamas_debug_trace(C.c_void_p(trace.data_ptr()))
    out, idx = c.decode_step(to_dev(q, True), to_dev(K[t], True), to_dev(V[t], True), budget)
    L.adamas_debug_trace(None)
    torch.cuda.synchronize()
    _, sc, eidx, _ = oracle_decode(o, K[:t + 1], V[:t + 1], q, budget)
    bad = np.nonzero((idx.cpu().numpy() != eidx).any(1))[0].tolist()
    tr = trace.cpu().numpy().view(np.uint16)
    n = t + 1
    # swizzle-free comparison: multiset of distances of head 0 (CTA 0 = kv-head 0, q-head 0 at G = 1)
    row0, row1 = tr[:n], tr[262144:262144 + n]
    ti = trace.cpu().numpy().view(np.int32)
    exp = np.sort(sc[0])
    print(f"step {st}: bad {bad}; T kernel {ti[200000]} fallback {ti[200008]} T oracle {exp[budget - 1]}; "
          f"after-scan row == oracle multiset {np.array_equal(np.sort(row0), exp)}; end row == after-scan {np.array_equal(row0, row1)}; "
          f"diff positions {np.nonzero(row0 != row1)[0][:10].tolist()}", flush=True)
    if 0 in bad:
        got = idx.cpu().numpy()[0]
        e = eidx[0]
        extra = sorted(set(got) - set(e)); miss = sorted(set(e) - set(got))
        print("   nsel", ti[200016], "below kernel", ti[200024], "below oracle", int((sc[0] < exp[budget - 1]).sum()))
        print("   extra", [(int(x), int(sc[0][x])) for x in extra], "missing", [(int(x), int(sc[0][x])) for x in miss])
        selk = ti[210000:210000 + budget]
        print("   sel == idx", np.array_equal(np.sort(selk[:len(got)]), np.sort(got)), "sel sorted", np.all(np.diff(selk) > 0))
        print("   idx sorted", np.all(np.diff(got) > 0), "dups", len(got) - len(set(got)))
