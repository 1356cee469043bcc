"""Per-CTA start / end (globaltimer) of one traced fused launch in steady
state (graph of back-to-back layers): which CTAs finish last."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ADAMAS_DBG"] = "64"
# phase stamps exist only in the diagnostics build (build.py --diag)
_diag = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2510_18413_b200",
                     "libadamas_b200_diag.so")
if "ADAMAS_LIB" not in os.environ:
    if not os.path.exists(_diag):
        sys.exit("needs the diagnostics build: python paper_2510_18413_b200/build.py --diag")
    os.environ["ADAMAS_LIB"] = _diag
import torch  # noqa: E402

import paper_2510_18413_b200 as ad  # noqa: E402
from paper_2510_18413_b200._lib import load  # noqa: E402

L = load()
S, H, layers = 32768, 32, 8
gen = torch.Generator(device="cuda").manual_seed(0)
caches = []
for _ in range(layers):
    c = ad.KvCache(H, S + 1, torch.bfloat16)
    for s0 in range(0, S - 1, 4096):
        n = min(4096, S - 1 - s0)
        c.update(torch.randn((n, H, 128), generator=gen, device="cuda").bfloat16(),
                 torch.randn((n, H, 128), generator=gen, device="cuda").bfloat16())
    caches.append(c)
q = torch.randn((H, 128), generator=gen, device="cuda").bfloat16()
k = torch.randn((H, 128), generator=gen, device="cuda").bfloat16()
traces = [torch.zeros(4096 * 16, dtype=torch.int64, device="cuda") for _ in range(2)]
tl = [layers // 2, layers // 2 + 1]


def run():
    for i, c in enumerate(caches):
        tr = traces[tl.index(i)] if i in tl else None
        L.adamas_debug_trace(C.c_void_p(tr.data_ptr()) if tr is not None else None)
        c.decode_step(q, k, k, 128)
        c.truncate(S - 1)
    L.adamas_debug_trace(None)


run()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    run()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
t0 = None
for li, tr in zip(tl, traces):
    t = tr.view(-1, 16).cpu()
    n = int((t[:, 14] > 0).sum())
    st, en = t[:n, 14].double(), t[:n, 15].double()
    if t0 is None:
        t0 = st.min()
    st, en = (st - t0) / 1000, (en - t0) / 1000
    print(f"layer {li}: {n} CTAs  start [{st.min():.2f}, {st.max():.2f}] us  end [{en.min():.2f}, {en.max():.2f}] us")
    order = torch.argsort(en)
    last = order[-12:].tolist()
    print("  last 12 to end (block, rank-in-cluster, head, end us):",
          [(b, b % 4, b // 4, round(float(en[b]), 2)) for b in last])
    for r in range(4):
        sel = torch.arange(n) % 4 == r
        print(f"  rank {r}: end mean {en[sel].mean():.2f} max {en[sel].max():.2f}; start mean {st[sel].mean():.2f}")
    early = (st < st.min() + 1.0).sum().item()
    print(f"  CTAs starting within 1 us of the first: {early}")
