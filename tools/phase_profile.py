"""Per-phase timing of the fused decode kernel in steady state.

    python tools/phase_profile.py [--heads 32 --kv-heads 32 --seq 32768 --budget 128 --cluster 4 --layers 8]

The last of `layers` back-to-back launches (captured in a CUDA graph, like
bench.py) is traced. To keep the probe from perturbing what it measures, each
graph records ONE phase stamp (selected through ADAMAS_DBG bits 8..12) plus the
CTA start/end globaltimer stamps; the script re-captures once per phase and
reports, per phase boundary, the mean / max over CTAs of the time since the
CTA started (globaltimer, ns resolution ~32 ns).
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# phase stamps exist only in the diagnostics build (build.py --diag)
_diag = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2510_18413_b200",
                     "libadamas_b200_diag.so")
if "ADAMAS_LIB" not in os.environ:
    if not os.path.exists(_diag):
        sys.exit("needs the diagnostics build: python paper_2510_18413_b200/build.py --diag")
    os.environ["ADAMAS_LIB"] = _diag
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--heads", type=int, default=32)
ap.add_argument("--kv-heads", type=int, default=32)
ap.add_argument("--seq", type=int, default=32768)
ap.add_argument("--budget", type=int, default=128)
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--cluster", default="")
ap.add_argument("--traced", type=int, default=-2, help="index of the traced layer")
ap.add_argument("--seqs", type=int, default=1, help="independent sequences per launch (batched decode)")
args = ap.parse_args()
if args.cluster:
    os.environ["ADAMAS_CLUSTER"] = args.cluster
import paper_2510_18413_b200 as ad  # noqa: E402
from paper_2510_18413_b200._lib import load  # noqa: E402

L = load()
gen = torch.Generator(device="cuda").manual_seed(0)
caches = []  # [layer][sequence]
for _ in range(args.layers):
    per = []
    for _ in range(args.seqs):
        c = ad.KvCache(args.kv_heads, args.seq + 1, torch.bfloat16)
        for s0 in range(0, args.seq - 1, 4096):
            n = min(4096, args.seq - 1 - s0)
            c.update(torch.randn((n, args.kv_heads, 128), generator=gen, device="cuda").bfloat16(),
                     torch.randn((n, args.kv_heads, 128), generator=gen, device="cuda").bfloat16())
        per.append(c)
    caches.append(per)
q = torch.randn((args.seqs, args.heads, 128), generator=gen, device="cuda").bfloat16()
k = torch.randn((args.seqs, args.kv_heads, 128), generator=gen, device="cuda").bfloat16()
trace = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")
trace_prev = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")  # launch before the traced one (start/end)
names = ["start", "prologue (zero, q load, barrier init)", "encode + append", "scan", "hist exchange",
         "threshold", "compact count (+L2 prefetch) + scan", "compact emit",
         "attend gather", "attend combine + push", "inbox wait", "merge"]
prev_end = None
base_dbg = int(os.environ.get("ADAMAS_DBG", "0")) & 0xff


def run_layers():
    for li, per in enumerate(caches):
        traced = li == (args.traced % len(caches))
        before = li == (args.traced % len(caches)) - 1
        buf = trace if traced else (trace_prev if before else None)
        L.adamas_debug_trace(C.c_void_p(buf.data_ptr()) if buf is not None else None)
        if args.seqs == 1:
            per[0].decode_step(q[0], k[0], k[0], args.budget)
        else:
            ad.decode_step_batched(per, q, k, k, args.budget)
        for c in per:
            c.truncate(args.seq - 1)
    L.adamas_debug_trace(None)


def timed_graph(stamp):
    ad.set_tuning(dbg=base_dbg | ((stamp + 1) << 8 if stamp >= 0 else 0))
    trace.zero_()
    trace_prev.zero_()
    run_layers()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run_layers()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    t = trace.view(-1, 16).cpu()
    n = int((t[:, 14] > 0).sum())
    t = t[:n].double()
    tp = trace_prev.view(-1, 16).cpu()
    tp = tp[: int((tp[:, 14] > 0).sum())].double()
    if not (base_dbg & 64):  # clock64 stamps -> ns
        t = t / float(os.environ.get("SM_GHZ", "1.965"))
    global prev_end
    prev_end = float(tp[:, 15].max()) if (base_dbg & 64) and tp.shape[0] else None
    return e0.elapsed_time(e1) * 1000 / len(caches), t


us, t = timed_graph(-1)
span = (t[:, 15] - t[:, 14]) / 1000.0
print(f"graph: {us:.2f} us per layer; traced launch: {t.shape[0]} CTAs, per-CTA span mean {span.mean():.2f} "
      f"max {span.max():.2f}" + (f", CTA start spread {(t[:, 14].max() - t[:, 14].min()) / 1000:.2f} us, first start"
                                 f" -> last end {(t[:, 15].max() - t[:, 14].min()) / 1000:.2f} us"
                                 if base_dbg & 64 else " (clock64 stamps; ADAMAS_DBG=64 for globaltimer)"))
prev = torch.zeros(t.shape[0], dtype=torch.float64)
if prev_end is not None:  # globaltimer: the critical path, from the previous launch's last CTA end
    print(f"traced launch vs the previous launch's last CTA end: first CTA start {(t[:, 14].min() - prev_end) / 1000:+.2f} us, "
          f"last CTA end {(t[:, 15].max() - prev_end) / 1000:+.2f} us, CTA end spread {(t[:, 15].max() - t[:, 15].min()) / 1000:.2f} us")
    print(f"{'phase (ends at stamp), since prev end':42s} {'mean':>8s} {'min':>8s} {'max':>8s}")
print(f"{'phase (ends at stamp)':42s} {'cum mean':>9s} {'cum max':>9s} {'delta':>7s}")
for i in range(1, 12):
    us_i, ti = timed_graph(i)
    if prev_end is not None:
        rel = (ti[:, i] - prev_end) / 1000.0
        print(f"{names[i]:42s} {rel.mean():8.2f} {rel.min():8.2f} {rel.max():8.2f}   (graph {us_i:.2f} us/layer)")
        continue
    cum = (ti[:, i] - ti[:, 14]) / 1000.0
    d = cum.mean() - prev.mean()
    print(f"{names[i]:42s} {cum.mean():9.2f} {cum.max():9.2f} {d:7.2f}   (graph {us_i:.2f} us/layer)")
    prev = cum
for i, what in ((12, "compaction masks done (before the prefix)"), (13, "emit done (before the -1 fill)")):
    us_i, ti = timed_graph(i)
    if prev_end is not None:
        rel = (ti[:, i] - prev_end) / 1000.0
        print(f"stamp {i} {what}: since prev end mean {rel.mean():.2f} max {rel.max():.2f}")
        continue
    cum = (ti[:, i] - ti[:, 14]) / 1000.0
    print(f"stamp {i} {what}: cum mean {cum.mean():.2f} max {cum.max():.2f}")
ad.set_tuning(dbg=base_dbg)
