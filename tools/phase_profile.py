"""Per-phase timing of the fused decode kernel (globaltimer stamps per CTA).

    python tools/phase_profile.py [--heads 32 --kv-heads 32 --seq 32768 --budget 128 --cluster 4]
Prints mean / max over CTAs of each phase's duration (us) for one layer's launch.
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--heads", type=int, default=32)
ap.add_argument("--kv-heads", type=int, default=32)
ap.add_argument("--seq", type=int, default=32768)
ap.add_argument("--budget", type=int, default=128)
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--cluster", default="")
args = ap.parse_args()
if args.cluster:
    os.environ["ADAMAS_CLUSTER"] = args.cluster
import paper_2510_18413_b200 as ad  # noqa: E402
from paper_2510_18413_b200._lib import load  # noqa: E402

L = load()
g = torch.Generator(device="cuda").manual_seed(0)
caches = []
for _ in range(args.layers):
    c = ad.KvCache(args.kv_heads, args.seq + 1, torch.bfloat16)
    for s0 in range(0, args.seq - 1, 4096):
        n = min(4096, args.seq - 1 - s0)
        c.update(torch.randn((n, args.kv_heads, 128), generator=g, device="cuda").bfloat16(),
                 torch.randn((n, args.kv_heads, 128), generator=g, device="cuda").bfloat16())
    caches.append(c)
q = torch.randn((args.heads, 128), device="cuda").bfloat16()
k = torch.randn((args.kv_heads, 128), device="cuda").bfloat16()
trace = torch.zeros(4096 * 16 + 4096 * 16 * 4, dtype=torch.int64, device="cuda")
names = ["tma+zero", "encode+append", "scan", "hist_exchange", "threshold", "compact_count", "compact_emit",
         "attend_gather", "attend_combine", "inbox_wait", "merge"]
for rep in range(3):
    for c in caches:  # layers back to back, the last one is traced
        L.adamas_debug_trace(C.c_void_p(trace.data_ptr()) if c is caches[-1] else None)
        c.decode_step(q, k, k, args.budget)
        c.truncate(args.seq - 1)
    torch.cuda.synchronize()
L.adamas_debug_trace(None)
wt = trace[4096 * 16:].view(4096, 16, 4).cpu().double()
t = trace[:4096 * 16].view(-1, 16).cpu()
n = int((t[:, 0] > 0).sum())
gt = t[:n, 14:16].double() / 1000.0  # globaltimer ns -> us
print(f"globaltimer: CTA start spread {(gt[:, 0].max() - gt[:, 0].min()):.2f} us, first start -> last end "
      f"{(gt[:, 1].max() - gt[:, 0].min()):.2f} us, end spread {(gt[:, 1].max() - gt[:, 1].min()):.2f} us")
t = t[:n, :14].double()
GHZ = float(os.environ.get("SM_GHZ", "1.965"))  # clock64 stamps -> us
t = t / (GHZ * 1000.0)
print(f"CTAs {n}; per-CTA span mean {(t[:, 11] - t[:, 0]).mean():.2f} us max {(t[:, 11] - t[:, 0]).max():.2f} us")
if os.environ.get("ADAMAS_DBG", "0") == "8":
    d = t[:, 5] - t[:, 7]
    print(f"  [bare barrier after p1: mean {d.mean():.2f} max {d.max():.2f}]")
if int(os.environ.get("ADAMAS_DBG", "0")) & 16:
    w = wt[:n] / (GHZ * 1000.0)
    a = (w[:, :, 1] - w[:, :, 0])
    b = (w[:, :, 2] - w[:, :, 1])
    print(f"  [p2 per-warp: cnt-loop mean {a.mean():.3f} max {a.max():.3f}; emit mean {b.mean():.3f} max {b.max():.3f}]")
    endw = w[:, :, 2]
    print(f"  [p2 end spread within CTA: mean {(endw.max(1).values - endw.min(1).values).mean():.3f}]")
for i, nm in enumerate(names):
    d = (t[:, i + 1] - t[:, i])
    print(f"{nm:14s} mean {d.mean():7.2f} us  max {d.max():7.2f} us  min {d.min():7.2f}")
