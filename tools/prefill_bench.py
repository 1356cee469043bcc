"""Bulk prefill: encode + append of a whole prompt into a
layer's cache (the reference's build_cache loop, sweep.cpp:38-50), as achieved
HBM GB/s: per (token, kv-head) 2 x 128 elements read + written, 32 B of codes.

    python tools/prefill_bench.py [--kv-heads 32 --tokens 32768 --chunk 32768]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_18413_b200 as ad  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kv-heads", type=int, default=32)
ap.add_argument("--tokens", type=int, default=32768)
ap.add_argument("--chunk", type=int, default=32768)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
dt = torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(0)
K = torch.randn((a.tokens, a.kv_heads, 128), generator=g, device="cuda").to(dt)
V = torch.randn((a.tokens, a.kv_heads, 128), generator=g, device="cuda").to(dt)
caches = [ad.KvCache(a.kv_heads, a.tokens, dt) for _ in range(a.reps + 1)]


def fill(c):
    for s in range(0, a.tokens, a.chunk):
        c.update(K[s:s + a.chunk], V[s:s + a.chunk])


fill(caches[0])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for c in caches[1:]:
    fill(c)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
vec = a.tokens * a.kv_heads
bytes_ = vec * (2 * 128 * 2 * 2 + 32)
print(json.dumps({"prefill_us": ms * 1000, "vectors": vec, "GBps": bytes_ / (ms * 1e-3) / 1e9,
                  "ns_per_vector": ms * 1e6 / vec, "chunk": a.chunk}))
for c in caches:
    c.raise_on_degenerate()
