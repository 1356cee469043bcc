"""Probe: one harness build (hsel_encode over 100 x 8192 x 128 fp64 keys) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_18413_b200 import harness as H  # noqa: E402

K = torch.randn((100, 8192, 128), dtype=torch.float64, device="cuda")
Q = torch.randn((100, 128), dtype=torch.float64, device="cuda")
sel = H.HarnessSelector(128, 2, True)
for _ in range(3):
    sel.build(K)
    sel.select(Q, 64, "l1", 1)
pg = H.PageSelector(16, 128)
pg.build(K)
pg.select(Q, 64, 1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    sel.build(K)
e1.record()
torch.cuda.synchronize()
print("build ms", e0.elapsed_time(e1) / 10)
