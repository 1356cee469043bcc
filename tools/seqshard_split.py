"""Time split of the sequence-sharded step (N = 1 emulation of one rank of 8):
local candidates alone, + select/attend, + merge (CUDA graph, 16 layers)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_18413_b200 as ad
from paper_2510_18413_b200.seqshard import CudaSeqOps
S, L, n_q, n_kv, B, W = 131072, 16, 32, 8, 128, 8
gen = torch.Generator(device="cuda").manual_seed(0)
caches = []
for _ in range(L):
    c = ad.KvCache(n_kv, S + 1, torch.bfloat16)
    for s0 in range(0, S - 1, 8192):
        n = min(8192, S - 1 - s0)
        c.update(torch.randn((n, n_kv, 128), generator=gen, device="cuda").bfloat16(),
                 torch.randn((n, n_kv, 128), generator=gen, device="cuda").bfloat16())
    caches.append(c)
q = torch.randn((L, n_q, 128), generator=gen, device="cuda").bfloat16()
ops = CudaSeqOps()
keys_all = torch.empty((L, W, n_q, B), dtype=torch.int32, device="cuda")
parts_all = torch.empty((L, W, n_q, 132), dtype=torch.float32, device="cuda")
off = (torch.arange(W, device="cuda", dtype=torch.int32) * S).view(-1, 1, 1)

def run(mode, st):
    for l in range(L):
        keys = ops.local_candidates(caches[l], q[l], None, None, False, 0, B, stream=st)
        if mode >= 1:
            torch.add(keys.unsqueeze(0), off, out=keys_all[l])
        if mode >= 2:
            part, _ = ops.select_attend(caches[l], q[l], keys_all[l], B, W * S, 0, stream=st)
        if mode >= 3:
            parts_all[l].copy_(part.unsqueeze(0).expand(W, -1, -1))
        if mode >= 4:
            ops.lse_merge(parts_all[l], stream=st)

for mode in range(5):
    run(mode, torch.cuda.current_stream())
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(5):
            run(mode, torch.cuda.current_stream())
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    print(["local", "+keys synth", "+select/attend", "+partials copy", "+merge"][mode], round(e0.elapsed_time(e1) * 1000 / (5 * L), 2), "us/layer")
