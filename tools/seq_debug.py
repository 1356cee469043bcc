"""Debug: sequence-shard step at the config-4 per-rank shape (8 kv / 32 q, 131072 tokens per shard), W shards."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2510_18413_b200 as ad
from paper_2510_18413_b200.seqshard import Mailbox, SeqShardedDecoder, simulate_step_p2p, simulate_step
W = int(sys.argv[1]) if len(sys.argv) > 1 else 2
per = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
mode = sys.argv[3] if len(sys.argv) > 3 else "p2p"
n_kv, n_q, budget = 8, 32, 128
gen = torch.Generator(device="cuda").manual_seed(44)
r = lambda *s: torch.randn(s, generator=gen, device="cuda").to(torch.bfloat16)
lengths = [per] * (W - 1) + [per - 1]
decs = []
for i in range(W):
    c = ad.KvCache(n_kv, per + 4, torch.bfloat16)
    K, V = r(lengths[i], n_kv, 128), r(lengths[i], n_kv, 128)
    for s0 in range(0, lengths[i], 8192):
        c.update(K[s0:s0 + 8192].contiguous(), V[s0:s0 + 8192].contiguous())
    decs.append(SeqShardedDecoder(c, i, W, lengths))
torch.cuda.synchronize()
print("filled", flush=True)
q = r(n_q, 128)
kn, vn = r(n_kv, 128), r(n_kv, 128)
if mode == "p2p":
    boxes = [Mailbox(i, W, n_q, budget) for i in range(W)]
    Mailbox.connect_local(boxes)
    outs, gidx = simulate_step_p2p(decs, boxes, [q] * W, kn, vn, want_idx=True)
else:
    outs, gidx = simulate_step(decs, [q] * W, kn, vn, budget, want_idx=True)
torch.cuda.synchronize()
print("ok", outs[0].abs().sum().item(), flush=True)
