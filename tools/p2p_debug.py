import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_18413_b200 as gpu
from paper_2510_18413_b200.seqshard import Mailbox, SeqShardedDecoder, simulate_step, simulate_step_p2p
from tests.gpu_helpers import make_inputs, to_dev
S, W, n_kv, G, budget, bf16 = 3000, 2, 2, 1, 64, True
n_q = n_kv * G; steps = 3
K, V, _ = make_inputs(S + steps, n_kv, n_q, bf16, S + W + 1)
cuts = np.linspace(0, S, W + 1).astype(int)
lengths = [int(cuts[r + 1] - cuts[r]) for r in range(W)]
def shards():
    out = []
    for r in range(W):
        c = gpu.KvCache(n_kv, lengths[r] + steps + 4, torch.bfloat16)
        c.update(to_dev(K[cuts[r]:cuts[r + 1]], bf16), to_dev(V[cuts[r]:cuts[r + 1]], bf16))
        out.append(SeqShardedDecoder(c, r, W, lengths))
    return out
p2p, ag, ag2 = shards(), shards(), shards()
boxes = [Mailbox(r, W, n_q, budget) for r in range(W)]
Mailbox.connect_local(boxes)
for st in range(steps):
    t = S + st
    q = make_inputs(1, 1, n_q, bf16, 11 * S + st)[2]
    qd = [to_dev(q, bf16)] * W
    kd, vd = to_dev(K[t], bf16), to_dev(V[t], bf16)
    outs, gidx = simulate_step_p2p(p2p, boxes, qd, kd, vd, want_idx=True)
    aouts, agidx = simulate_step(ag, qd, kd, vd, budget, want_idx=True)
    a2, _ = simulate_step(ag2, qd, kd, vd, budget, want_idx=True)
    torch.cuda.synchronize()
    print(st, "p2p r0==r1", torch.equal(outs[0], outs[1]), "ag r0==r1", torch.equal(aouts[0], aouts[1]),
          "ag==ag2", torch.equal(aouts[0], a2[0]), "p2p==ag", torch.equal(outs[0], aouts[0]),
          "maxdiff", (outs[0] - aouts[0]).abs().max().item(), [b.status() for b in boxes])
    for r in range(W):
        print("  keys equal seq_len", p2p[r].cache.seq_len, ag[r].cache.seq_len,
              torch.equal(p2p[r].cache.keys()[:, :p2p[r].cache.seq_len], ag[r].cache.keys()[:, :ag[r].cache.seq_len]),
              torch.equal(p2p[r].cache.code_words(), ag[r].cache.code_words()))
