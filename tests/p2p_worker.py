"""Worker of tests/test_gpu_seqshard.py::test_seq_sharded_peer_exchange_two_processes:
rank r of 2 (both on cuda:0) holds half of a sequence, exchanges candidates and
partials through the peer mailboxes, and checks the global selection and the
output against the oracle decode of the whole sequence."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main(out_dir):
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    import paper_2510_18413_b200 as ad
    from oracle.bindings import Oracle
    from paper_2510_18413_b200.seqshard import Mailbox, SeqShardedDecoder, connect_mailboxes
    from tests.gpu_helpers import make_inputs, oracle_decode, rel_err, to_dev

    S, n_kv, G, budget, steps = 4000, 2, 2, 128, 3
    n_q = n_kv * G
    K, V, _ = make_inputs(S + steps, n_kv, n_q, True, 99)
    cuts = [0, S // 2, S]
    lengths = [cuts[1] - cuts[0], cuts[2] - cuts[1]]
    c = ad.KvCache(n_kv, lengths[rank] + steps + 4, torch.bfloat16)
    c.update(to_dev(K[cuts[rank]:cuts[rank + 1]], True), to_dev(V[cuts[rank]:cuts[rank + 1]], True))
    dec = SeqShardedDecoder(c, rank, world, lengths)
    box = Mailbox(rank, world, n_q, budget)
    connect_mailboxes(box)
    oracle = Oracle()
    for st in range(steps):
        t = S + st
        q = make_inputs(1, 1, n_q, True, 500 + st)[2]
        out, gidx = dec.decode_step_p2p(box, to_dev(q, True), to_dev(K[t], True), to_dev(V[t], True), want_idx=True)
        torch.cuda.synchronize()
        _, _, eidx, eout = oracle_decode(oracle, K[:t + 1], V[:t + 1], q, budget)
        assert np.array_equal(gidx.cpu().numpy(), eidx), (rank, st)
        assert rel_err(out.cpu().numpy(), eout).max() <= 1e-2, (rank, st)
        dist.barrier()
    assert box.status() == 0
    box.close()
    with open(os.path.join(out_dir, f"ok{rank}"), "w") as f:
        f.write("ok")
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
