"""CPU, world_size 2 over gloo: the sequence-sharded decode protocol
(paper_2510_18413_b200/seqshard.py: ranges, bases, tail appends, phase order,
the two all-gathers, the LSE merge) reproduces the single-device oracle decode
— indices bit-exact, output within 1e-9 (double phases) — with the phases
supplied by the CPU reference ops (tests/seqshard_ref.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, S, n_kv, G, budget, steps, seed):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        # the protocol module only; the CUDA library is not loaded on this path
        import importlib.util
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        spec = importlib.util.spec_from_file_location(
            "seqshard_proto", os.path.join(root, "paper_2510_18413_b200", "seqshard.py"),
            submodule_search_locations=None)
        import re
        src = re.sub(r"^from \._lib import .*$", "check = load = None\nADAMAS_STATUS_PEER_TIMEOUT = 8\n"
                     "AdamasRuntimeError = RuntimeError", open(spec.origin).read(), flags=re.M)
        proto = type(sys)("seqshard_proto")
        exec(compile(src, spec.origin, "exec"), proto.__dict__)

        from oracle.bindings import Oracle
        from tests.gpu_helpers import make_inputs
        from tests.seqshard_ref import RefSeqOps, RefShard
        o = Oracle()
        n_q = n_kv * G
        K, V, _ = make_inputs(S + steps, n_kv, n_q, True, seed)
        # uneven split of the prefix S over the ranks, in order
        cuts = [0] + sorted(np.random.default_rng(seed).choice(np.arange(1, S), world - 1, replace=False).tolist()) + [S]
        lo, hi = cuts[rank], cuts[rank + 1]
        shard = RefShard(o, K[lo:hi], V[lo:hi])
        dec = proto.SeqShardedDecoder(shard, rank, world, [cuts[r + 1] - cuts[r] for r in range(world)],
                                      ops=RefSeqOps(o))
        gather = proto.torch_allgather()
        for st in range(steps):
            q = make_inputs(1, 1, n_q, True, seed * 100 + st)[2]
            t = S + st
            out, gidx = dec.decode_step(torch.from_numpy(q), torch.from_numpy(K[t]), torch.from_numpy(V[t]),
                                        budget, gather, want_idx=True)
            # single-device oracle over tokens [0, t]
            words = [o.encode_pack_rows(K[:t + 1, h].astype(np.float64)) for h in range(n_kv)]
            keep = min(budget, t + 1)
            for h in range(n_q):
                _, _, eidx, eout = o.decode_head(q[h].astype(np.float64), K[:t + 1, h // G].astype(np.float64),
                                                 V[:t + 1, h // G].astype(np.float64), words[h // G], budget)
                assert np.array_equal(gidx[h, :keep].numpy(), eidx), (rank, st, h)
                err = np.linalg.norm(out[h].numpy() - eout) / np.linalg.norm(eout)
                assert err < 1e-6, (rank, st, h, err)
        assert dec.total == S + steps
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("S,n_kv,G,budget", [(600, 2, 2, 32), (257, 1, 4, 300)])
def test_seq_sharded_protocol_gloo_world2(S, n_kv, G, budget):
    mp.spawn(_worker, args=(2, _free_port(), S, n_kv, G, budget, 2, 17), nprocs=2, join=True)


def test_seq_sharded_protocol_gloo_world3_ties():
    # few tokens, many equal distances across ranks: the lowest-index rule decides
    mp.spawn(_worker, args=(3, _free_port(), 90, 1, 1, 40, 1, 5), nprocs=3, join=True)
