"""-m gpu: sequence-sharded decode kernels (adamas_seq_local_candidates,
adamas_seq_select_attend, adamas_lse_merge) through the host protocol with W
shards simulated on one GPU: local keys bit-exact against the reference ops,
global indices bit-exact and the merged output within tolerance of the
single-device oracle decode over the whole sequence."""
import numpy as np
import pytest
import torch

from tests.gpu_helpers import make_inputs, oracle_decode, rel_err, to_dev
from tests.seqshard_ref import RefSeqOps, RefShard

pytestmark = pytest.mark.gpu
TOL = {False: 1e-3, True: 1e-2}


@pytest.mark.parametrize("S,W,n_kv,G,budget,bf16", [
    (3000, 2, 2, 1, 64, True),
    (5000, 4, 2, 4, 128, True),    # GQA, Llama-style group
    (777, 3, 1, 2, 300, False),    # budget > per-shard length on some shards
    (64, 4, 1, 1, 128, True),      # budget > whole sequence
])
def test_seq_sharded_decode_matches_single_device(gpu, oracle, S, W, n_kv, G, budget, bf16):
    from paper_2510_18413_b200.seqshard import SeqShardedDecoder, simulate_step
    n_q = n_kv * G
    steps = 2
    K, V, _ = make_inputs(S + steps, n_kv, n_q, bf16, S + W)
    cuts = np.linspace(0, S, W + 1).astype(int)
    lengths = [int(cuts[r + 1] - cuts[r]) for r in range(W)]
    dt = torch.bfloat16 if bf16 else torch.float32
    decs, refs = [], []
    for r in range(W):
        c = gpu.KvCache(n_kv, lengths[r] + steps + 4, dt)
        if lengths[r]:
            c.update(to_dev(K[cuts[r]:cuts[r + 1]], bf16), to_dev(V[cuts[r]:cuts[r + 1]], bf16))
        decs.append(SeqShardedDecoder(c, r, W, lengths))
        refs.append(RefShard(oracle, K[cuts[r]:cuts[r + 1]], V[cuts[r]:cuts[r + 1]]))
    ref_ops = RefSeqOps(oracle)
    for st in range(steps):
        t = S + st
        q = make_inputs(1, 1, n_q, bf16, 7 * S + st)[2]
        qd = [to_dev(q, bf16)] * W
        kd, vd = to_dev(K[t], bf16), to_dev(V[t], bf16)
        # phase 1 alone, against the reference contract (bit-exact keys)
        base = sum(lengths[:W - 1])
        keys = decs[-1].ops.local_candidates(decs[-1].cache, qd[0], kd, vd, True, base, budget)
        decs[-1].cache.truncate(decs[-1].cache.seq_len - 1)
        ekeys = ref_ops.local_candidates(refs[-1], torch.from_numpy(q), torch.from_numpy(K[t]),
                                         torch.from_numpy(V[t]), True, base, budget)
        assert np.array_equal(keys.cpu().numpy(), ekeys.numpy()), st
        outs, gidx = simulate_step(decs, qd, kd, vd, budget, want_idx=True)
        lengths[-1] += 1
        _, _, eidx, eout = oracle_decode(oracle, K[:t + 1], V[:t + 1], q, budget)
        keep = min(budget, t + 1)
        for r in range(W):
            g = gidx[r].cpu().numpy()
            assert np.array_equal(g[:, :keep], eidx), (st, r)
            assert (g[:, keep:] == -1).all()
            assert rel_err(outs[r].cpu().numpy(), eout).max() <= TOL[bf16], (st, r)
    assert sum(d.cache.seq_len for d in decs) == S + steps


@pytest.mark.parametrize("S,W,n_kv,G,budget,bf16", [
    (3000, 2, 2, 1, 64, True),
    (5000, 4, 2, 4, 128, True),
    (777, 3, 1, 2, 300, False),
    (64, 4, 1, 1, 128, True),      # empty shards publish empty keys
    (20000, 8, 2, 4, 128, True),   # the largest world
])
def test_seq_sharded_peer_exchange(gpu, oracle, S, W, n_kv, G, budget, bf16):
    """Peer-memory exchange (mailboxes, epoch flags) instead of all-gathers:
    global indices bit-exact, outputs equal to the all-gather path's."""
    from paper_2510_18413_b200.seqshard import Mailbox, SeqShardedDecoder, simulate_step, simulate_step_p2p
    n_q = n_kv * G
    steps = 3
    K, V, _ = make_inputs(S + steps, n_kv, n_q, bf16, S + W + 1)
    cuts = np.linspace(0, S, W + 1).astype(int)
    lengths = [int(cuts[r + 1] - cuts[r]) for r in range(W)]
    dt = torch.bfloat16 if bf16 else torch.float32

    def shards():
        out = []
        for r in range(W):
            c = gpu.KvCache(n_kv, lengths[r] + steps + 4, dt)
            if lengths[r]:
                c.update(to_dev(K[cuts[r]:cuts[r + 1]], bf16), to_dev(V[cuts[r]:cuts[r + 1]], bf16))
            out.append(SeqShardedDecoder(c, r, W, lengths))
        return out

    p2p, ag = shards(), shards()
    boxes = [Mailbox(r, W, n_q, budget) for r in range(W)]
    Mailbox.connect_local(boxes)
    for st in range(steps):
        t = S + st
        q = make_inputs(1, 1, n_q, bf16, 11 * S + st)[2]
        qd = [to_dev(q, bf16)] * W
        kd, vd = to_dev(K[t], bf16), to_dev(V[t], bf16)
        outs, gidx = simulate_step_p2p(p2p, boxes, qd, kd, vd, want_idx=True)
        aouts, agidx = simulate_step(ag, qd, kd, vd, budget, want_idx=True)
        _, _, eidx, eout = oracle_decode(oracle, K[:t + 1], V[:t + 1], q, budget)
        keep = min(budget, t + 1)
        torch.cuda.synchronize()
        for r in range(W):
            g = gidx[r].cpu().numpy()
            assert np.array_equal(g[:, :keep], eidx), (st, r)
            assert np.array_equal(g, agidx[r].cpu().numpy())
            assert torch.equal(outs[r], aouts[r]), (st, r)
            assert rel_err(outs[r].cpu().numpy(), eout).max() <= TOL[bf16], (st, r)
    assert all(b.status() == 0 for b in boxes)


def test_seq_sharded_peer_exchange_two_processes(gpu, tmp_path):
    """Two ranks in two processes sharing one GPU through CUDA IPC mailboxes
    (gloo only exchanges the handles at setup): the cross-process protocol
    (stores into a peer's memory, release/acquire epochs) end to end."""
    import os
    import subprocess
    import sys
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    import socket
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as sk:  # a free rendezvous port
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(root, "tests", "p2p_worker.py"),
           str(tmp_path)]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=root)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    for r in range(2):
        assert (tmp_path / f"ok{r}").read_text() == "ok", r


def test_mailbox_errors(gpu):
    from paper_2510_18413_b200._lib import ConfigError
    from paper_2510_18413_b200.seqshard import Mailbox, SeqShardedDecoder
    with pytest.raises(ConfigError):
        Mailbox(2, 2, 4, 128)          # rank out of range
    with pytest.raises(ConfigError):
        Mailbox(0, 9, 4, 128)          # more than 8 ranks
    with pytest.raises(ConfigError):
        Mailbox(0, 8, 4, 2048)         # world * budget > 8192
    box = Mailbox(0, 2, 4, 64)         # peer 1 never connected
    c = gpu.KvCache(1, 64, torch.bfloat16)
    c.update(torch.randn(32, 1, 128, device="cuda").bfloat16(), torch.randn(32, 1, 128, device="cuda").bfloat16())
    dec = SeqShardedDecoder(c, 0, 2, [32, 32])
    q = torch.randn(4, 128, device="cuda").bfloat16()
    with pytest.raises(ConfigError, match="not connected"):
        dec.local_p2p(box, q, None, None)
    assert len(box.ipc_handle()) == Mailbox.HANDLE_BYTES


@pytest.mark.parametrize("W,n_kv,G,budget,bf16", [(8, 2, 4, 128, True), (3, 1, 2, 64, False), (12, 1, 4, 64, True)])
def test_select_attend_merge_equals_two_launches(gpu, oracle, W, n_kv, G, budget, bf16):
    """adamas_seq_select_attend_merge (one launch: this rank's partial into its
    slot, then the log-sum-exp merge over every slot) against
    adamas_seq_select_attend + adamas_lse_merge: identical outputs and indices,
    and the oracle's selection over the whole sequence."""
    from paper_2510_18413_b200.seqshard import CudaSeqOps
    ops = CudaSeqOps()
    S = 600 * W
    n_q = n_kv * G
    K, V, q = make_inputs(S, n_kv, n_q, bf16, 31 + W)
    dt = torch.bfloat16 if bf16 else torch.float32
    per = S // W
    caches = []
    for r in range(W):
        c = gpu.KvCache(n_kv, per + 4, dt)
        c.update(to_dev(K[r * per:(r + 1) * per], bf16), to_dev(V[r * per:(r + 1) * per], bf16))
        caches.append(c)
    qd = to_dev(q, bf16)
    keys = torch.stack([ops.local_candidates(caches[r], qd, None, None, False, r * per, budget) for r in range(W)])
    parts = torch.stack([ops.select_attend(caches[r], qd, keys, budget, S, r * per)[0] for r in range(W)])
    ref_out = ops.lse_merge(parts)
    _, ref_idx = ops.select_attend(caches[0], qd, keys, budget, S, 0, want_idx=True)
    _, _, eidx, _ = oracle_decode(oracle, K, V, q, budget)
    assert np.array_equal(ref_idx.cpu().numpy(), eidx)
    for r in range(W):
        buf = parts.clone()
        buf[r].fill_(float("nan"))  # this rank's slot is written by the launch itself
        out, gidx = ops.select_attend_merge(caches[r], qd, keys, budget, S, r * per, buf, r, want_idx=True)
        torch.cuda.synchronize()
        assert torch.equal(out, ref_out), r
        assert torch.equal(buf[r], parts[r]), r
        assert np.array_equal(gidx.cpu().numpy(), eidx), r
