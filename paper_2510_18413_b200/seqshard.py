"""Sequence-sharded Adamas decode across ranks (BASELINE config 4).

The reference decodes one head over its whole cache on one thread
(select adamas branch, sweep.cpp:87-98: score_all + top_k, estimator.cpp:45-90,
then sparse_attention, attention.cpp:40-45). Here a sequence is split into
contiguous token ranges, one per rank (one process per GPU); the rank owning
the tail appends the new token. One decode step is three device phases with
two small collectives between them:

  1. local   (every rank)  append (tail rank) + encode q + scan + local top-k:
                            keys (distance << 23 | global index), [n_q][budget]
     all-gather keys        [world][n_q][budget] uint32 (16 KB/rank at 32 q-heads, k = 128)
  2. attend  (every rank)  rebuild the global top-k from the keys (bit-exact: a
                            global survivor has < k predecessors in its own
                            range, so it is among that range's keys), attend
                            over this rank's survivors -> partial (m, l, o[128])
     all-gather partials    [world][n_q][132] float32
  3. merge   (every rank)  log-sum-exp merge -> out [n_q][128]

`SeqShardedDecoder` is the host logic (ranges, bases, tail appends, the phase
order); the kernels come from `ops` (default: the sm_100a kernels through the
C ABI) and the collective from `allgather(tensor) -> [world, *shape]`.

Peer-memory exchange (`Mailbox`, `decode_step_p2p`): the same phases with
both all-gathers replaced by the kernels' own stores into every rank's mailbox
over NVLink (CUDA IPC mappings) and epoch flags (include/adamas_b200.h,
"sequence sharding over peer memory"): no NCCL call and no host sync per step.
"""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import ADAMAS_STATUS_PEER_TIMEOUT, AdamasRuntimeError, check, load

HEAD_DIM = 128
PARTIAL_STRIDE = 132
KEY_INDEX_BITS = 23  # global token index field of a key


def _ptr(t):
    return C.c_void_p(0 if t is None else t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class CudaSeqOps:
    """The three device phases through the C ABI (include/adamas_b200.h)."""

    def __init__(self):
        self.L = load()

    def local_candidates(self, cache, q, k_new, v_new, append: bool, base: int, budget: int, stream=None, out=None):
        n_q = q.numel() // HEAD_DIM
        keys = out if out is not None else torch.empty((n_q, budget), dtype=torch.int32, device=q.device)  # u32 bits
        check(self.L.adamas_seq_local_candidates(cache.h, _ptr(q), n_q, _ptr(k_new if append else None),
                                                 _ptr(v_new if append else None), int(append), base, budget,
                                                 _ptr(keys), _stream(stream)))
        return keys

    def select_attend(self, cache, q, gathered, budget: int, total_len: int, base: int, want_idx=False,
                      stream=None, out=None):
        n_q = q.numel() // HEAD_DIM
        world = gathered.shape[0]
        partial = out if out is not None else torch.empty((n_q, PARTIAL_STRIDE), dtype=torch.float32, device=q.device)
        gidx = torch.empty((n_q, budget), dtype=torch.int32, device=q.device) if want_idx else None
        check(self.L.adamas_seq_select_attend(cache.h, _ptr(q), n_q, _ptr(gathered.contiguous()), world, budget,
                                              total_len, base, _ptr(partial), _ptr(gidx), _stream(stream)))
        return partial, gidx

    def select_attend_merge(self, cache, q, gathered, budget: int, total_len: int, base: int, partials,
                            my_slot: int, want_idx=False, stream=None, out=None):
        """select_attend + lse_merge in one launch, for partials of the other
        ranks already in place (this rank's goes to partials[my_slot])."""
        n_q = q.numel() // HEAD_DIM
        world = gathered.shape[0]
        out = out if out is not None else torch.empty((n_q, HEAD_DIM), dtype=torch.float32, device=q.device)
        gidx = torch.empty((n_q, budget), dtype=torch.int32, device=q.device) if want_idx else None
        check(self.L.adamas_seq_select_attend_merge(cache.h, _ptr(q), n_q, _ptr(gathered.contiguous()), world, budget,
                                                    total_len, base, _ptr(partials), my_slot, _ptr(out), _ptr(gidx),
                                                    _stream(stream)))
        return out, gidx

    def lse_merge(self, partials, stream=None, out=None):
        world, n_q = partials.shape[0], partials.shape[1]
        out = out if out is not None else torch.empty((n_q, HEAD_DIM), dtype=torch.float32, device=partials.device)
        check(self.L.adamas_lse_merge(_ptr(partials.contiguous()), world, n_q, _ptr(out), _stream(stream)))
        return out


class SeqShardedDecoder:
    """One layer's decode over a sequence split across `world` ranks.

    cache     this rank's KvCache (or any object the ops accept) holding its
              contiguous token range; ranks are ordered: rank r's tokens precede
              rank r + 1's.
    lengths   tokens currently held by every rank (identical on all ranks; the
              host keeps it in step, no collective needed: only the tail rank
              appends, and everyone knows which rank that is).
    """

    def __init__(self, cache, rank: int, world: int, lengths, ops=None):
        if len(lengths) != world:
            raise ValueError("lengths must list every rank")
        self.cache, self.rank, self.world = cache, rank, world
        self.lengths = [int(x) for x in lengths]
        self.ops = ops if ops is not None else CudaSeqOps()
        self.tail = world - 1  # the last rank owns the sequence tail: global indices stay contiguous
        if sum(self.lengths) + 1 >= (1 << KEY_INDEX_BITS):
            raise ValueError("sequence too long for 23-bit global indices")

    @property
    def base(self) -> int:
        return sum(self.lengths[:self.rank])

    @property
    def total(self) -> int:
        return sum(self.lengths)

    # -- phases (the collective runs between them) -----------------------------
    def local(self, q, k_new, v_new, budget: int):
        append = self.rank == self.tail
        keys = self.ops.local_candidates(self.cache, q, k_new, v_new, append, self.base, budget)
        self.lengths[self.tail] += 1  # every rank: the tail rank appended
        return keys

    def attend(self, q, gathered, budget: int, want_idx=False):
        return self.ops.select_attend(self.cache, q, gathered, budget, self.total, self.base, want_idx)

    def merge(self, partials):
        return self.ops.lse_merge(partials)

    # -- one step with a collective ---------------------------------------------
    # -- peer-memory exchange ------------------------------------------------------
    def local_p2p(self, mailbox: Mailbox, q, k_new, v_new, stream=None):
        append = self.rank == self.tail
        n_q = q.numel() // HEAD_DIM
        check(self.ops.L.adamas_seq_p2p_local(self.cache.h, mailbox.h, _ptr(q), n_q, _ptr(k_new if append else None),
                                              _ptr(v_new if append else None), int(append), self.base,
                                              _stream(stream)))
        self.lengths[self.tail] += 1

    def attend_p2p(self, mailbox: Mailbox, q, want_idx=False, stream=None):
        n_q = q.numel() // HEAD_DIM
        gidx = torch.empty((n_q, mailbox.budget), dtype=torch.int32, device=q.device) if want_idx else None
        check(self.ops.L.adamas_seq_p2p_select_attend(self.cache.h, mailbox.h, _ptr(q), n_q, self.total, self.base,
                                                      _ptr(gidx), _stream(stream)))
        return gidx

    def merge_p2p(self, mailbox: Mailbox, stream=None):
        out = torch.empty((mailbox.n_q, HEAD_DIM), dtype=torch.float32, device="cuda")
        check(self.ops.L.adamas_seq_p2p_merge(mailbox.h, _ptr(out), _stream(stream)))
        return out

    def decode_step_p2p(self, mailbox: Mailbox, q, k_new, v_new, want_idx=False, check_status=True, stream=None):
        """One step over peer memory (every rank calls it; no collective call):
        adamas_seq_step_p2p, whose select/attend launch also does the merge.
        Ranks must run concurrently (one per GPU / process); ranks simulated
        in one stream use simulate_step_p2p's phase-by-phase order instead.
        check_status (default) synchronizes and raises if a peer wait timed
        out (the outputs of such a step are invalid); a tight loop may pass
        False and call mailbox.raise_on_timeout() periodically instead."""
        append = self.rank == self.tail
        n_q = q.numel() // HEAD_DIM
        out = torch.empty((n_q, HEAD_DIM), dtype=torch.float32, device=q.device)
        gidx = torch.empty((n_q, mailbox.budget), dtype=torch.int32, device=q.device) if want_idx else None
        total = self.total + 1  # after this step's append
        check(self.ops.L.adamas_seq_step_p2p(self.cache.h, mailbox.h, _ptr(q), n_q, _ptr(k_new if append else None),
                                             _ptr(v_new if append else None), int(append), self.base, total,
                                             _ptr(out), _ptr(gidx), _stream(stream)))
        self.lengths[self.tail] += 1
        if check_status:
            mailbox.raise_on_timeout()
        return out, gidx

    def decode_step(self, q, k_new, v_new, budget: int, allgather, want_idx=False):
        """allgather(t) -> tensor [world, *t.shape] in rank order."""
        keys = self.local(q, k_new, v_new, budget)
        gathered = allgather(keys)
        partial, gidx = self.attend(q, gathered, budget, want_idx)
        partials = allgather(partial)
        return self.merge(partials), gidx


class Mailbox:
    """One rank's mailbox of the peer-memory exchange (adamas_mailbox_*)."""

    HANDLE_BYTES = 64

    def __init__(self, rank: int, world: int, n_q: int, budget: int):
        self.L = load()
        self.h = None
        h = C.c_void_p()
        check(self.L.adamas_mailbox_create(C.byref(h), rank, world, n_q, budget))
        self.h, self.rank, self.world, self.n_q, self.budget = h, rank, world, n_q, budget

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(self.HANDLE_BYTES)
        check(self.L.adamas_mailbox_ipc_handle(self.h, buf))
        return buf.raw

    def connect(self, handles) -> None:
        """handles: every rank's ipc_handle(), rank order."""
        blob = b"".join(handles)
        check(self.L.adamas_mailbox_connect(self.h, C.create_string_buffer(blob, len(blob))))

    @staticmethod
    def connect_local(boxes) -> None:
        arr = (C.c_void_p * len(boxes))(*[b.h for b in boxes])
        check(load().adamas_mailbox_connect_local(arr, len(boxes)))

    def status(self) -> int:
        v = C.c_int(0)
        check(self.L.adamas_mailbox_status(self.h, C.byref(v)))
        return v.value

    def raise_on_timeout(self) -> None:
        """A peer wait that gave up (ADAMAS_STATUS_PEER_TIMEOUT) means this
        step read stale keys / partials: its outputs are invalid."""
        st = self.status()
        if st & ADAMAS_STATUS_PEER_TIMEOUT:
            raise AdamasRuntimeError(f"peer-memory exchange timed out on rank {self.rank} (status {st:#x}); "
                                     "the step's outputs are invalid")

    def close(self):
        if self.h:
            self.L.adamas_mailbox_destroy(self.h)
            self.h = None

    __del__ = close


def connect_mailboxes(mailbox: Mailbox, group=None) -> None:
    """Exchange the IPC handles over torch.distributed (setup only) and map every rank's mailbox."""
    import torch.distributed as dist
    handles = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, mailbox.ipc_handle(), group=group)
    mailbox.connect(handles)


def torch_allgather(group=None):
    """all_gather over torch.distributed (NCCL on GPUs, gloo on CPU)."""
    import torch.distributed as dist

    def gather(t):
        world = dist.get_world_size(group)
        t = t.contiguous()
        out = torch.empty((world * t.shape[0], *t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t, group=group)  # rank-major concatenation along dim 0
        return out.view(world, *t.shape)

    return gather


def simulate_step_p2p(decoders, mailboxes, qs, k_new, v_new, want_idx=False, check_status=True):
    """All ranks of one process over locally connected mailboxes, phase by phase."""
    for d, m, q in zip(decoders, mailboxes, qs):
        d.local_p2p(m, q, k_new, v_new)
    gidx = [d.attend_p2p(m, q, want_idx) for d, m, q in zip(decoders, mailboxes, qs)]
    outs = [d.merge_p2p(m) for d, m in zip(decoders, mailboxes)]
    if check_status:
        for m in mailboxes:
            m.raise_on_timeout()
    return outs, gidx


def simulate_step(decoders, qs, k_new, v_new, budget: int, want_idx=False):
    """All ranks of one process (e.g. several shards on one GPU): the same
    phases, with the all-gathers done by stacking."""
    keys = [d.local(q, k_new, v_new, budget) for d, q in zip(decoders, qs)]
    gathered = torch.stack(keys)
    parts = [d.attend(q, gathered, budget, want_idx) for d, q in zip(decoders, qs)]
    partials = torch.stack([p for p, _ in parts])
    outs = [d.merge(partials) for d in decoders]
    return outs, [g for _, g in parts]
