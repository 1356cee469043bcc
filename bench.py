#!/usr/bin/env python3
"""Adamas decode hot-path benchmark (BASELINE.json metric).

metric  decode self-attn us/token/layer @32K, budget 128 (lower is better),
        plus the dominant kernel's achieved HBM GB/s against the measured peak.
config  LongChat-7B attention shape (BASELINE configs[1]): 32 heads x 128,
        S = 32768, batch 1, budget 128, bf16 K/V, synthetic data; one "step"
        decodes one token through all 32 layers' attention (32 distinct
        per-layer caches, 17 GiB > L2, so no flush is needed between layers or
        steps). Each layer runs the full hot path in ONE fused launch: append
        (k, v, codes), encode q, code scan, top-k select, sparse attention.
N > 1   one rank per GPU, heads sharded across ranks (no data-path collective;
        the layer's time is the max over ranks) -> "scaling": "strong".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode self-attn µs/token/layer @32K, budget 128; code-scan HBM GB/s vs peak"
UNIT = "us/token/layer"

# BASELINE.json configs (shapes per step; "seqs" = independent requests)
CONFIGS = {
    "longchat": dict(heads=32, kv_heads=32, seq=32768, budget=128, layers=32, seqs=1),
    "llama128k": dict(heads=32, kv_heads=8, seq=131072, budget=128, layers=16, seqs=1),
    "batched16": dict(heads=32, kv_heads=8, seq=32768, budget=128, layers=4, seqs=16),
    "seqshard1m": dict(heads=32, kv_heads=8, seq=1048576 // 8, budget=128, layers=16, seqs=1),
}
WORKLOAD = {
    "longchat": "LongChat-7B attention decode: {heads} heads ({kv_heads} kv) x 128, S={seq}, batch 1, budget {budget}",
    "llama128k": "Llama-3.1-8B GQA attention decode: {heads} q / {kv_heads} kv heads x 128, S={seq}, batch 1, "
                 "budget {budget}",
    "batched16": "batched decode: {seqs} requests x S={seq}, Llama-3.1-8B shape ({heads} q / {kv_heads} kv), "
                 "per-request top-{budget}",
    "seqshard1m": "1M-token context, {heads} q / {kv_heads} kv heads, one rank's share of an 8-way sequence split "
                  "(S={seq} per rank): local candidates + distributed select/attend + LSE merge, budget {budget}",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="longchat", choices=sorted(CONFIGS) + ["harness_needle"],
                    help="BASELINE.json config: longchat (configs[1], the headline), llama128k (configs[2]), "
                         "batched16 (configs[3]), seqshard1m (configs[4], per-rank work of the 8-way split)")
    ap.add_argument("--heads", type=int, default=None)
    ap.add_argument("--kv-heads", type=int, default=None)
    ap.add_argument("--seq", type=int, default=None)
    ap.add_argument("--budget", type=int, default=None)
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--seqs", type=int, default=None, help="independent sequences (requests) per step")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=11)
    ap.add_argument("--no-check", action="store_true",
                    help="skip the oracle check of the last timed step (default: checked, outside the timed region)")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="seqshard1m at N > 1: peer-memory mailboxes (default) or NCCL all-gathers")
    a = ap.parse_args()
    for k, v in CONFIGS.get(a.config, {}).items():
        if getattr(a, k) is None:
            setattr(a, k, v)
    return a


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


TRAFFIC_KEY = {"longchat": "fused_decode_kernel", "llama128k": "fused_decode_kernel[llama128k]",
               "batched16": "fused_decode_kernel[batched16]",
               "seqshard1m": "fused_decode_kernel[seqshard1m candidates]"}


def load_traffic(config="longchat"):
    """dram bytes per launch of the config's fused kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(TRAFFIC_KEY.get(config, ""), {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """Samples SM clocks and throttle reasons through NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index=0, period=0.002):
        self.period = period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------- reference arm
def cpu_reference(args, n_heads, steps, warmup):
    """The unmodified reference operators (oracle/_ref) on the host cores:
    one layer of n_heads per-head caches (S tokens), each step = append +
    encode(q) + score_all + top_k + sparse_attention for every head, heads over
    all host threads. Returns (median us per layer-step, threads, sample)."""
    from oracle.bindings import Reference
    ref = Reference()
    threads = os.cpu_count() or 1
    layer = ref.layer_build(n_heads, args.seq - 1, 128, args.dtype == "bf16", 4242, threads)
    try:
        t = ref.layer_decode(layer, args.budget, threads, warmup + steps)
    finally:
        ref.layer_free(layer)
    t = list(t[warmup:])
    # the reference is single-threaded: also one thread, a shorter sample
    layer1 = ref.layer_build(n_heads, args.seq - 1, 128, args.dtype == "bf16", 4242, threads)
    try:
        t1 = list(ref.layer_decode(layer1, args.budget, 1, 1 + 3)[1:])
    finally:
        ref.layer_free(layer1)
    sample = (f"1 layer = {n_heads} heads x S={args.seq} (reference KvCache per head, prebuilt), "
              f"{len(t)} decode steps, median, heads over {threads} threads; 1 thread: "
              f"{statistics.median(t1):.1f} us ({len(t1)} steps); simd={ref.simd_level()}; cpu={_cpu_model()}")
    return float(statistics.median(t)), threads, sample


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    ws, rank, _ = dist_setup()
    if rank != 0:
        return
    v, threads, sample = cpu_reference(args, args.heads, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v / 1000.0, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"LongChat-7B attention decode, {args.heads} heads x 128, S={args.seq}, "
                               f"budget {args.budget}, {args.dtype}-valued K/V widened to f64, 1 layer per step",
                   "layers_per_step": 1},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ----------------------------------------------------------------------------- our arm
def _prefill(ad, torch, n_kv, S, dtype, gen, cap_extra=1):
    """A cache with S tokens (bulk encode-append, 4096 tokens per launch)."""
    c = ad.KvCache(n_kv, S + cap_extra, dtype)
    done = 0
    while done < S:
        n = min(4096, S - done)
        k = torch.randn((n, n_kv, 128), generator=gen, device="cuda").to(dtype)
        v = torch.randn((n, n_kv, 128), generator=gen, device="cuda").to(dtype)
        c.update(k, v)
        done += n
    return c


def parity_check(torch, caches, qs, out, idx, s_last, S, B, layers):
    """Checker, outside every timed region (the oracle is test infrastructure
    and is never measured): the LAST TIMED step's selection and output of the
    given layers (request 0), as the timed graph left them, against the CPU
    oracle over the cache contents that step saw (S tokens, the appended one
    included). Indices bit-exact, output within the north-star tolerance."""
    import numpy as np

    from oracle.bindings import Oracle  # checker only
    from tests.gpu_helpers import oracle_decode, rel_err

    oracle = Oracle()
    worst = 0.0
    for l in layers:
        c = caches[l][0]
        K = c.keys()[:, :S].float().permute(1, 0, 2).contiguous().cpu().numpy()
        V = c.values()[:, :S].float().permute(1, 0, 2).contiguous().cpu().numpy()
        q = qs[s_last, l, 0].float().cpu().numpy()
        _, _, eidx, eout = oracle_decode(oracle, K, V, q, B)
        got_idx = idx[l, 0].cpu().numpy()
        keep = min(B, S)
        if not np.array_equal(got_idx[:, :keep], eidx):
            bad = int((got_idx[:, :keep] != eidx).any(axis=1).sum())
            return {"status": "MISMATCH", "detail": f"layer {l}: indices differ in {bad} of {q.shape[0]} heads"}
        err = float(rel_err(out[l, 0].cpu().numpy(), eout).max())
        worst = max(worst, err)
        if err > (1e-2 if c.dtype == torch.bfloat16 else 1e-3):
            return {"status": "MISMATCH", "detail": f"layer {l}: output rel err {err:.2e}"}
    return {"status": "ok", "checked": f"last timed step, layers {list(layers)}, request 0, every q-head: indices "
                                       f"bit-exact vs the oracle, max output rel err {worst:.2e}"}


def _timed_graph(torch, dist, ws, body, steps, local, sample_clocks=False):
    """Capture `steps` calls of body(s, stream) in one CUDA graph, warm replay,
    then time one replay with CUDA events on the capture stream (max over
    ranks). Returns (elapsed_ms, clock summary or None)."""
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        st = torch.cuda.current_stream()
        for s in range(steps):
            body(s, st)
    graph.replay()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(local) if sample_clocks else None
    if clk:
        clk.__enter__()
    e0.record(stream)
    graph.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    if clk:
        clk.__exit__()
    ms = e0.elapsed_time(e1)
    if ws > 1:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt[0])
        dist.barrier()
    del graph
    return ms, (clk.summary() if clk else None)


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2510_18413_b200 as ad

    ws, rank, local = dist_setup()
    # protocol checks of the N > 1 paths on a one-GPU box (never for numbers):
    # ADAMAS_BENCH_SAME_DEVICE=1 puts every rank on cuda:0, ADAMAS_BENCH_BACKEND=gloo
    if os.environ.get("ADAMAS_BENCH_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    if ws > 1:
        backend = os.environ.get("ADAMAS_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    seqshard = args.config == "seqshard1m"
    if not seqshard and (args.heads % ws or args.kv_heads % ws):
        raise SystemExit("heads must divide across ranks")
    n_q, n_kv = (args.heads, args.kv_heads) if seqshard else (args.heads // ws, args.kv_heads // ws)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    es = 2 if dtype == torch.bfloat16 else 4
    S, L, B, NS = args.seq, args.layers, args.budget, args.seqs
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1234 + rank)

    # prefill S-1 tokens per (layer, sequence); the timed step appends token S
    caches = [[_prefill(ad, torch, n_kv, S - 1, dtype, gen) for _ in range(NS)] for _ in range(L)]
    torch.cuda.synchronize()
    for row in caches:
        for c in row:
            c.raise_on_degenerate()

    total_steps = args.warmup + args.steps
    qs = torch.randn((total_steps, L, NS, n_q, 128), generator=gen, device="cuda").to(dtype)
    ks = torch.randn((total_steps, L, NS, n_kv, 128), generator=gen, device="cuda").to(dtype)
    vs = torch.randn((total_steps, L, NS, n_kv, 128), generator=gen, device="cuda").to(dtype)
    out = torch.empty((L, NS, n_q, 128), dtype=torch.float32, device="cuda")
    idx = torch.empty((L, NS, n_q, B), dtype=torch.int32, device="cuda")

    if seqshard:
        # N = 1: one rank's share of the 8-way split (the other shards' keys
        # are synthesized from this shard's keys with shifted indices, one
        # kernel). N > 1: a world-way split of an N x S context, rank r owning
        # [r S, (r + 1) S); the two exchanges go through peer memory (the
        # kernels store into every rank's CUDA-IPC mailbox, --exchange p2p,
        # default) or NCCL all-gathers (--exchange nccl).
        from paper_2510_18413_b200.seqshard import CudaSeqOps, Mailbox, connect_mailboxes, torch_allgather
        ops = CudaSeqOps()
        n_virtual = 8 if ws == 1 else ws
        my_slot = rank % n_virtual
        base = my_slot * S
        tail = my_slot == n_virtual - 1
        if ws > 1 and args.exchange == "p2p":
            mbox = Mailbox(rank, ws, n_q, B)
            connect_mailboxes(mbox)
            Lh = ops.L
            from paper_2510_18413_b200.seqshard import _ptr, _stream

            def step(s, st):
                for l in range(L):
                    c = caches[l][0]
                    rc = Lh.adamas_seq_step_p2p(c.h, mbox.h, _ptr(qs[s, l, 0]), n_q, _ptr(ks[s, l, 0]),
                                                _ptr(vs[s, l, 0]), int(tail), base, n_virtual * S, _ptr(out[l, 0]),
                                                None, _stream(st))
                    if rc:
                        raise RuntimeError(Lh.adamas_last_error().decode())
                    if tail:
                        c.truncate(S - 1)
        else:
            gather = torch_allgather() if ws > 1 else None
            keys_all = torch.empty((L, n_virtual, n_q, B), dtype=torch.int32, device="cuda")
            parts_all = torch.empty((L, n_virtual, n_q, 132), dtype=torch.float32, device="cuda")
            if gather is None:
                # N = 1: the other 7 shards' slots of the gathered keys and partials are filled ONCE, before
                # the timed region, from this shard's first step (same distances, indices moved to their
                # ranges); each timed step's kernels write this rank's slot in place, so the step is exactly
                # this rank's three launches (candidates, select/attend, merge) with no data-path copies
                shard_off = ((torch.arange(n_virtual, device="cuda", dtype=torch.int32) - my_slot) * S).view(-1, 1, 1)
                for l in range(L):
                    c = caches[l][0]
                    k0 = ops.local_candidates(c, qs[0, l, 0], ks[0, l, 0], vs[0, l, 0], tail, base, B)
                    keys_all[l].copy_(k0.unsqueeze(0) + shard_off)
                    p0, _ = ops.select_attend(c, qs[0, l, 0], keys_all[l], B, n_virtual * S, base)
                    parts_all[l].copy_(p0.unsqueeze(0).expand(n_virtual, -1, -1))
                    if tail:
                        c.truncate(S - 1)

            def step(s, st):
                for l in range(L):
                    c = caches[l][0]
                    if gather is not None:
                        keys = ops.local_candidates(c, qs[s, l, 0], ks[s, l, 0], vs[s, l, 0], tail, base, B, stream=st)
                        keys_all[l].copy_(gather(keys))
                        part, _ = ops.select_attend(c, qs[s, l, 0], keys_all[l], B, n_virtual * S, base, stream=st)
                        parts_all[l].copy_(gather(part))
                        ops.lse_merge(parts_all[l], stream=st, out=out[l, 0])
                    else:
                        # the default N > 1 flow (peer memory) fuses select / attend / merge into one
                        # launch; here the other shards' partials are in place, so the same fusion applies
                        ops.local_candidates(c, qs[s, l, 0], ks[s, l, 0], vs[s, l, 0], tail, base, B, stream=st,
                                             out=keys_all[l, my_slot])
                        ops.select_attend_merge(c, qs[s, l, 0], keys_all[l], B, n_virtual * S, base, parts_all[l],
                                                my_slot, stream=st, out=out[l, 0])
                    if tail:
                        c.truncate(S - 1)
    else:
        def step(s, st):
            for l in range(L):
                if NS == 1:
                    caches[l][0].decode_step(qs[s, l, 0], ks[s, l, 0], vs[s, l, 0], B, out=out[l, 0],
                                             idx=idx[l, 0], stream=st)
                else:
                    ad.decode_step_batched(caches[l], qs[s, l], ks[s, l], vs[s, l], B, out=out[l], idx=idx[l],
                                           stream=st)
            for row in caches:  # keep S fixed: the next step re-appends at position S-1
                for c in row:
                    c.truncate(S - 1)

    stream0 = torch.cuda.current_stream()
    for s in range(args.warmup):  # eager warm-up (also configures the kernels)
        step(s, stream0)
    torch.cuda.synchronize()

    # The timed steps run as one CUDA graph (no host launch overhead in the
    # device timeline); kernel time per launch is bounded by elapsed / launches.
    elapsed_ms, clocks = _timed_graph(torch, dist, ws, lambda s, st: step(args.warmup + s, st), args.steps, local,
                                      sample_clocks=True)
    parity = None
    if not args.no_check and not seqshard:  # every rank checks its own heads
        parity = parity_check(torch, caches, qs, out, idx, args.warmup + args.steps - 1, S, B,
                              sorted({0, L // 2, L - 1}))
        if ws > 1:
            bad = torch.tensor([0 if parity["status"] == "ok" else 1 + rank], device="cuda")
            dist.all_reduce(bad, op=dist.ReduceOp.MAX)
            if int(bad[0]) and parity["status"] == "ok":
                parity = {"status": "MISMATCH", "detail": f"on rank {int(bad[0]) - 1}"}
            elif parity["status"] == "ok":
                parity["checked"] += f"; every one of the {ws} ranks checked its own heads"
    # Isolated latency: the same timed graph with programmatic dependent launch
    # off, so no launch overlaps its predecessor (what a layer costs when other
    # kernels sit between attention layers and none of them releases it early).
    isolated = None
    if not seqshard:
        saved_tuning = ad.get_tuning()
        ad.set_tuning(no_pdl=1)
        n_iso = min(args.steps, 10)
        iso_ms, _ = _timed_graph(torch, dist, ws, lambda s, st: step(args.warmup + s, st), n_iso, local)
        ad.set_tuning(**saved_tuning)
        isolated = {"value": iso_ms * 1000.0 / (n_iso * L * NS), "unit": UNIT,
                    "note": "same steps with programmatic dependent launch off: no layer overlaps its predecessor"}
    # seqshard: candidates + select / attend / merge (N = 1 proxy and the p2p step when every select CTA
    # is co-resident: 2 launches per layer); the NCCL flow adds lse_merge (3)
    launches_per_step = L * ((3 if ws > 1 and args.exchange == "nccl" else 2) if seqshard else 1)
    ms_per_step = elapsed_ms / args.steps
    tokens_per_layer = NS  # one decoded token per sequence per layer
    us_per_token_layer = ms_per_step * 1000.0 / (L * tokens_per_layer)
    kern_ms = elapsed_ms / (args.steps * L)  # per layer launch (all phases of the layer)

    # e2e through the public API with HOST buffers: per step the pinned H2D of
    # q, k, v, the decode launches and the D2H of the attention outputs, all
    # captured as one graph the way a serving loop drives the library: inputs
    # and outputs double-buffered, copies on side streams, so step s + 1's
    # upload and step s - 1's download overlap step s's decode (every step's
    # copies stay inside the timed region).
    n_e2e = min(args.steps, 16)
    hq = qs[:n_e2e].cpu().pin_memory()
    hk = ks[:n_e2e].cpu().pin_memory()
    hv = vs[:n_e2e].cpu().pin_memory()
    hout = torch.empty((n_e2e, L, NS, n_q, 128), dtype=torch.float32).pin_memory()
    dq = [torch.empty_like(qs[:1]) for _ in range(2)]
    dk = [torch.empty_like(ks[:1]) for _ in range(2)]
    dv = [torch.empty_like(vs[:1]) for _ in range(2)]
    dout = [torch.empty_like(out) for _ in range(2)]
    qs_save, ks_save, vs_save, out_save = qs, ks, vs, out
    up, down = torch.cuda.Stream(), torch.cuda.Stream()

    def e2e_graph():
        nonlocal qs, ks, vs, out
        st = torch.cuda.current_stream()
        ev = lambda: torch.cuda.Event()  # noqa: E731
        ready, done, freed = [ev(), ev()], [ev(), ev()], [ev(), ev()]
        fork = ev()
        fork.record(st)
        up.wait_event(fork)
        down.wait_event(fork)
        for s in range(n_e2e):
            b = s & 1
            with torch.cuda.stream(up):
                if s >= 2:
                    up.wait_event(done[b])  # step s - 2 has consumed input buffer b
                dq[b][0].copy_(hq[s], non_blocking=True)
                dk[b][0].copy_(hk[s], non_blocking=True)
                dv[b][0].copy_(hv[s], non_blocking=True)
                ready[b].record(up)
            st.wait_event(ready[b])
            if s >= 2:
                st.wait_event(freed[b])  # step s - 2's output has been downloaded
            qs, ks, vs, out = dq[b], dk[b], dv[b], dout[b]
            step(0, st)
            qs, ks, vs, out = qs_save, ks_save, vs_save, out_save
            done[b].record(st)
            with torch.cuda.stream(down):
                down.wait_event(done[b])
                hout[s].copy_(dout[b], non_blocking=True)
                freed[b].record(down)
        st.wait_stream(up)
        st.wait_stream(down)

    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):
        e2e_graph()
    g2.replay()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    g2.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if ws > 1:
        tt = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt[0])
    del g2
    if not torch.isfinite(hout).all() and not int(os.environ.get("ADAMAS_DBG", "0")):
        raise SystemExit("non-finite attention output")
    h2d = (hq[0].numel() + hk[0].numel() + hv[0].numel()) * es
    d2h = hout[0].numel() * 4

    # roofline of the fused kernel: algorithmic bytes per launch
    bytes_launch = NS * (n_kv * S * 32 + n_q * min(B, S) * 2 * 128 * es)
    if seqshard:  # this shard's survivors only: about B / 8 rows per q-head
        bytes_launch = n_kv * S * 32 + n_q * (B // 8) * 2 * 128 * es
    achieved = bytes_launch / (kern_ms * 1e-3) / 1e9
    peak, peak_kind = load_peaks()
    traffic = load_traffic(args.config)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and args.config == "longchat":
        try:
            v, threads, sample = cpu_reference(args, args.heads, args.cpu_steps, 2)
            cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample}
        except Exception as e:  # reference build absent
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        par = (f"sequence-shard x{n_virtual} (rank {my_slot} of the split, world {ws}"
               + (f", {args.exchange} exchange)" if ws > 1 else ", other shards synthesized)") if seqshard
               else f"head-shard x{ws}")
        line = {
            "metric": METRIC, "value": us_per_token_layer, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False,
            "scaling": "weak" if seqshard else "strong", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic",
            "config": {"workload": WORKLOAD[args.config].format(**vars(args)) + f", {args.dtype} K/V, "
                                   f"{L} layers per step",
                       "name": args.config, "layers_per_step": L, "sequences": NS, "heads_per_rank": n_q,
                       "kv_heads_per_rank": n_kv, "parallelism": par,
                       "us_per_layer_step": ms_per_step * 1000.0 / L,
                       "l2": f"no flush: {L * NS} distinct per-(layer, request) caches, "
                             f"{L * NS * n_kv * S * (256 * es + 32) / 2**30:.1f} GiB > 126 MB L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "frac_of_8tbs": achieved / 8000.0,
                         "kernel": ("fused candidates + seq_select_attend with the merge (2 launches per layer; "
                                    "+ lse_merge with --exchange nccl at N > 1)"
                                    if seqshard else "fused_decode_kernel"), "bytes_per_launch": bytes_launch,
                         "kernel_us": kern_ms * 1000.0, "peak_source": peak_kind},
            "e2e": {"value": e2e_ms * 1000.0 / (n_e2e * L * tokens_per_layer), "unit": UNIT,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": args.steps * launches_per_step,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "parity": parity,
            "isolated": isolated,
        }
        print(json.dumps(line))
        if parity and parity["status"] != "ok":
            raise SystemExit(f"parity check failed: {parity['detail']}")
    if ws > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- f3: the sweep harness
HARNESS_METRIC = "needle sweep us/query (adamas + window + quest x budgets 16/32/64 + recall reference)"
HARNESS_UNIT = "us/query"
HARNESS = dict(seq=8192, head_dim=128, queries=100, budgets=(16, 32, 64), position=4096, snr=10.0)


def _harness_sweep(H):
    return H.SweepConfig(budgets=list(HARNESS["budgets"]),
                         policies=[H.PolicySpec("adamas"), H.PolicySpec("window", sink=4),
                                   H.PolicySpec("quest", page_size=16)], measure_output_error=False)


def harness_cpu_reference(n_queries):
    """The reference's run_sweep (oracle/_ref) over the acceptance needle shape
    (acceptance.cpp:290-325) on n_queries queries, minus its own workload
    generation (timed separately through Workload::instance). Returns
    (us per query, sample text)."""
    from oracle.bindings import Reference
    from paper_2510_18413_b200 import harness as H

    ref = Reference()
    spec = H.WorkloadSpec(seed=2024, seq_len=HARNESS["seq"], head_dim=HARNESS["head_dim"], num_queries=n_queries,
                          distribution="planted_needle", position=HARNESS["position"], snr=HARNESS["snr"])
    t0 = time.perf_counter()
    ref.run_sweep(spec, _harness_sweep(H))
    t_sweep = time.perf_counter() - t0
    t0 = time.perf_counter()
    for qi in range(n_queries):
        ref.workload_instance(spec, qi)
    t_gen = time.perf_counter() - t0
    us = (t_sweep - t_gen) * 1e6 / n_queries
    sample = (f"reference run_sweep, planted needle S={HARNESS['seq']} d={HARNESS['head_dim']}, {n_queries} queries "
              f"x budgets {list(HARNESS['budgets'])} x adamas/window/quest, 1 thread: {t_sweep:.2f} s minus its "
              f"workload generation {t_gen:.2f} s")
    return us, sample


def run_harness(args):
    """f3: the sweep harness's per-query work on the GPU. One step = one sweep
    over HARNESS['queries'] planted-needle instances (each its own 8K x 128 fp64
    keys, 839 MB per step, > L2): build_cache, adamas select, quest select and
    the dot-product recall reference for every budget. `value`: instances
    resident in HBM; `e2e`: harness.run_sweep on host instances (H2D of keys,
    values and queries, D2H of the selections, host-side rows)."""
    import numpy as np
    import torch

    from paper_2510_18413_b200 import harness as H

    ws, rank, local = dist_setup()
    torch.cuda.set_device(local)
    S, d, nq, budgets = HARNESS["seq"], HARNESS["head_dim"], HARNESS["queries"], HARNESS["budgets"]
    rng = np.random.default_rng(1234 + rank)
    insts = []
    for qi in range(nq):  # workload.cpp:136-152's planted needle, numpy RNG
        q = rng.standard_normal(d)
        K = rng.standard_normal((S, d))
        K[HARNESS["position"]] = HARNESS["snr"] * np.sqrt(d) / np.linalg.norm(q) * q + rng.standard_normal(d)
        insts.append(H.Instance(qi, q, K, rng.standard_normal((S, d)), HARNESS["position"]))
    Kd = torch.empty((nq, S, d), dtype=torch.float64, device="cuda")
    for i, x in enumerate(insts):
        Kd[i].copy_(torch.from_numpy(x.keys))
    Qd = torch.as_tensor(np.stack([x.query for x in insts]), device="cuda")
    sel = H.HarnessSelector(d, 2, True)
    pages = H.PageSelector(16, d)
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    parts = {"build": [], "select": [], "quest": [], "recall": []}

    def step(record):
        marks = [ev() for _ in range(5)]
        marks[0].record(stream)
        sel.build(Kd)
        marks[1].record(stream)
        for b in budgets:
            sel.select(Qd, b, "l1", 1)
        marks[2].record(stream)
        pages.build(Kd)
        for b in budgets:
            pages.select(Qd, b, 1)
        marks[3].record(stream)
        _, dots = H.dot_topk(Qd, Kd, 0, 1, want_scores=True)
        for b in budgets:
            H.topk_scores(dots, b)
        marks[4].record(stream)
        if record is not None:
            record.append(marks)

    for _ in range(args.warmup):
        step(None)
    torch.cuda.synchronize()
    rec = []
    clk = ClockSampler(local)
    with clk:
        e0, e1 = ev(), ev()
        e0.record(stream)
        for _ in range(args.steps):
            step(rec)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    for m in rec:
        for i, k in enumerate(parts):
            parts[k].append(m[i].elapsed_time(m[i + 1]))
    part_ms = {k: statistics.median(v) for k, v in parts.items()}
    # algorithmic bytes per phase (reads of keys / codes / scores, writes of codes / scores)
    key_b, code_b = nq * S * d * 8, nq * S * 32
    nb = len(budgets)
    n_pages = (S + 15) // 16
    alg = {"build": key_b + code_b, "select": nb * (code_b + 2 * nq * S * 4),
           "quest": key_b + (1 + nb) * 2 * nq * n_pages * d * 8, "recall": key_b + nq * S * 8 * (1 + nb)}
    dom = max(part_ms, key=part_ms.get)
    peak, peak_kind = load_peaks()
    achieved = alg[dom] / (part_ms[dom] * 1e-3) / 1e9
    # e2e: the public run_sweep on host instances
    sweep = _harness_sweep(H)
    n_e2e = max(1, min(args.steps, 3))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        rows = H.run_sweep(insts, sweep)
    torch.cuda.synchronize()
    e2e_us = (time.perf_counter() - t0) * 1e6 / (n_e2e * nq)
    hits = {c.budget: c.needle_fraction for c in H.needle_report(rows) if c.policy == "adamas-2bit-l1"}
    cpu = None
    if not args.no_cpu_baseline:
        v, sample = harness_cpu_reference(4)
        cpu = {"value": v, "unit": HARNESS_UNIT, "cores": 1, "kind": "reference", "sample": sample}
    launches = 1 + 3 * nb + 1 + 3 * nb + 1 + nb
    line = {
        "metric": HARNESS_METRIC, "value": ms * 1000.0 / nq, "unit": HARNESS_UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"acceptance needle sweep (acceptance.cpp:290-325 shape): {nq} planted-needle "
                               f"queries per step, S={S}, d={d}, budgets {list(budgets)}, adamas-2bit-l1 + "
                               f"window-sink4 + quest-p16, recall reference; numpy-generated instances",
                   "l2": f"no flush: {key_b / 2**20:.0f} MiB of keys per step > 126 MB L2",
                   "phase_ms": part_ms, "adamas_needle_fraction": hits},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "kernel": {"build": "hsel_encode_kernel", "select": "hsel_score+topk",
                                                 "quest": "hsel_page_*", "recall": "hsel_dot+topk"}[dom],
                     "bytes_per_launch": alg[dom], "phase": dom, "peak_source": peak_kind},
        "e2e": {"value": e2e_us, "unit": HARNESS_UNIT,
                "h2d_bytes_per_step": key_b + nq * d * 8, "d2h_bytes_per_step": nq * nb * 8 * (2 * 64 + 64)},
        "gpu_launches": args.steps * launches,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line))


def run_harness_reference(args):
    ws, rank, _ = dist_setup()
    if rank != 0:
        return
    v, sample = harness_cpu_reference(max(2, min(args.steps, 8)))
    print(json.dumps({
        "impl": "reference", "metric": HARNESS_METRIC, "value": v, "unit": HARNESS_UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v / 1000.0, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "acceptance needle sweep (reference run_sweep, per query)"},
        "cpu_baseline": {"value": v, "unit": HARNESS_UNIT, "cores": 1, "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": HARNESS_UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    args = parse()
    if args.config == "harness_needle":
        return run_harness_reference(args) if args.impl == "reference" else run_harness(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
