"""-m gpu: the head-sharded multi-GPU path of bench.py (heads are
independent) run as TWO processes through torchrun. On a one-GPU
box both ranks share cuda:0 (ADAMAS_BENCH_SAME_DEVICE=1) and the barrier /
max-over-ranks timing go over gloo (ADAMAS_BENCH_BACKEND=gloo); each rank
decodes its half of the heads and checks its last timed step against the
oracle (bench.py's parity check), and rank 0 reports the combined verdict."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config,extra", [
    ("longchat", ["--layers", "2"]),
    ("batched16", ["--layers", "1", "--seqs", "4"]),
])
def test_bench_head_shard_world2(config, extra):
    env = dict(os.environ, ADAMAS_BENCH_SAME_DEVICE="1", ADAMAS_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + (os.getpid() % 500)),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", config, "--steps", "2", "--warmup", "3",
           "--no-cpu-baseline", *extra]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "head-shard x2"
    assert d["config"]["heads_per_rank"] == 16
    assert d["parity"]["status"] == "ok", d["parity"]
    assert "every one of the 2 ranks" in d["parity"]["checked"]
