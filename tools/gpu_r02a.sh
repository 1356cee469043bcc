#!/bin/bash
# round 2: new boundary/shape/head-shard tests, full gpu suite, bench with the parity check, proxies
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
for h in 16 8 4; do
  timeout 600 python bench.py --heads $h --kv-heads $h --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/proxy_longchat_h$h.json 2>&1
done
for kv in 4 2 1; do
  timeout 600 python bench.py --config batched16 --heads $((kv*4)) --kv-heads $kv --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/proxy_batched_kv$kv.json 2>&1
done
ls -la gpurun_out
