#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
for h in 16 8 4; do
  timeout 600 python bench.py --heads $h --kv-heads $h --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/proxy_longchat_h$h.json 2>&1
done
timeout 600 python bench.py --config seqshard1m --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_seqshard1m.json 2> gpurun_out/cfg_seqshard1m.err
