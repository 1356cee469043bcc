#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in llama128k batched16 seqshard1m; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
done
for b in 64 256; do timeout 600 python bench.py --budget $b --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_longchat_k$b.json 2>&1; done
for h in 16 8 4; do
  timeout 600 python bench.py --heads $h --kv-heads $h --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/proxy_longchat_h$h.json 2>&1
done
for kv in 4 2 1; do
  timeout 600 python bench.py --config batched16 --heads $((kv*4)) --kv-heads $kv --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/proxy_batched_kv$kv.json 2>&1
done
timeout 300 python tools/prefill_bench.py > gpurun_out/prefill.json 2>&1
