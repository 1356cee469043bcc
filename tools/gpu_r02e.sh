#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
for c in llama128k batched16 seqshard1m; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
done
for h in 16 8 4; do
  timeout 600 python bench.py --heads $h --kv-heads $h --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/proxy_longchat_h$h.json 2>&1
done
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_sizes or exchange_topologies or heavy_ties or batched" > gpurun_out/san_memcheck.txt 2>&1
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_sizes[4] or heavy_ties" > gpurun_out/san_racecheck.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_sizes or exchange_topologies or heavy_ties" > gpurun_out/san_synccheck.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_seqshard.py -q -x -k "not two_processes" > gpurun_out/san_memcheck_seq.txt 2>&1
