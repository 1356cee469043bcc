#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
ADAMAS_SPEC_MARGIN=-1 timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/bench_nospec.json 2>&1
ADAMAS_SPEC_MARGIN=3 timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/bench_m3.json 2>&1
ADAMAS_SPEC_MARGIN=10 timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/bench_m10.json 2>&1
for c in llama128k batched16 seqshard1m; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
done
ADAMAS_DBG=64 timeout 300 python tools/phase_profile.py --cluster 4 --layers 8 > gpurun_out/phase_c4_gt.txt 2>&1
