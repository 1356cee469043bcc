#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 300 python tools/prefill_bench.py > gpurun_out/prefill.json 2>&1
timeout 300 python tools/prefill_bench.py --chunk 4096 > gpurun_out/prefill_c4096.json 2>&1
timeout 600 python bench.py --config seqshard1m --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_seqshard1m.json 2> gpurun_out/cfg_seqshard1m.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:append8 -c 1 -o gpurun_out/prefill_append8 python tools/prefill_bench.py --reps 1 > gpurun_out/prefill_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seq_select -s 20 -c 1 -o gpurun_out/seq_sel2 python bench.py --config seqshard1m --steps 2 --warmup 1 --no-cpu-baseline --no-check > gpurun_out/seq_ncu3.log 2>&1
