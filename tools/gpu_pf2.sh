#!/bin/bash
mkdir -p gpurun_out
bash tools/ab.sh base2:0 pfn:0 nopf:0 > gpurun_out/ab_pf.txt 2>&1
timeout 300 python tools/prefill_bench.py > gpurun_out/prefill.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:append_kernel -c 1 -o gpurun_out/prefill_append python tools/prefill_bench.py --reps 1 > gpurun_out/prefill_ncu.log 2>&1
