#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:adamas_dev --csv --log-file gpurun_out/seq_launches.csv python bench.py --config seqshard1m --steps 2 --warmup 1 --no-cpu-baseline --no-check > gpurun_out/seq_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_decode -s 20 -c 1 -o gpurun_out/seq_fused python bench.py --config seqshard1m --steps 2 --warmup 1 --no-cpu-baseline --no-check > gpurun_out/seq_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seq_select -s 20 -c 1 -o gpurun_out/seq_sel python bench.py --config seqshard1m --steps 2 --warmup 1 --no-cpu-baseline --no-check > gpurun_out/seq_ncu3.log 2>&1
