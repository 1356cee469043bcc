#!/bin/bash
mkdir -p gpurun_out
bash tools/ab.sh base fence l2pf w8 w8l2pf > gpurun_out/ab3.txt 2>&1
AB_ARGS="--config llama128k --steps 20" bash tools/ab.sh base > gpurun_out/ab3_llama.txt 2>&1
AB_ARGS="--config seqshard1m --steps 20" bash tools/ab.sh base > gpurun_out/ab3_seq.txt 2>&1
ADAMAS_LIB=$PWD/variants/fence.so timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_sizes[4] or heavy_ties" > gpurun_out/san_racecheck2.txt 2>&1
timeout 300 python tools/prefill_bench.py > gpurun_out/prefill.json 2>&1
