#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
AB_ARGS="--config batched16" bash tools/ab.sh base15:0 collsel:0 > gpurun_out/ab_collsel.txt 2>&1
bash tools/ab.sh base15:0 collsel:0 >> gpurun_out/ab_collsel.txt 2>&1
AB_ARGS="--config llama128k" bash tools/ab.sh base15:0 collsel:0 >> gpurun_out/ab_collsel.txt 2>&1
AB_ARGS="--config seqshard1m" bash tools/ab.sh base15:0 collsel:0 >> gpurun_out/ab_collsel.txt 2>&1
