#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_seqshard.py tests/test_gpu_shapes.py tests/test_gpu_parity.py -k "seq or merge or config4 or cand" -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_staged.txt
AB_ARGS="--config seqshard1m" bash tools/ab.sh base18:0 staged:0 > gpurun_out/ab_staged.txt 2>&1
