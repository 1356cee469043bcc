#!/bin/bash
mkdir -p gpurun_out
AB_ARGS="--config seqshard1m" bash tools/ab.sh base5:0 mbweak:0 > gpurun_out/ab_mbweak.txt 2>&1
ADAMAS_LIB=$PWD/variants/mbweak.so timeout 900 python -m pytest tests/test_gpu_seqshard.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_mbweak.txt
