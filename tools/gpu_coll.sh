#!/bin/bash
mkdir -p gpurun_out
ADAMAS_LIB=$PWD/variants/coll.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_multistep.py tests/test_gpu_seqshard.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_coll.txt
AB_ARGS="--config batched16" bash tools/ab.sh base15:0 coll:0 > gpurun_out/ab_coll.txt 2>&1
bash tools/ab.sh base15:0 coll:0 >> gpurun_out/ab_coll.txt 2>&1
AB_ARGS="--config llama128k" bash tools/ab.sh base15:0 coll:0 >> gpurun_out/ab_coll.txt 2>&1
