#!/bin/bash
mkdir -p gpurun_out
AB_ARGS="--config batched16" bash tools/ab.sh d6:0 d7:0 d8:0 > gpurun_out/ab_d6.txt 2>&1
AB_ARGS="--config llama128k" bash tools/ab.sh d6:0 d7:0 d8:0 >> gpurun_out/ab_d6.txt 2>&1
bash tools/ab.sh d6:0 d7:0 d8:0 >> gpurun_out/ab_d6.txt 2>&1
