#!/bin/bash
mkdir -p gpurun_out
AB_ARGS="--config batched16" bash tools/ab.sh base12:0 lop3:0 > gpurun_out/ab_lop3.txt 2>&1
AB_ARGS="--config llama128k" bash tools/ab.sh base12:0 lop3:0 >> gpurun_out/ab_lop3.txt 2>&1
bash tools/ab.sh base12:0 lop3:0 >> gpurun_out/ab_lop3.txt 2>&1
