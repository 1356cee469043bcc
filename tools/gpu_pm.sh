#!/bin/bash
mkdir -p gpurun_out
bash tools/ab.sh base8:0 pmerge:0 > gpurun_out/ab_pmerge.txt 2>&1
AB_ARGS="--config llama128k" bash tools/ab.sh base8:0 pmerge:0 >> gpurun_out/ab_pmerge.txt 2>&1
