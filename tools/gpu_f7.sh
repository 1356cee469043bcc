#!/bin/bash
mkdir -p gpurun_out
AB_ARGS="--config llama128k" bash tools/ab.sh base13:0 f7all:0 > gpurun_out/ab_f7all.txt 2>&1
bash tools/ab.sh base13:0 f7all:0 >> gpurun_out/ab_f7all.txt 2>&1
