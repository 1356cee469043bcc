#!/bin/bash
mkdir -p gpurun_out
AB_ARGS="--config seqshard1m" bash tools/ab.sh base8:0 late:0 > gpurun_out/ab_late.txt 2>&1
