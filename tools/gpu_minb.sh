#!/bin/bash
mkdir -p gpurun_out
AB_ARGS="--config seqshard1m" bash tools/ab.sh base7:0 minb2:0 minb3:0 > gpurun_out/ab_minb.txt 2>&1
