#!/bin/bash
mkdir -p gpurun_out
AB_ARGS="--config seqshard1m" bash tools/ab.sh base7:0 sel3:0 sel6:0 sel5:0 > gpurun_out/ab_sel5.txt 2>&1
