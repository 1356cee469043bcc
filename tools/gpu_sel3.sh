#!/bin/bash
mkdir -p gpurun_out
AB_ARGS="--config seqshard1m" bash tools/ab.sh base7:0 sel9:0 sel1:0 sel2:0 sel3:0 sel4:0 > gpurun_out/ab_sel3.txt 2>&1
