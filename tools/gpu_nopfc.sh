#!/bin/bash
mkdir -p gpurun_out
AB_ARGS="--config seqshard1m" bash tools/ab.sh base11:0 nopfc:0 > gpurun_out/ab_nopfc.txt 2>&1
