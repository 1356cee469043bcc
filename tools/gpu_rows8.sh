#!/bin/bash
mkdir -p gpurun_out
AB_ARGS="--config batched16" bash tools/ab.sh base16:0 rows8:0 > gpurun_out/ab_rows8.txt 2>&1
