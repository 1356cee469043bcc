#!/bin/bash
# ablation of the fused step (diagnostics build): which phases set the period
mkdir -p gpurun_out
bash tools/ab.sh prod:0 diag:0 diag:65536 diag:131072 diag:524288 diag:262144 diag:8 diag:65544 > gpurun_out/abl_32layers.txt 2>&1
AB_ARGS="--layers 1" bash tools/ab.sh prod:0 diag:0 diag:65536 diag:131072 > gpurun_out/abl_1layer.txt 2>&1
