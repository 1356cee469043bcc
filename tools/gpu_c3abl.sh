#!/bin/bash
# config 3 (batched 16 x 32K): which phases set the period (diagnostics build stop switches)
mkdir -p gpurun_out
AB_ARGS="--config batched16" bash tools/ab.sh prod:0 diag:0 diag:65536 diag:131072 diag:524288 diag:262144 > gpurun_out/abl_batched16.txt 2>&1
ADAMAS_DBG=64 timeout 600 python tools/phase_profile.py --heads 32 --kv-heads 8 --seq 32768 --layers 4 --seqs 16 > gpurun_out/phase_batched16.txt 2>&1
