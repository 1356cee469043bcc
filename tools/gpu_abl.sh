#!/bin/bash
mkdir -p gpurun_out
bash tools/ab.sh diag:0 diag:524288 diag:131072 diag_nopf:0 diag_nopf:524288 > gpurun_out/ablation2.txt 2>&1
