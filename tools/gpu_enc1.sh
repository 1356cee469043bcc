#!/bin/bash
mkdir -p gpurun_out
bash tools/ab.sh base3:0 enc1:0 nofp64:0 > gpurun_out/ab_enc1.txt 2>&1
