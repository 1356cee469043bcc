#!/bin/bash
mkdir -p gpurun_out
bash tools/ab.sh base4:0 ms16:0 > gpurun_out/ab_ms16.txt 2>&1
