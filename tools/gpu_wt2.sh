#!/bin/bash
mkdir -p gpurun_out
bash tools/ab.sh base:0 wt2:0 wt2pf:0 > gpurun_out/ab_wt2.txt 2>&1
