#!/bin/bash
mkdir -p gpurun_out
bash tools/ab.sh base4:0 st512:0 > gpurun_out/ab_st512.txt 2>&1
ADAMAS_LIB=$PWD/variants/st512.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/st512_bench.json 2>&1
