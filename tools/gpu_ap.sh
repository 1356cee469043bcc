#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/prefill_ab.txt
for rep in 1 2; do for v in base ap2 ap4 ap8; do
  echo "$v: $(ADAMAS_LIB=$PWD/variants/$v.so timeout 120 python tools/prefill_bench.py 2>&1 | tail -1)" >> gpurun_out/prefill_ab.txt
done; done
