#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do for v in base14 stcs; do
  echo "$v rep$rep: $(ADAMAS_LIB=$PWD/variants/$v.so timeout 300 python tools/prefill_bench.py 2>/dev/null)"
done; done > gpurun_out/ab_ap4.txt
