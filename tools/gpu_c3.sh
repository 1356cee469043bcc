#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab_c3.txt
for c in 4 3 2; do for v in qpf qpf_l2pf; do
  r=$(ADAMAS_CLUSTER=$c ADAMAS_LIB=$PWD/variants/$v.so timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), d['parity']['status'])" 2>&1 | tail -1)
  echo "C=$c $v: $r" >> gpurun_out/ab_c3.txt
done; done
