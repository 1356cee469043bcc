#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab_ldg.txt
for rep in 1 2; do for v in qpf ldg; do for a in "--no-prefetch" ""; do
  r=$(ADAMAS_LIB=$PWD/variants/$v.so timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline $a 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['e2e']['value'],3), d['parity']['status'])" 2>&1 | tail -1)
  echo "$v $a: $r" >> gpurun_out/ab_ldg.txt
done; done; done
for v in qpf ldg; do
  r=$(ADAMAS_LIB=$PWD/variants/$v.so timeout 300 python bench.py --config llama128k --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), d['parity']['status'])" 2>&1 | tail -1)
  echo "llama $v: $r" >> gpurun_out/ab_ldg.txt
done
