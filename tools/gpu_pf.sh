#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab_pf.txt
for rep in 1 2; do for a in "" "--no-prefetch"; do
  r=$(timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline $a 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['e2e']['value'],3), d['parity']['status'])" 2>&1 | tail -1)
  echo "longchat $a: $r" >> gpurun_out/ab_pf.txt
done; done
ADAMAS_DBG=64 timeout 300 python tools/phase_profile.py --cluster 4 --layers 8 > gpurun_out/phase_pf.txt 2>&1
