#!/bin/bash
# Phase profile of the fused decode kernel at the bench shape, several cluster sizes.
mkdir -p gpurun_out
for c in ${CLUSTERS:-4 8}; do echo "== cluster $c"; timeout 200 python tools/phase_profile.py --cluster $c --layers 4 2>&1; done > gpurun_out/phase.txt
for c in ${CLUSTERS:-4 8}; do echo "== cluster $c"; ADAMAS_CLUSTER=$c timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'])"; done >> gpurun_out/phase.txt 2>&1
