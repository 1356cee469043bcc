#!/bin/bash
# A/B with env settings: args "variant|ENV=V ENV2=V" ...
for rep in 1 2; do
  for spec in "$@"; do
    v=${spec%%|*}; e=""; [[ "$spec" == *"|"* ]] && e=${spec#*|}
    r=$(env $e ADAMAS_LIB=$PWD/variants/$v.so timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['e2e']['value'],3))")
    echo "$spec rep$rep: $r"
  done
done
