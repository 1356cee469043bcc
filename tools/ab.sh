#!/bin/bash
# A/B of library builds (and ADAMAS_DBG settings) on the same box: bench value
# per variant, interleaved. Args: variant[:dbg] ...
for rep in 1 2; do
  for vd in "$@"; do
    v=${vd%%:*}; d=0; [[ "$vd" == *:* ]] && d=${vd##*:}
    r=$(ADAMAS_DBG=$d ADAMAS_LIB=$PWD/variants/$v.so timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-check $AB_ARGS 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['e2e']['value'],3))")
    echo "$vd rep$rep: $r"
  done
done
