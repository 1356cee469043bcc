#!/bin/bash
mkdir -p gpurun_out
for spec in "0 0" "1 2" "1 4" "2 2"; do
  set -- $spec
  if [ "$1" = "0" ]; then
    r=$(timeout 300 python bench.py --config batched16 --steps 10 --warmup 3 --no-cpu-baseline --no-check 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['value'])")
  else
    r=$(ADAMAS_QSPLIT=$1 ADAMAS_CLUSTER=$2 timeout 300 python bench.py --config batched16 --steps 10 --warmup 3 --no-cpu-baseline --no-check 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['value'])")
  fi
  echo "qsplit $1 cluster $2: $r"
done > gpurun_out/c3plan.txt
