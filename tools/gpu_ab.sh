#!/bin/bash
# Parity suite on the current build, then an interleaved A/B of variants/*.so
# at the bench config (args: variant names), plus optional extra configs.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
tail -3 gpurun_out/pytest_gpu.txt
bash tools/ab.sh "$@" 2>&1 | tee gpurun_out/ab.txt
for c in ${AB_CONFIGS:-}; do
  for v in "$@"; do
    r=$(ADAMAS_LIB=$PWD/variants/$v.so timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3))")
    echo "$c $v: $r" | tee -a gpurun_out/ab.txt
  done
done
