#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
bash tools/ab.sh base2:0 owner:0 > gpurun_out/ab_owner.txt 2>&1
for c in llama128k batched16; do
  for v in base2 owner; do
    ADAMAS_LIB=$PWD/variants/$v.so timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/${v}_$c.json 2>&1
  done
done
