#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_multistep.py -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_wt.txt
bash tools/ab.sh base:0 wt:0 wtpf:0 > gpurun_out/ab_wt.txt 2>&1
for c in llama128k batched16; do
  for v in base wtpf; do
    ADAMAS_LIB=$PWD/variants/$v.so timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/${v}_$c.json 2>&1
  done
done
