#!/bin/bash
# A/B: two CTAs per SM (consecutive launches co-reside) and/or an L2 prefetch of the rank's codes beyond the ring
mkdir -p gpurun_out
bash tools/ab.sh base:0 v2:0 v2pf:0 v1pf:0 > gpurun_out/ab2cta.txt 2>&1
ADAMAS_LIB=$PWD/variants/v2pf.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/v2pf_bench.json 2>&1
for c in llama128k batched16; do
  for v in base v2pf; do
    ADAMAS_LIB=$PWD/variants/$v.so timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/${v}_$c.json 2>&1
  done
done
