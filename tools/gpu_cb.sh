#!/bin/bash
mkdir -p gpurun_out
ADAMAS_LIB=$PWD/variants/cb.so timeout 900 python -m pytest tests/test_gpu_parity.py -k "append or encode" -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_cb.txt
for rep in 1 2; do for v in base17 cb; do
  echo "$v rep$rep: $(ADAMAS_LIB=$PWD/variants/$v.so timeout 300 python tools/prefill_bench.py 2>/dev/null | cut -c1-60)"
done; done > gpurun_out/ab_cb.txt
