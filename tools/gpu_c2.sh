#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_seqshard.py tests/test_gpu_parity.py -k "seq" -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_seq.txt
timeout 600 python bench.py --config seqshard1m --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_seqshard1m.json 2> gpurun_out/cfg_seqshard1m.err
for spec in "1 4 4" "2 2 4" "1 2 8" "4 1 4"; do
  set -- $spec
  ADAMAS_QSPLIT=$1 ADAMAS_P=$2 ADAMAS_CLUSTER=$3 timeout 300 python bench.py --config llama128k --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/c2_q$1_p$2_c$3.json 2>&1
done
