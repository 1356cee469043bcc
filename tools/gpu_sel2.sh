#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_seqshard.py tests/test_gpu_shapes.py tests/test_gpu_parity.py -k "seq or merge or config4" -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_seq.txt
timeout 600 python bench.py --config seqshard1m --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_seqshard1m.json 2> gpurun_out/cfg_seqshard1m.err
