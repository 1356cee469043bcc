#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/spec_debug.py > gpurun_out/spec_debug.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_spec.py tests/test_gpu_seqshard.py -q 2>&1 | tail -30 > gpurun_out/pytest_spec.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python -m pytest tests/test_gpu_shapes.py -q -x -k config4 2>&1 | tail -30 > gpurun_out/pytest_cfg4.txt
