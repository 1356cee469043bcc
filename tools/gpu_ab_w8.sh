#!/bin/bash
# correctness of the 8-warp build through the GPU tests, then A/B vs the 16-warp build
ADAMAS_LIB=$PWD/variants/lib_w8.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
bash tools/ab.sh lib_w16 lib_w8
