#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/spec_debug2.py > gpurun_out/spec_debug2.txt 2>&1
timeout 300 python tools/seq_debug.py 2 131072 p2p > gpurun_out/seq_debug.txt 2>&1
timeout 300 python tools/seq_debug.py 2 131072 ag >> gpurun_out/seq_debug.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/seq_debug.py 2 131072 ag > gpurun_out/seq_memcheck.txt 2>&1
