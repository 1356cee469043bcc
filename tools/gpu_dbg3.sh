#!/bin/bash
mkdir -p gpurun_out
for a in "40 1 1 12000" "40 1 1 5000" "40 1 1 8000" "40 1 1 9000" "40 1 1 16000" "40 2 1 24000" "6 1 1 12000" "-1 1 1 12000"; do timeout 120 python tools/spec_debug3.py $a 2>&1 | grep -v Warn; done > gpurun_out/spec_debug3.txt
timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python tools/spec_debug3.py 40 1 1 12000 > gpurun_out/spec_racecheck.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python tools/spec_debug3.py 40 1 1 12000 > gpurun_out/spec_memcheck.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck --print-limit 10 python tools/spec_debug3.py 40 1 1 12000 > gpurun_out/spec_synccheck.txt 2>&1
timeout 300 python tools/seq_debug.py 2 131072 p2p > gpurun_out/seq_debug.txt 2>&1
