#!/bin/bash
mkdir -p gpurun_out
{ for a in "40 1 1 8000" "40 1 1 8000" "-1 1 1 8000" "6 1 1 8000"; do timeout 120 python tools/spec_debug5.py $a; done; } 2>&1 | grep -v Warn > gpurun_out/spec_debug5.txt
