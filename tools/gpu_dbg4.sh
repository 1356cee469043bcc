#!/bin/bash
mkdir -p gpurun_out
{
for i in 1 2; do timeout 120 python tools/spec_debug3.py 40 1 1 8000; done
for i in 1 2; do ADAMAS_NO_PDL=1 timeout 120 python tools/spec_debug3.py 40 1 1 8000; done
for i in 1 2; do ADAMAS_STAGES=8 ADAMAS_SMEM_KB=226 timeout 120 python tools/spec_debug3.py 40 1 1 8000; done
for i in 1 2; do ADAMAS_STAGES=2 timeout 120 python tools/spec_debug3.py 40 1 1 8000; done
for i in 1 2; do ADAMAS_STAGES=2 timeout 120 python tools/spec_debug3.py -1 1 1 8000; done
for i in 1 2; do ADAMAS_STAGES=2 timeout 120 python tools/spec_debug3.py 40 4 1 24000; done
} 2>&1 | grep -v Warn > gpurun_out/spec_debug4.txt
