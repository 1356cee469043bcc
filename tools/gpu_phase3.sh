#!/bin/bash
mkdir -p gpurun_out
ADAMAS_DBG=64 timeout 600 python tools/phase_profile.py --layers 2 > gpurun_out/phase_l2res.txt 2>&1
ADAMAS_DBG=65600 timeout 600 python tools/phase_profile.py --layers 8 > gpurun_out/phase_scanonly.txt 2>&1
ADAMAS_DBG=65600 timeout 600 python tools/phase_profile.py --layers 2 > gpurun_out/phase_scanonly_l2res.txt 2>&1
