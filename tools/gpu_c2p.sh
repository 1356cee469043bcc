#!/bin/bash
mkdir -p gpurun_out
ADAMAS_DBG=64 ADAMAS_QSPLIT=1 ADAMAS_P=4 ADAMAS_CLUSTER=4 timeout 600 python tools/phase_profile.py --heads 32 --kv-heads 8 --seq 131072 --layers 8 > gpurun_out/phase_c2_p4.txt 2>&1
ADAMAS_DBG=64 timeout 600 python tools/phase_profile.py --heads 32 --kv-heads 8 --seq 131072 --layers 8 > gpurun_out/phase_c2_q4.txt 2>&1
timeout 600 python bench.py --config seqshard1m --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_seqshard1m.json 2> gpurun_out/cfg_seqshard1m.err
