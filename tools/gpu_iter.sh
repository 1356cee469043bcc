#!/bin/bash
# One GPU iteration: parity tests, phase profile, short bench (with and without PDL).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/pytest_gpu.txt
python paper_2510_18413_b200/build.py --diag > /dev/null 2>&1; timeout 300 python tools/phase_profile.py --cluster ${CLUSTER:-4} --layers 8 > gpurun_out/phase.txt 2>&1
timeout 400 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err
ADAMAS_NO_PDL=1 timeout 400 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_iter_nopdl.json 2>> gpurun_out/bench_iter.err
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/phase.txt
for f in bench_iter bench_iter_nopdl; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', round(d['value'],3), 'e2e', round(d['e2e']['value'],3), 'frac', round(d['roofline']['frac'],3))"; done
