#!/bin/bash
# One GPU round: parity tests, smoke, bench line (+ reference arm), every
# config, prefill, ncu launch list + one full capture of the fused kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in llama128k batched16 seqshard1m harness_needle; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
done
timeout 300 python tools/prefill_bench.py > gpurun_out/prefill.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --layers 4 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_decode -s 8 -c 1 -o gpurun_out/prof_fused python bench.py --steps 2 --warmup 3 --layers 4 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
# config 2 (Llama GQA 128K): the q-split scan's L2 traffic
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_decode -s 4 -c 1 -o gpurun_out/prof_llama python bench.py --config llama128k --steps 2 --warmup 3 --layers 2 --no-cpu-baseline > gpurun_out/ncu_llama.log 2>&1
ls -la gpurun_out
