#!/bin/bash
# ncu captures of every kernel on a measured path (current build), one process each (never multi-rank);
# summarised ON the box into gpurun_out/summ/ (the .ncu-rep files are too large to bring back)
mkdir -p gpurun_out/summ /tmp/ncu
NCU="ncu --set full --clock-control none --import-source on"
TAG=${TAG:-r02}
timeout 600 $NCU -k regex:fused_decode -s 8 -c 1 -o /tmp/ncu/fused -f python bench.py --steps 2 --warmup 3 --layers 4 --no-cpu-baseline --no-check > gpurun_out/ncu_fused.log 2>&1
timeout 600 $NCU -k regex:fused_decode -s 4 -c 1 -o /tmp/ncu/llama -f python bench.py --config llama128k --steps 2 --warmup 3 --layers 2 --no-cpu-baseline --no-check > gpurun_out/ncu_llama.log 2>&1
timeout 600 $NCU -k regex:fused_decode -s 4 -c 1 -o /tmp/ncu/batched -f python bench.py --config batched16 --steps 2 --warmup 3 --layers 2 --no-cpu-baseline --no-check > gpurun_out/ncu_batched.log 2>&1
timeout 600 $NCU -k regex:"fused_decode|seq_select|lse_merge" -s 12 -c 3 -o /tmp/ncu/seq -f python bench.py --config seqshard1m --steps 2 --warmup 3 --layers 2 --no-cpu-baseline > gpurun_out/ncu_seq.log 2>&1
timeout 600 $NCU -k regex:append_kernel -s 1 -c 1 -o /tmp/ncu/append -f python tools/prefill_bench.py --reps 1 > gpurun_out/ncu_append.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --layers 4 --no-cpu-baseline --no-check > gpurun_out/b_ncu.log 2>&1
for n in fused llama batched seq append; do
  [ -f /tmp/ncu/$n.ncu-rep ] && python tools/summarize_ncu.py --tag $TAG --rep /tmp/ncu/$n.ncu-rep --name $n --launches /none --out-dir gpurun_out/summ >> gpurun_out/summ.log 2>&1
done
python tools/summarize_ncu.py --tag $TAG --rep /none --launches gpurun_out/launches.csv --out-dir gpurun_out/summ >> gpurun_out/summ.log 2>&1
ls -la gpurun_out/summ
