#!/bin/bash
# current-build ncu of the config-1 and config-2 fused instances (distance fold 6) + the >8-rank merge test
mkdir -p gpurun_out/summ9 /tmp/ncu
timeout 600 python -m pytest tests/test_gpu_seqshard.py -k merge -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_merge.txt
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:fused_decode -s 8 -c 1 -o /tmp/ncu/fused -f python bench.py --steps 2 --warmup 3 --layers 4 --no-cpu-baseline --no-check > gpurun_out/ncu_fused.log 2>&1
timeout 600 $NCU -k regex:fused_decode -s 4 -c 1 -o /tmp/ncu/llama -f python bench.py --config llama128k --steps 2 --warmup 3 --layers 2 --no-cpu-baseline --no-check > gpurun_out/ncu_llama.log 2>&1
timeout 600 $NCU -k regex:fused_decode -s 4 -c 1 -o /tmp/ncu/batched -f python bench.py --config batched16 --steps 2 --warmup 3 --layers 2 --no-cpu-baseline --no-check > gpurun_out/ncu_batched.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --layers 4 --no-cpu-baseline --no-check > gpurun_out/b_ncu.log 2>&1
for n in fused llama batched; do
  python tools/summarize_ncu.py --tag r02z9 --rep /tmp/ncu/$n.ncu-rep --name $n --launches /none --out-dir gpurun_out/summ9 >> gpurun_out/summ9.log 2>&1
done
python tools/summarize_ncu.py --tag r02z9 --rep /none --launches gpurun_out/launches.csv --out-dir gpurun_out/summ9 >> gpurun_out/summ9.log 2>&1
timeout 600 $NCU -k regex:"fused_decode|seq_select" -s 8 -c 2 -o /tmp/ncu/seq -f python bench.py --config seqshard1m --steps 2 --warmup 3 --layers 2 --no-cpu-baseline > gpurun_out/ncu_seq.log 2>&1
python tools/summarize_ncu.py --tag r02z9 --rep /tmp/ncu/seq.ncu-rep --name seq --launches /none --out-dir gpurun_out/summ9 >> gpurun_out/summ9.log 2>&1
