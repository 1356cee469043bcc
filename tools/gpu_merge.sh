#!/bin/bash
mkdir -p gpurun_out/summ2 /tmp/ncu
timeout 900 python -m pytest tests/test_gpu_seqshard.py tests/test_gpu_parity.py tests/test_gpu_shapes.py -k "seq or config4" -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_seq.txt
timeout 600 python bench.py --config seqshard1m --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_seqshard1m.json 2> gpurun_out/cfg_seqshard1m.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"seq_select|lse_merge" -s 8 -c 2 -o /tmp/ncu/seq2 -f python bench.py --config seqshard1m --steps 2 --warmup 3 --layers 2 --no-cpu-baseline > gpurun_out/ncu_seq2.log 2>&1
python tools/summarize_ncu.py --tag r02z2 --rep /tmp/ncu/seq2.ncu-rep --name seq --launches /none --out-dir gpurun_out/summ2 >> gpurun_out/summ2.log 2>&1
for h in 8 4; do for c in 4 8 16; do
  ADAMAS_CLUSTER=$c timeout 300 python bench.py --heads $h --kv-heads $h --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/proxy_h${h}_c$c.json 2>&1
done; done
