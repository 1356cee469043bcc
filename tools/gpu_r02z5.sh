#!/bin/bash
# after the per-instance distance fold: pytest -m gpu and every bench line
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
for c in llama128k batched16 seqshard1m; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
done
for b in 64 256; do timeout 600 python bench.py --budget $b --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_longchat_k$b.json 2>&1; done
for h in 16 8 4; do
  timeout 600 python bench.py --heads $h --kv-heads $h --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/proxy_longchat_h$h.json 2>&1
done
for kv in 4 2 1; do
  timeout 600 python bench.py --config batched16 --heads $((kv*4)) --kv-heads $kv --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/proxy_batched_kv$kv.json 2>&1
done
