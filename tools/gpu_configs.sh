#!/bin/bash
# bench lines for every BASELINE config on one GPU
mkdir -p gpurun_out
timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/cfg_longchat.json 2> gpurun_out/cfg_longchat.err
for c in llama128k batched16 seqshard1m; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
done
for c in longchat llama128k batched16 seqshard1m; do
  echo "== $c"; python -c "import json; d=json.load(open('gpurun_out/cfg_$c.json')); print(round(d['value'],3), 'us/token/layer; per layer-step', round(d['config']['us_per_layer_step'],2), 'us; e2e', round(d['e2e']['value'],3), 'frac', round(d['roofline']['frac'],3), 'clocks', d['clocks'])" || tail -5 gpurun_out/cfg_$c.err
done
