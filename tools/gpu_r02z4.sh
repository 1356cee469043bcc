#!/bin/bash
# closing evidence after the sequence-shard work: smoke, pytest -m gpu, every bench line,
# ncu of the sequence-shard kernels, sanitizers over the fused / seq subset
mkdir -p gpurun_out/summ4 /tmp/ncu
TAG=r02z4
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in llama128k batched16 seqshard1m; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
done
for b in 64 256; do timeout 600 python bench.py --budget $b --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_longchat_k$b.json 2>&1; done
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:"fused_decode|seq_select" -s 8 -c 2 -o /tmp/ncu/seq -f python bench.py --config seqshard1m --steps 2 --warmup 3 --layers 2 --no-cpu-baseline > gpurun_out/ncu_seq.log 2>&1
python tools/summarize_ncu.py --tag $TAG --rep /tmp/ncu/seq.ncu-rep --name seq --launches /none --out-dir gpurun_out/summ4 >> gpurun_out/summ4.log 2>&1
SUB="tests/test_gpu_parity.py::test_fused_decode_step_matches_oracle tests/test_gpu_parity.py::test_seq_shard_candidates_multi_cluster tests/test_gpu_seqshard.py"
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --kernel-name kns=adamas_dev \
    python -m pytest $SUB -m gpu -q -x -p no:cacheprovider > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_$tool.txt
done
ls -la gpurun_out/summ4
