#!/bin/bash
# Round-2 closing evidence on one B200: pytest -m gpu, every bench line (configs 1-4, budgets,
# reference arm, head-shard proxies, prefill), ncu captures of every kernel on a measured path
# (summarised on the box: the .ncu-rep files are too large to bring back), the launch list,
# sanitizer logs and the config-1 phase timeline (diagnostics build).
mkdir -p gpurun_out/summ /tmp/ncu
TAG=${TAG:-r02z}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
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
timeout 300 python tools/prefill_bench.py > gpurun_out/prefill.json 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:fused_decode -s 8 -c 1 -o /tmp/ncu/fused -f python bench.py --steps 2 --warmup 3 --layers 4 --no-cpu-baseline --no-check > gpurun_out/ncu_fused.log 2>&1
timeout 600 $NCU -k regex:fused_decode -s 4 -c 1 -o /tmp/ncu/llama -f python bench.py --config llama128k --steps 2 --warmup 3 --layers 2 --no-cpu-baseline --no-check > gpurun_out/ncu_llama.log 2>&1
timeout 600 $NCU -k regex:fused_decode -s 4 -c 1 -o /tmp/ncu/batched -f python bench.py --config batched16 --steps 2 --warmup 3 --layers 2 --no-cpu-baseline --no-check > gpurun_out/ncu_batched.log 2>&1
timeout 600 $NCU -k regex:"fused_decode|seq_select|lse_merge" -s 12 -c 3 -o /tmp/ncu/seq -f python bench.py --config seqshard1m --steps 2 --warmup 3 --layers 2 --no-cpu-baseline > gpurun_out/ncu_seq.log 2>&1
timeout 600 $NCU -k regex:append -s 1 -c 1 -o /tmp/ncu/append -f python tools/prefill_bench.py --reps 1 > gpurun_out/ncu_append.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --layers 4 --no-cpu-baseline --no-check > gpurun_out/b_ncu.log 2>&1
for n in fused llama batched seq append; do
  [ -f /tmp/ncu/$n.ncu-rep ] && python tools/summarize_ncu.py --tag $TAG --rep /tmp/ncu/$n.ncu-rep --name $n --launches /none --out-dir gpurun_out/summ >> gpurun_out/summ.log 2>&1
done
python tools/summarize_ncu.py --tag $TAG --rep /none --launches gpurun_out/launches.csv --out-dir gpurun_out/summ >> gpurun_out/summ.log 2>&1
SUB_FUSED="tests/test_gpu_parity.py::test_fused_decode_step_matches_oracle tests/test_gpu_parity.py::test_fused_decode_cluster_sizes tests/test_gpu_parity.py::test_fused_decode_heavy_ties tests/test_gpu_parity.py::test_fused_decode_multi_cluster_units tests/test_gpu_parity.py::test_top_k_matches_oracle_dense_ties tests/test_gpu_parity.py::test_sparse_attention_tolerance tests/test_gpu_parity.py::test_encode_append_codes_bit_exact tests/test_gpu_parity.py::test_bulk_append_near_threshold_keys"
SUB_SEQ="tests/test_gpu_seqshard.py::test_seq_sharded_decode_matches_single_device tests/test_gpu_seqshard.py::test_seq_sharded_peer_exchange"
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --kernel-name kns=adamas_dev \
    python -m pytest $SUB_FUSED $SUB_SEQ -m gpu -q -x -p no:cacheprovider > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_$tool.txt
done
ADAMAS_DBG=64 timeout 600 python tools/phase_profile.py --layers 8 > gpurun_out/phase_longchat.txt 2>&1
ls -la gpurun_out gpurun_out/summ
