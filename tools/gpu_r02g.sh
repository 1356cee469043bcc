#!/bin/bash
# round 2 (session 3): state check after the container restore + sanitizer logs
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
for c in llama128k batched16 seqshard1m; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
done
SUB_FUSED="tests/test_gpu_parity.py::test_fused_decode_step_matches_oracle tests/test_gpu_parity.py::test_fused_decode_cluster_sizes tests/test_gpu_parity.py::test_fused_decode_heavy_ties tests/test_gpu_parity.py::test_fused_decode_multi_cluster_units tests/test_gpu_parity.py::test_top_k_matches_oracle_dense_ties tests/test_gpu_parity.py::test_sparse_attention_tolerance"
SUB_SEQ="tests/test_gpu_seqshard.py::test_seq_sharded_decode_matches_single_device tests/test_gpu_seqshard.py::test_seq_sharded_peer_exchange"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --kernel-name kns=adamas_dev \
    python -m pytest $SUB_FUSED $SUB_SEQ -m gpu -q -x -p no:cacheprovider > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_$tool.txt
done
ls -la gpurun_out
