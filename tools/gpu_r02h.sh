#!/bin/bash
# sanitizer logs over the fused / sequence-shard subset + a critical-path phase timeline (diagnostics build)
mkdir -p gpurun_out
SUB_FUSED="tests/test_gpu_parity.py::test_fused_decode_step_matches_oracle tests/test_gpu_parity.py::test_fused_decode_cluster_sizes tests/test_gpu_parity.py::test_fused_decode_heavy_ties tests/test_gpu_parity.py::test_fused_decode_multi_cluster_units tests/test_gpu_parity.py::test_top_k_matches_oracle_dense_ties tests/test_gpu_parity.py::test_sparse_attention_tolerance"
SUB_SEQ="tests/test_gpu_seqshard.py::test_seq_sharded_decode_matches_single_device tests/test_gpu_seqshard.py::test_seq_sharded_peer_exchange"
ADAMAS_DBG=64 timeout 600 python tools/phase_profile.py --layers 8 > gpurun_out/phase_longchat.txt 2>&1
ADAMAS_DBG=64 timeout 600 python tools/phase_profile.py --layers 8 --heads 32 --kv-heads 8 --seq 131072 > gpurun_out/phase_llama.txt 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --kernel-name kns=adamas_dev \
    python -m pytest $SUB_FUSED $SUB_SEQ -m gpu -q -x -p no:cacheprovider > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_$tool.txt
done
ls -la gpurun_out
