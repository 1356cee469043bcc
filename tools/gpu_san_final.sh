#!/bin/bash
# sanitizers over the final build's fused instances (incl. the collected-mask and lean-candidates ones)
mkdir -p gpurun_out
SUB="tests/test_gpu_parity.py::test_fused_decode_step_matches_oracle tests/test_gpu_parity.py::test_fused_compaction_span_sizes tests/test_gpu_parity.py::test_fused_decode_heavy_ties tests/test_gpu_parity.py::test_batched_decode_matches_single tests/test_gpu_parity.py::test_encode_append_codes_bit_exact tests/test_gpu_parity.py::test_bulk_append_near_threshold_keys tests/test_gpu_seqshard.py"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --kernel-name kns=adamas_dev \
    python -m pytest $SUB -m gpu -q -x -p no:cacheprovider > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_$tool.txt
done
