#!/bin/bash
mkdir -p gpurun_out
./tools/cluster_occ 200 > gpurun_out/cluster_occ.txt 2>&1; ./tools/cluster_occ 100 >> gpurun_out/cluster_occ.txt 2>&1
timeout 300 python tools/phase_profile.py --cluster 4 --layers 8 > gpurun_out/phase_c4.txt 2>&1
ADAMAS_DBG=64 timeout 300 python tools/phase_profile.py --cluster 4 --layers 8 > gpurun_out/phase_c4_gt.txt 2>&1
for e in "ADAMAS_CLUSTER=4" "ADAMAS_CLUSTER=4 ADAMAS_P=2" "ADAMAS_CLUSTER=2 ADAMAS_P=4"; do
  echo "== h16 $e" >> gpurun_out/proxy2.txt
  env $e timeout 300 python bench.py --heads 16 --kv-heads 16 --steps 20 --warmup 3 --no-cpu-baseline --no-check 2>&1 | tail -1 | head -c 200 >> gpurun_out/proxy2.txt; echo >> gpurun_out/proxy2.txt
  echo "== h4 $e" >> gpurun_out/proxy2.txt
  env $e timeout 300 python bench.py --heads 4 --kv-heads 4 --steps 20 --warmup 3 --no-cpu-baseline --no-check 2>&1 | tail -1 | head -c 200 >> gpurun_out/proxy2.txt; echo >> gpurun_out/proxy2.txt
done
