timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_decode -s 8 -c 1 -o gpurun_out/prof_fused python bench.py --steps 2 --warmup 2 --layers 4 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 400 python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>&1 | tail -1
