set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 2 --layers 4 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_decode -s 8 -c 2 -o gpurun_out/prof_fused python bench.py --steps 2 --warmup 2 --layers 4 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
