# one GPU iteration: parity tests, phase profile, short bench
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for c in 4 8; do echo "== cluster $c"; timeout 200 python tools/phase_profile.py --cluster $c --layers 4; done 2>&1
timeout 400 python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>&1 | tail -1
