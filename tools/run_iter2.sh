timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in 4 8; do echo "== cluster $c"; ADAMAS_CLUSTER=$c timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'])"; done
timeout 200 python tools/phase_profile.py --cluster 8 --layers 4 2>&1 | grep -v "thr_scan\|dsmem"
