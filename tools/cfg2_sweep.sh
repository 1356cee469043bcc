for rep in 1 2; do
for e in "X=0" "ADAMAS_QSPLIT=1 ADAMAS_CLUSTER=4 ADAMAS_P=4" "ADAMAS_QSPLIT=2 ADAMAS_CLUSTER=4 ADAMAS_P=2" "ADAMAS_QSPLIT=2 ADAMAS_CLUSTER=8" "ADAMAS_QSPLIT=1 ADAMAS_CLUSTER=8 ADAMAS_P=2"; do
  r=$(env $e timeout 300 python bench.py --config llama128k --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3))" 2>&1 | tail -1)
  echo "$e: $r"
done; done
