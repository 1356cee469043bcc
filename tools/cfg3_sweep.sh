# batched16 split options (qsplit / cluster / smem cap), one bench line each
for e in "X=0" "ADAMAS_CLUSTER=2 ADAMAS_SMEM_KB=220" "ADAMAS_QSPLIT=4 ADAMAS_CLUSTER=1 ADAMAS_SMEM_KB=220" "ADAMAS_QSPLIT=1 ADAMAS_CLUSTER=2 ADAMAS_SMEM_KB=220" "ADAMAS_QSPLIT=2 ADAMAS_CLUSTER=1 ADAMAS_SMEM_KB=220 ADAMAS_STAGES=2" "ADAMAS_QSPLIT=4 ADAMAS_CLUSTER=2 ADAMAS_SMEM_KB=220"; do
  r=$(env $e timeout 300 python bench.py --config batched16 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['config'].get('us_per_layer_step',0),1))" 2>&1 | tail -1)
  echo "$e: $r"
done
