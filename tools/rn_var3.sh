# K2 variants at the cfg-4 shape (2^24 rows): rownorm stage ms
for v in "X=1" "FCT_ROWNORM_NOKEEP=1" "FCT_ROWNORM_NOKEEP=1 FCT_ROWNORM_VAR=3" "FCT_ROWNORM_NOKEEP=1 FCT_ROWNORM_VAR=2"; do
  printf "%s " "$v"; env $v timeout 300 python bench.py --config 4 --rows 16777216 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rownorm ms', round(d['stages_ms']['rownorm']['mean'],3))"
done > gpurun_out/rn_var3.txt 2>&1
