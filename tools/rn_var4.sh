for v in "X=1" "FCT_ROWNORM_VAR=3" "FCT_ROWNORM_VAR=2"; do
  printf "%s " "$v"; env $v timeout 300 python bench.py --config 4 --rows 16777216 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rownorm ms', round(d['stages_ms']['rownorm']['mean'],3))"
  env $v FCT_DEBUG=1 timeout 300 python bench.py --config 4 --rows 1048576 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 >/dev/null | grep "rownorm_ws2<" | head -1
done > gpurun_out/rn_var4.txt 2>&1
