mkdir -p gpurun_out; : > gpurun_out/rn_var.txt
run() { echo "== $1" >> gpurun_out/rn_var.txt; env $1 timeout 300 python bench.py --config 4 --rows 16777216 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rownorm ms', round(d['stages_ms']['rownorm']['mean'],3))" >> gpurun_out/rn_var.txt; env $1 FCT_ROWNORM_DIAG=8 timeout 300 python bench.py --config 4 --rows 16777216 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 >/dev/null | grep "waited" | awk '{print $4, $6}' | sort | uniq -c | head -8 >> gpurun_out/rn_var.txt; }
run X=1
run FCT_ROWNORM_NOKEEP=1
run FCT_ROWNORM_VAR=2
run FCT_ROWNORM_VAR=0
run FCT_ROWNORM_VAR=3
cat gpurun_out/rn_var.txt
