# K2 variants: fp64 M in shared vs global memory (one more tile buffer), epilogue group counts; 2^24 rows, cfg-4 shape
mkdir -p gpurun_out; : > gpurun_out/rn_m64.txt
run() { echo "== $1" >> gpurun_out/rn_m64.txt; env $1 timeout 300 python bench.py --config 4 --rows 16777216 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rownorm ms', round(d['stages_ms']['rownorm']['mean'],3))" >> gpurun_out/rn_m64.txt; env $1 FCT_DEBUG=1 FCT_ROWNORM_DIAG=8 timeout 300 python bench.py --config 4 --rows 16777216 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 >/dev/null | grep "rownorm_ws2<\|waited" | sort | uniq | head -30 >> gpurun_out/rn_m64.txt; }
run X=1
run FCT_ROWNORM_M64G=1
run "FCT_ROWNORM_M64G=1 FCT_ROWNORM_VAR=3"
run "FCT_ROWNORM_M64G=1 FCT_ROWNORM_VAR=2"
cat gpurun_out/rn_m64.txt
