mkdir -p gpurun_out; : > gpurun_out/rn_bo.txt
for h in 0 20 50 100 200; do
  echo "backoff $h: $(FCT_RN_BACKOFF=$h timeout 300 python bench.py --config 4 --rows 16777216 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['stages_ms']['rownorm']['mean'],3))")" >> gpurun_out/rn_bo.txt
done
cat gpurun_out/rn_bo.txt
