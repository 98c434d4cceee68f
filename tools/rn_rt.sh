# K2 RT (row in TMEM) vs the KEEP path: parity, timeline and stage time at 2^24 rows of the cfg-4 shape
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rownorm" 2>&1 | tail -3 > gpurun_out/rn_rt_tests.txt
{
for v in "X=1" "FCT_ROWNORM_NORT=1" "FCT_ROWNORM_DIAG=32"; do
  echo "== $v"
  env $v timeout 300 python bench.py --config 4 --rows 16777216 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rownorm ms', round(d['stages_ms']['rownorm']['mean'],3))"
  env $v FCT_ROWNORM_DIAG=$(( ${v#FCT_ROWNORM_DIAG=} + 16 )) timeout 300 python bench.py --config 4 --rows 16777216 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 >/dev/null | grep "fct trace" | grep -v "trace] *[0-9]*:" | grep -v "event [0-5]" | tail -8
done
} > gpurun_out/rn_rt.txt 2>&1
cat gpurun_out/rn_rt_tests.txt
