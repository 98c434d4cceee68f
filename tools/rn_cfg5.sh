# K2 at the cfg-5 shard geometry (2^25 x 100, k = 29): stage breakdown by FCT_ROWNORM_DIAG and per-warp waits
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
R=${ROWS:-33554432}
: > gpurun_out/rn_cfg5.txt
for v in "X=1" "FCT_ROWNORM_DIAG=1" "FCT_ROWNORM_DIAG=2" "FCT_ROWNORM_DIAG=3" ${EXTRA}; do
  echo "== $v" >> gpurun_out/rn_cfg5.txt
  env $v timeout 300 python bench.py --config 5 --rows $R --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>gpurun_out/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rownorm ms', round(d['stages_ms']['rownorm']['mean'],3), 'sketch ms', round(d['stages_ms']['sketch']['mean'],3), d['roofline_all']['l1_rownorm']['kernel_instance'])" >> gpurun_out/rn_cfg5.txt 2>&1 || tail -5 gpurun_out/err.txt >> gpurun_out/rn_cfg5.txt
done
echo "== DIAG=8" >> gpurun_out/rn_cfg5.txt
FCT_ROWNORM_DIAG=8 timeout 300 python bench.py --config 5 --rows $R --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 >/dev/null | grep "fct prof" | grep -v "cta " >> gpurun_out/rn_cfg5.txt
cat gpurun_out/rn_cfg5.txt
