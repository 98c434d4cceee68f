# K2 stage times on a config shape: default, DIAG=1 (no fp64 recompute), DIAG=2 (no epilogue arithmetic), per-warp waits
# usage: CFG=5 ROWS=33554432 VARS="X=1 FCT_ROWNORM_DIAG=1" bash tools/rn_stage.sh
CFG=${CFG:-5}; R=${ROWS:-33554432}; OUT=gpurun_out/rn_stage_c${CFG}.txt
: > $OUT
for v in ${VARS:-X=1 FCT_ROWNORM_DIAG=1 FCT_ROWNORM_DIAG=2}; do
  echo "== cfg $CFG rows $R $v" >> $OUT
  env $v timeout 300 python bench.py --config $CFG --rows $R --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>gpurun_out/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rownorm ms', round(d['stages_ms']['rownorm']['mean'],3), 'sketch ms', round(d['stages_ms']['sketch']['mean'],3), 'step ms', round(d['ms_per_step'],3), d['roofline_all']['l1_rownorm']['kernel_instance'])" >> $OUT 2>&1 || tail -5 gpurun_out/err.txt >> $OUT
done
if [ -n "$PROF" ]; then
  echo "== DIAG=8" >> $OUT
  FCT_ROWNORM_DIAG=8 timeout 300 python bench.py --config $CFG --rows $R --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 >/dev/null | grep "fct prof" | grep -v "cta " | sort | uniq -c | sort -rn | head -12 >> $OUT
fi
cat $OUT
