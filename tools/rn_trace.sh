# K2 CTA-0 timeline (FCT_ROWNORM_DIAG bit 16), cfg-4 shape, 2^24 rows; DIAG 17 = no fp64 recompute, 18 = no epilogue arithmetic
mkdir -p gpurun_out
for v in "FCT_ROWNORM_DIAG=16" "FCT_ROWNORM_DIAG=17" "FCT_ROWNORM_DIAG=18" "FCT_ROWNORM_DIAG=16 FCT_ROWNORM_NOKEEP=1" "FCT_ROWNORM_DIAG=16 FCT_ROWNORM_NOKEEP=1 FCT_ROWNORM_VAR=3"; do
  echo "== $v"; env $v timeout 300 python bench.py --config 4 --rows 16777216 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 >/dev/null | grep "fct trace" | grep -v "trace] *[0-9]*:" 
done > gpurun_out/rn_trace.txt 2>&1
