# K2 CTA-0 timeline (needs kTraceBuild = true in rownorm_ws2.cu), cfg-4 shape, 2^24 rows
for v in "FCT_ROWNORM_DIAG=16" "FCT_ROWNORM_DIAG=17" "FCT_ROWNORM_DIAG=18" "FCT_ROWNORM_DIAG=16 FCT_ROWNORM_SS=1"; do
  echo "== $v"; env $v timeout 300 python bench.py --config 4 --rows 16777216 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 >/dev/null | grep "fct trace" | grep -v "trace] *[0-9]*:" | grep -v "event [0-5]" | tail -8
done > gpurun_out/rn_trace2.txt 2>&1
