# K2: CTA end-time spread (DIAG=8) and the CTA-0 timeline (rebuild with kTraceBuild = true) at cfg 5 and cfg 4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for c in "5 33554432" "4 67108864"; do set -- $c
  echo "== cfg $1 spread"; FCT_ROWNORM_DIAG=8 timeout 300 python bench.py --config $1 --rows $2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 >/dev/null | grep "CTAs:" | tail -2
done > gpurun_out/rn_trace_c5.txt 2>&1
sed -i 's/constexpr bool kTraceBuild = false/constexpr bool kTraceBuild = true/' paper_1207_4684_b200/csrc/rownorm_ws2.cu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for c in "5 33554432" "4 16777216"; do set -- $c
  for v in "FCT_ROWNORM_DIAG=16" "FCT_ROWNORM_DIAG=17"; do
    echo "== cfg $1 $v"; env $v timeout 300 python bench.py --config $1 --rows $2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 >/dev/null | grep "fct trace" | grep -v "trace] *[0-9]*:" | grep -v "event [0-5]" | tail -8
  done
done >> gpurun_out/rn_trace_c5.txt 2>&1
sed -i 's/constexpr bool kTraceBuild = true/constexpr bool kTraceBuild = false/' paper_1207_4684_b200/csrc/rownorm_ws2.cu
cat gpurun_out/rn_trace_c5.txt
