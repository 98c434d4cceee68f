# K2 CTA-0 timeline at the cfg-5 and cfg-4 geometries (rebuilds with kTraceBuild = true on the box)
sed -i 's/constexpr bool kTraceBuild = false/constexpr bool kTraceBuild = true/' paper_1207_4684_b200/csrc/rownorm_ws2.cu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for c in "5 33554432" "4 16777216"; do set -- $c
  for v in "FCT_ROWNORM_DIAG=16" "FCT_ROWNORM_DIAG=17"; do
    echo "== cfg $1 $v"; env $v timeout 300 python bench.py --config $1 --rows $2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 >/dev/null | grep "fct trace" | grep -v "trace] *[0-9]*:" | grep -v "event [0-5]" | tail -8
  done
done > gpurun_out/rn_trace_c5.txt 2>&1
cat gpurun_out/rn_trace_c5.txt
