# ncu --set full (source counters) of K2 at the cfg-4 and cfg-5 geometries, 2^22 rows each
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for c in 4 5; do
  ncu --set full --clock-control none --import-source on -k regex:rownorm_ws2 -s 1 -c 1 -o gpurun_out/k2l_c$c python bench.py --config $c --rows 4194304 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k2l_c$c.log 2>&1
  echo "ncu c$c rc=$?"
done
