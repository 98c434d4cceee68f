# ncu --set full (source counters) of K2 at the cfg-5 geometry, 2^22 rows
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python bench.py --config 3 --rows 4194304 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/k2c3_plain.json 2> gpurun_out/k2c3_plain.err || exit 1
ncu --set full --clock-control none --import-source on -k regex:rownorm_ws2 -s 1 -c 1 -o gpurun_out/k2_c3 python bench.py --config 3 --rows 4194304 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k2c3.log 2>&1
echo "ncu rc=$?"
