# full-size evidence for the round (GPU box): default bench line (cfg 4, N = 1) and cfg 3 / cfg-5 shard lines,
# the ncu launch list of the default command, one ncu --set full capture of each of the two dominant kernels
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
python bench.py --config 3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg3.json 2>/dev/null; echo "cfg3 rc=$?"
python bench.py --config 5 --rows 33554432 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg5.json 2>/dev/null; echo "cfg5 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k "regex:sketch_v5|rownorm_ws2" -s 2 -c 2 -o gpurun_out/full_cfg4 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
