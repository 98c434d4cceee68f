# ncu --set full of the fused probabilities + sampling kernel (cfg 4)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:probs_sample -s 1 -c 1 -o gpurun_out/samp_c4 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_samp.log 2>&1
echo "ncu rc=$?"
