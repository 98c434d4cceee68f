mkdir -p gpurun_out
python bench.py --config 4 --rows 4194304 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/k2_plain.json 2> gpurun_out/k2_plain.err
ncu --set full --clock-control none --import-source on -k regex:rownorm_ws2 -s 1 -c 1 -o gpurun_out/k2_22 python bench.py --config 4 --rows 4194304 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k2.log 2>&1
echo "ncu rc=$?"
