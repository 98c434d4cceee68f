# one ncu --set full capture of the sketch kernel at 2^22 rows (cfg-4 shape), plus a timing run first
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,pci.bus_id,clocks.sm,clocks.max.sm,power.draw,temperature.gpu,ecc.mode.current,compute_mode --format=csv > gpurun_out/smi.txt 2>&1
python tools/bench_sketch.py 4 4194304 cas 0 > gpurun_out/sk22.jsonl 2>&1
ncu --set full --clock-control none --import-source on -k regex:sketch_v1 -c 1 -o gpurun_out/sk22 python tools/bench_sketch.py --child 4 4194304 cas 0 > gpurun_out/ncu_sk22.log 2>&1
echo "ncu rc=$?"
cat gpurun_out/smi.txt gpurun_out/sk22.jsonl
