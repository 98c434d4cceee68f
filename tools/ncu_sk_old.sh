mkdir -p gpurun_out
export FCT_LIB=$PWD/tools/libfct_r1.so
python tools/bench_sketch.py 4 4194304 cas 0 > gpurun_out/sk22old.jsonl 2>&1
ncu --set full --clock-control none --import-source on -k regex:sketch_v1 -c 1 -o gpurun_out/sk22old python tools/bench_sketch.py --child 4 4194304 cas 0 > gpurun_out/ncu_sk22old.log 2>&1
echo "ncu rc=$?"
cat gpurun_out/sk22old.jsonl
