mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:sketch_v -c 1 -o gpurun_out/v5_22 python tools/bench_sketch.py --child 4 4194304 exch 0 > gpurun_out/ncu_v5.log 2>&1
FCT_SKETCH_V1=1 ncu --set full --clock-control none --import-source on -k regex:sketch_v -c 1 -o gpurun_out/v1x_22 python tools/bench_sketch.py --child 4 4194304 exch 0 >> gpurun_out/ncu_v5.log 2>&1
echo done
