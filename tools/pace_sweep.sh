mkdir -p gpurun_out
for p in 0 4 8 16 32; do FCT_SKETCH_PACE=$p timeout 300 python tools/bench_sketch.py 4 0 exch 0; done > gpurun_out/pace.jsonl 2>&1
FCT_SKETCH_PACE=8 ncu --clock-control none -k regex:sketch_v5 -c 1 --metrics gpu__time_duration.sum,dram__bytes_read.sum python tools/bench_sketch.py --child 4 0 exch 0 > gpurun_out/ncu_pace8.txt 2>&1
FCT_SKETCH_PACE=0 ncu --clock-control none -k regex:sketch_v5 -c 1 --metrics gpu__time_duration.sum,dram__bytes_read.sum python tools/bench_sketch.py --child 4 0 exch 0 > gpurun_out/ncu_pace0.txt 2>&1
cut -c1-120 gpurun_out/pace.jsonl; grep -E "dram|duration" gpurun_out/ncu_pace8.txt gpurun_out/ncu_pace0.txt
