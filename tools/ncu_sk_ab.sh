mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,launch__grid_size,launch__block_size,launch__shared_mem_per_block_dynamic,smsp__inst_executed_op_shared_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,dram__bytes_read.sum,smsp__inst_executed_op_branch.sum
FCT_LIB=$PWD/tools/libfct_r1.so ncu --clock-control none -k regex:sketch_v1 -c 1 --metrics $M python tools/bench_sketch.py --child 4 4194304 cas 0 > gpurun_out/ncu_ab_old.txt 2>&1
ncu --clock-control none -k regex:sketch_v1 -c 1 --metrics $M python tools/bench_sketch.py --child 4 4194304 cas 0 > gpurun_out/ncu_ab_new.txt 2>&1
grep -E "sketch_v1|duration|inst_exec|grid|block_size|shared_mem|atom|wavefr|dram|branch|lib" gpurun_out/ncu_ab_old.txt gpurun_out/ncu_ab_new.txt
