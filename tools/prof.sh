#!/bin/bash
# usage (on the GPU box): tools/prof.sh <out-name> <kernel-regex> [bench.py args...]
# plain run of bench.py (must exit 0), then one ncu --set full capture of the first matching launch.
name=$1; kre=$2; shift 2
CMD="python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 3 $*"
mkdir -p gpurun_out
$CMD > gpurun_out/${name}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 0 -c 1 -o gpurun_out/$name $CMD > gpurun_out/${name}_ncu.log 2>&1
echo "ncu rc=$?"
