mkdir -p gpurun_out
out=gpurun_out/ngrp_sweep.jsonl; : > $out
for g in 0 35 41 47 53 59; do echo "ngrp=$g cfg5 2^25" >> $out; if [ $g = 0 ]; then unset FCT_SKETCH_NGRP; else export FCT_SKETCH_NGRP=$g; fi; timeout 120 python tools/bench_sketch.py 5 33554432 exch 0 >> $out 2>&1; done
for g in 0 35 41 47 53 59 65; do echo "ngrp=$g cfg5 2^28" >> $out; if [ $g = 0 ]; then unset FCT_SKETCH_NGRP; else export FCT_SKETCH_NGRP=$g; fi; timeout 200 python tools/bench_sketch.py 5 268435456 exch 0 >> $out 2>&1; done
for g in 0 37 55 74; do echo "ngrp=$g cfg4" >> $out; if [ $g = 0 ]; then unset FCT_SKETCH_NGRP; else export FCT_SKETCH_NGRP=$g; fi; timeout 120 python tools/bench_sketch.py 4 0 exch 0 >> $out 2>&1; done
cut -c1-140 $out
