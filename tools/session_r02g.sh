#!/bin/bash
# r02 session g: is the slower fused sweep of r02f the box or the code?  The
# r02e library (ablibs_e.so) and the current one, back to back on one box.
OUT=gpurun_out/r02g
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu --format=csv > $OUT/gpu.txt
for i in 1 2; do
  RAC_LIB_PATH=$PWD/ablibs_e.so AB_SET=fused timeout 300 python tools/ab_perf.py "[r02e-lib]" >> $OUT/ab_lib.log 2>&1
  AB_SET=fused timeout 300 python tools/ab_perf.py "[current]" >> $OUT/ab_lib.log 2>&1
done
cat $OUT/ab_lib.log
timeout 600 python bench.py --steps 500 --warmup 10 --cpu-budget 4 > $OUT/bench_default.json 2> $OUT/bench_default.err
python -c "import json;d=json.load(open('$OUT/bench_default.json'));print(d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
