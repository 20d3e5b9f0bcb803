#!/bin/bash
# r02 session y: ncu source-level profile of rac_batch_cl (current), to locate prep/stage time
OUT=gpurun_out/r02y
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rac_batch_cl -s 3 -c 1 -o $OUT/prof_c5 \
   python bench.py --workload c5-batch --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ncu_c5.log 2>&1
ncu -i $OUT/prof_c5.ncu-rep --page raw --csv > $OUT/prof_c5_raw.csv 2>/dev/null
ncu -i $OUT/prof_c5.ncu-rep --page source --csv > $OUT/prof_c5_source.csv 2>/dev/null
ls -la $OUT
