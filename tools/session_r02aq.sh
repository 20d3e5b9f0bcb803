#!/bin/bash
# r02 session aq: per-pass timeline of the seeded C3 call (and the others), ncu of c3-seed
OUT=gpurun_out/r02aq
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/timeline.py > $OUT/timeline.txt 2>&1; cat $OUT/timeline.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rac_fused -s 5 -c 1 -o $OUT/prof_c3_seed \
   python bench.py --workload c3-seed --steps 10 --warmup 3 --no-cpu-baseline > $OUT/ncu_c3_seed.log 2>&1
ncu -i $OUT/prof_c3_seed.ncu-rep --page raw --csv > $OUT/prof_c3_seed_raw.csv 2>/dev/null
ls $OUT
