#!/bin/bash
# r02 session ba: batch staging with 8 vs 4 variables in flight per warp (RAC_CL_STAGE_IF builds), same box
OUT=gpurun_out/r02ba
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
python -c "from paper_2407_11388_b200 import build; build.build(out='/tmp/librac_if4.so', defines=['RAC_CL_STAGE_IF=4'])" > $OUT/build.log 2>&1
for r in 1 2 3; do
  AB_SET=batch timeout 300 python tools/ab_perf.py if8 >> $OUT/ab.log 2>&1
  RAC_LIB_PATH=/tmp/librac_if4.so AB_SET=batch timeout 300 python tools/ab_perf.py if4 >> $OUT/ab.log 2>&1
done
cat $OUT/ab.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "batch" > $OUT/pytest_batch.log 2>&1; tail -2 $OUT/pytest_batch.log
timeout 300 python bench.py --workload c5-batch --steps 400 --warmup 10 --cpu-budget 3 > $OUT/bench_c5-batch.json 2> $OUT/bench_c5.err
python -c "import json;d=json.load(open('$OUT/bench_c5-batch.json'));print('c5', d['ms_per_step'], d['value'], d['roofline']['frac'])"
