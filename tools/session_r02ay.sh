#!/bin/bash
# r02 session ay: cluster batch kernel without the per-pass change-mask copy + block barrier (vs HEAD~, ab_src/old)
OUT=gpurun_out/r02ay
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
python -c "from paper_2407_11388_b200 import build; build.build(out='/tmp/librac_old.so', src_dir='ab_src/old')" > $OUT/build_old.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -k "batch" > $OUT/pytest_batch.log 2>&1; tail -2 $OUT/pytest_batch.log
for r in 1 2 3; do
  AB_SET=batch timeout 300 python tools/ab_perf.py new >> $OUT/ab.log 2>&1
  RAC_LIB_PATH=/tmp/librac_old.so AB_SET=batch timeout 300 python tools/ab_perf.py old >> $OUT/ab.log 2>&1
done
cat $OUT/ab.log
timeout 300 python bench.py --workload c5-batch --steps 400 --warmup 10 --cpu-budget 3 > $OUT/bench_c5-batch.json 2> $OUT/bench_c5.err
python -c "import json;d=json.load(open('$OUT/bench_c5-batch.json'));print('c5', d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'])"
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/batch_cl_timeline.py > $OUT/batch_cl_timeline.txt 2>&1; head -26 $OUT/batch_cl_timeline.txt
