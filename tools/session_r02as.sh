#!/bin/bash
# r02 session as: warp-aggregated removal atomics + one removal-flag atomic per warp (vs the previous revision, ab_src/old)
OUT=gpurun_out/r02as
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
python -c "from paper_2407_11388_b200 import build; build.build(out='/tmp/librac_old.so', src_dir='ab_src/old')" > $OUT/build_old.log 2>&1; tail -1 $OUT/build_old.log
for r in 1 2 3; do
  AB_SET=fused timeout 300 python tools/ab_perf.py new >> $OUT/ab_agg.log 2>&1
  RAC_LIB_PATH=/tmp/librac_old.so AB_SET=fused timeout 300 python tools/ab_perf.py old >> $OUT/ab_agg.log 2>&1
done
for r in 1 2; do
  AB_SET=sparse timeout 300 python tools/ab_perf.py new >> $OUT/ab_agg.log 2>&1
  RAC_LIB_PATH=/tmp/librac_old.so AB_SET=sparse timeout 300 python tools/ab_perf.py old >> $OUT/ab_agg.log 2>&1
done
cat $OUT/ab_agg.log
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/timeline.py > $OUT/timeline.txt 2>&1; grep "c3-seed\|c3-prop" $OUT/timeline.txt
timeout 300 python tools/cta_stamps.py --seed > $OUT/cta_seed.txt 2>&1; cat $OUT/cta_seed.txt
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
