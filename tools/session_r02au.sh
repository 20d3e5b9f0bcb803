#!/bin/bash
# r02 session au: row-sweep dynamic tail claims (one counter) vs static round robin (RAC_NO_CLAIM)
OUT=gpurun_out/r02au
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
for r in 1 2 3; do
  AB_SET=fused timeout 300 python tools/ab_perf.py claim >> $OUT/ab_claim.log 2>&1
  RAC_NO_CLAIM=1 AB_SET=fused timeout 300 python tools/ab_perf.py static >> $OUT/ab_claim.log 2>&1
done
cat $OUT/ab_claim.log
RAC_NO_CLAIM=1 RAC_DEBUG_TIMELINE=1 timeout 300 python tools/timeline.py > $OUT/timeline_static.txt 2>&1; grep "c3-seed\|c3-prop" $OUT/timeline_static.txt
