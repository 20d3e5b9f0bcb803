#!/bin/bash
# r02 session ag: partitioned tail claims, own partition only (RAC_COL_CLAIM=2 builds) vs static round robin, same box
OUT=gpurun_out/r02ag
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
python - <<'PY' > $OUT/build_variants.log 2>&1
from paper_2407_11388_b200 import build
build.build(out="/tmp/librac_claim8.so", defines=["RAC_COL_CLAIM=2"])
build.build(out="/tmp/librac_claim16.so", defines=["RAC_COL_CLAIM=2", "RAC_CLAIM_DIV=16"])
PY
for r in 1 2 3; do
  AB_SET=fused timeout 300 python tools/ab_perf.py default >> $OUT/ab_claim.log 2>&1
  RAC_LIB_PATH=/tmp/librac_claim8.so AB_SET=fused timeout 300 python tools/ab_perf.py claim8 >> $OUT/ab_claim.log 2>&1
  RAC_LIB_PATH=/tmp/librac_claim16.so AB_SET=fused timeout 300 python tools/ab_perf.py claim16 >> $OUT/ab_claim.log 2>&1
done
cat $OUT/ab_claim.log
RAC_LIB_PATH=/tmp/librac_claim8.so RAC_DEBUG_TIMELINE=1 timeout 300 python tools/timeline.py > $OUT/timeline_claim8.txt 2>&1; grep "c3-stream\|c3-prop" $OUT/timeline_claim8.txt
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/timeline.py > $OUT/timeline_default.txt 2>&1; grep "c3-stream\|c3-prop" $OUT/timeline_default.txt
