#!/bin/bash
# r02 session aa: same-box A/B of rac_batch_cl build variants at C5 (table build, staging)
OUT=gpurun_out/r02aa
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
python - <<'PY' > $OUT/build_variants.log 2>&1
from paper_2407_11388_b200 import build
build.build(out="/tmp/librac_item.so", defines=["RAC_CL_ITEM_TABLES=1"])
build.build(out="/tmp/librac_gstage.so", defines=["RAC_CL_GLOBAL_STAGE=1"])
build.build(out="/tmp/librac_both.so", defines=["RAC_CL_ITEM_TABLES=1", "RAC_CL_GLOBAL_STAGE=1"])
PY
tail -2 $OUT/build_variants.log
for r in 1 2 3; do
  AB_SET=batch timeout 300 python tools/ab_perf.py default >> $OUT/ab_variants.log 2>&1
  RAC_LIB_PATH=/tmp/librac_item.so AB_SET=batch timeout 300 python tools/ab_perf.py item >> $OUT/ab_variants.log 2>&1
  RAC_LIB_PATH=/tmp/librac_gstage.so AB_SET=batch timeout 300 python tools/ab_perf.py gstage >> $OUT/ab_variants.log 2>&1
  RAC_LIB_PATH=/tmp/librac_both.so AB_SET=batch timeout 300 python tools/ab_perf.py both >> $OUT/ab_variants.log 2>&1
done
cat $OUT/ab_variants.log
