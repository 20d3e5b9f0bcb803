#!/bin/bash
# r02 session ab: same-box A/B of rac_batch_cl table-store rotation (item tables, no local memory) + batch tests
OUT=gpurun_out/r02ab
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
python - <<'PY' > $OUT/build_variants.log 2>&1
from paper_2407_11388_b200 import build
build.build(out="/tmp/librac_rot.so", defines=["RAC_CL_ITEM_ROT=1"])
build.build(out="/tmp/librac_wcol.so", defines=["RAC_CL_ITEM_TABLES=0"])
PY
for r in 1 2 3; do
  AB_SET=batch timeout 300 python tools/ab_perf.py default >> $OUT/ab_variants.log 2>&1
  RAC_LIB_PATH=/tmp/librac_rot.so AB_SET=batch timeout 300 python tools/ab_perf.py rot >> $OUT/ab_variants.log 2>&1
  RAC_LIB_PATH=/tmp/librac_wcol.so AB_SET=batch timeout 300 python tools/ab_perf.py warpcol >> $OUT/ab_variants.log 2>&1
done
cat $OUT/ab_variants.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "batch" > $OUT/pytest_batch.log 2>&1; tail -2 $OUT/pytest_batch.log
RAC_LIB_PATH=/tmp/librac_rot.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "batch" > $OUT/pytest_batch_rot.log 2>&1; tail -2 $OUT/pytest_batch_rot.log
