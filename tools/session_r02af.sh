#!/bin/bash
# r02 session af: column sweep with partitioned tail claims (RAC_COL_CLAIM=2 build variants) vs static round robin, same box
OUT=gpurun_out/r02af
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
python - <<'PY' > $OUT/build_variants.log 2>&1
from paper_2407_11388_b200 import build
build.build(out="/tmp/librac_claim8.so", defines=["RAC_COL_CLAIM=2"])
build.build(out="/tmp/librac_claim16.so", defines=["RAC_COL_CLAIM=2", "RAC_CLAIM_DIV=16"])
build.build(out="/tmp/librac_claim4.so", defines=["RAC_COL_CLAIM=2", "RAC_CLAIM_DIV=4"])
PY
tail -1 $OUT/build_variants.log
for r in 1 2 3; do
  AB_SET=fused timeout 300 python tools/ab_perf.py default >> $OUT/ab_claim.log 2>&1
  RAC_LIB_PATH=/tmp/librac_claim8.so AB_SET=fused timeout 300 python tools/ab_perf.py claim8 >> $OUT/ab_claim.log 2>&1
  RAC_LIB_PATH=/tmp/librac_claim16.so AB_SET=fused timeout 300 python tools/ab_perf.py claim16 >> $OUT/ab_claim.log 2>&1
  RAC_LIB_PATH=/tmp/librac_claim4.so AB_SET=fused timeout 300 python tools/ab_perf.py claim4 >> $OUT/ab_claim.log 2>&1
done
cat $OUT/ab_claim.log
RAC_LIB_PATH=/tmp/librac_claim8.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_certify.py -q -x --timeout 900 > $OUT/pytest_claim8.log 2>&1; tail -2 $OUT/pytest_claim8.log
