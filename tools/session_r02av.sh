#!/bin/bash
# r02 session av: share of the row sweep's rows claimed dynamically (RAC_ROW_CLAIM_DIV builds: 1/2, 1/4, 1/8 default, 1/16)
OUT=gpurun_out/r02av
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
python - <<'PY' > $OUT/build_variants.log 2>&1
from paper_2407_11388_b200 import build
for d in (2, 4, 16):
    build.build(out="/tmp/librac_rc%d.so" % d, defines=["RAC_ROW_CLAIM_DIV=%d" % d])
PY
for r in 1 2 3; do
  AB_SET=fused timeout 300 python tools/ab_perf.py rc8 >> $OUT/ab_rc.log 2>&1
  for d in 2 4 16; do RAC_LIB_PATH=/tmp/librac_rc$d.so AB_SET=fused timeout 300 python tools/ab_perf.py rc$d >> $OUT/ab_rc.log 2>&1; done
done
cat $OUT/ab_rc.log
