#!/bin/bash
# r02 session am: cluster batch list sweep with u32 column indices and 8 / 16 masks in flight (RAC_CL_NB builds) vs default
OUT=gpurun_out/r02am
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
python - <<'PY' > $OUT/build_variants.log 2>&1
from paper_2407_11388_b200 import build
build.build(out="/tmp/librac_nb8.so", defines=["RAC_CL_NB=8"])
build.build(out="/tmp/librac_nb16.so", defines=["RAC_CL_NB=16"])
PY
for r in 1 2 3; do
  AB_SET=batch timeout 300 python tools/ab_perf.py default >> $OUT/ab_nb.log 2>&1
  RAC_LIB_PATH=/tmp/librac_nb8.so AB_SET=batch timeout 300 python tools/ab_perf.py nb8 >> $OUT/ab_nb.log 2>&1
  RAC_LIB_PATH=/tmp/librac_nb16.so AB_SET=batch timeout 300 python tools/ab_perf.py nb16 >> $OUT/ab_nb.log 2>&1
done
cat $OUT/ab_nb.log
RAC_LIB_PATH=/tmp/librac_nb16.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "batch" > $OUT/pytest_nb16.log 2>&1; tail -2 $OUT/pytest_nb16.log
