#!/bin/bash
# r02 session ac: rac_batch_cl column-group layout (8-byte loads per row per group) A/B vs per-column masks
OUT=gpurun_out/r02ac
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "batch" > $OUT/pytest_batch.log 2>&1; tail -2 $OUT/pytest_batch.log
RAC_CL_GROUPS=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "batch" > $OUT/pytest_batch_nogroups.log 2>&1; tail -2 $OUT/pytest_batch_nogroups.log
for r in 1 2 3; do
  AB_SET=batch timeout 300 python tools/ab_perf.py groups >> $OUT/ab_groups.log 2>&1
  RAC_CL_GROUPS=0 AB_SET=batch timeout 300 python tools/ab_perf.py columns >> $OUT/ab_groups.log 2>&1
done
cat $OUT/ab_groups.log
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/batch_cl_timeline.py > $OUT/batch_cl_timeline.txt 2>&1; head -30 $OUT/batch_cl_timeline.txt
