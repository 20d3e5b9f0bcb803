#!/bin/bash
# r02 session al: per-state sweep for words with <= 8 active states (RAC_CL_PS A/B), batch tests in every sweep mode
OUT=gpurun_out/r02al
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -k "batch" > $OUT/pytest_batch.log 2>&1; tail -3 $OUT/pytest_batch.log
for r in 1 2 3; do
  RAC_CL_PS=0 AB_SET=batch timeout 300 python tools/ab_perf.py ps0 >> $OUT/ab_ps.log 2>&1
  RAC_CL_PS=1 AB_SET=batch timeout 300 python tools/ab_perf.py ps1 >> $OUT/ab_ps.log 2>&1
  RAC_CL_PS=2 AB_SET=batch timeout 300 python tools/ab_perf.py ps2 >> $OUT/ab_ps.log 2>&1
done
cat $OUT/ab_ps.log
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/batch_cl_timeline.py > $OUT/batch_cl_timeline.txt 2>&1; head -30 $OUT/batch_cl_timeline.txt
