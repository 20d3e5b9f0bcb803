#!/bin/bash
# r02 session aw: row-sweep removals aggregated per CTA in shared memory (RAC_NO_ROW_AGG A/B), full GPU suite
OUT=gpurun_out/r02aw
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
for r in 1 2 3; do
  AB_SET=fused timeout 300 python tools/ab_perf.py agg >> $OUT/ab_agg.log 2>&1
  RAC_NO_ROW_AGG=1 AB_SET=fused timeout 300 python tools/ab_perf.py noagg >> $OUT/ab_agg.log 2>&1
done
cat $OUT/ab_agg.log
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/timeline.py > $OUT/timeline.txt 2>&1; grep "c3-seed\|c3-prop" $OUT/timeline.txt
timeout 2000 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
RAC_FORCE_LAYOUT=rows timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "corpus or c3 or forced" > $OUT/pytest_rows.log 2>&1; tail -2 $OUT/pytest_rows.log
