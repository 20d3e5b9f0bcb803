#!/bin/bash
# r02 session ai: does the row-major copy pay for itself?  RAC_NO_ROW_LAYOUT=1 (column-major only, half the memory) vs default
OUT=gpurun_out/r02ai
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
for r in 1 2; do
  AB_SET=fused timeout 300 python tools/ab_perf.py rows_on >> $OUT/ab_rows.log 2>&1
  RAC_NO_ROW_LAYOUT=1 AB_SET=fused timeout 300 python tools/ab_perf.py rows_off >> $OUT/ab_rows.log 2>&1
done
cat $OUT/ab_rows.log
