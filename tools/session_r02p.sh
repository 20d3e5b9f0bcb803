#!/bin/bash
# r02 session p: cluster-batch per-word timeline (C5), fused pass tail A/B (removal-flag read)
OUT=gpurun_out/r02p
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/batch_cl_timeline.py > $OUT/batch_cl_timeline.txt 2>&1; cp gpurun_out/batch_cl_timeline.json $OUT/ 2>/dev/null; head -60 $OUT/batch_cl_timeline.txt
for r in 1 2; do
  for ab in 0 4; do RAC_FUSED_AB=$ab AB_SET=fused timeout 300 python tools/ab_perf.py ab$ab >> $OUT/ab_fused.log 2>&1; done
done
cat $OUT/ab_fused.log
for ab in 0 4; do RAC_FUSED_AB=$ab RAC_DEBUG_TIMELINE=1 timeout 300 python tools/timeline.py > $OUT/timeline_ab$ab.txt 2>&1; grep c3-prop $OUT/timeline_ab$ab.txt; done
