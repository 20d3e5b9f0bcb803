#!/bin/bash
# r02 session f: chunked dynamic claiming of the column pass tail (pass-1 straggler)
OUT=gpurun_out/r02f
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
for v in "" "RAC_CLAIM_CH=4 RAC_CLAIM_DIV=16" "RAC_CLAIM_CH=8 RAC_CLAIM_DIV=16" "RAC_CLAIM_CH=8 RAC_CLAIM_DIV=8" "RAC_CLAIM_CH=16 RAC_CLAIM_DIV=8" "RAC_CLAIM_CH=4 RAC_CLAIM_DIV=32"; do
  env $v AB_SET=fused timeout 300 python tools/ab_perf.py "[$v]" >> $OUT/ab_claim.log 2>&1
done
cat $OUT/ab_claim.log
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/timeline.py > $OUT/timeline.txt 2>&1; cat $OUT/timeline.txt
for v in "" "RAC_STATE_T=32" "RAC_STATE_T=256"; do
  env $v AB_SET=small timeout 300 python tools/ab_perf.py "[$v]" >> $OUT/ab_small.log 2>&1
done
cat $OUT/ab_small.log
