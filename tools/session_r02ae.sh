#!/bin/bash
# r02 session ae: fused-kernel team mode (small late passes on K CTAs, the rest parked): parity + A/B; small-grid barrier probe
OUT=gpurun_out/r02ae
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 120 ./tools/probes/grid_barrier > $OUT/grid_barrier.jsonl 2>&1; grep -E '"grid": (8|16|32|64),' $OUT/grid_barrier.jsonl | grep one_counter
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -k "team" > $OUT/pytest_team.log 2>&1; tail -3 $OUT/pytest_team.log
for r in 1 2; do
  for k in 0 8 16 32; do RAC_TEAM_K=$k AB_SET=fused timeout 300 python tools/ab_perf.py k$k >> $OUT/ab_team.log 2>&1; done
  for k in 0 16; do RAC_TEAM_K=$k AB_SET=sparse timeout 300 python tools/ab_perf.py k$k >> $OUT/ab_team.log 2>&1; done
done
cat $OUT/ab_team.log
for k in 0 16; do RAC_TEAM_K=$k RAC_DEBUG_TIMELINE=1 timeout 300 python tools/timeline.py > $OUT/timeline_k$k.txt 2>&1; grep "c3-prop\|c3s-prop" $OUT/timeline_k$k.txt; done
