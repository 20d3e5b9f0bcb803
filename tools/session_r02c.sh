#!/bin/bash
# r02 session c: fused-kernel pass tail (listed apply, release-reduction barrier)
# A/B, one-block kernel with the relation staged in smem (C1), zero-copy
# blocking API, wide search; full GPU suite.
OUT=gpurun_out/r02c
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
for v in "" "RAC_FUSED_AB=1" "RAC_FUSED_AB=2" "RAC_FUSED_AB=3"; do
  env $v timeout 300 python tools/ab_perf.py "[$v]" >> $OUT/ab_fused.log 2>&1
done
cat $OUT/ab_fused.log
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/timeline.py > $OUT/timeline.txt 2>&1; cat $OUT/timeline.txt
for w in c1-seed c3-prop c3-stream; do
  timeout 600 python bench.py --workload $w --steps 500 --warmup 10 --cpu-budget 6 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python -c "import json;d=json.load(open('$OUT/bench_$w.json'));print('$w', d['ms_per_step'], d['e2e']['value'], d['roofline'] and d['roofline']['frac'], d['cpu_baseline']['value'], d['cpu_baseline']['cores'])"
done
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
