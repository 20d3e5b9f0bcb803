#!/bin/bash
# r02 session q (after the container re-creation): full GPU suite, bench lines, session p's timeline / A/B
OUT=gpurun_out/r02q
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; cat $OUT/bench_default.json
for w in c3-prop c5-batch c1-seed w128-batch; do
  timeout 600 python bench.py --workload $w --steps 200 --warmup 10 --cpu-budget 5 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python -c "import json;d=json.load(open('$OUT/bench_$w.json'));print('$w', d['ms_per_step'], d['value'], d['unit'], d['roofline'] and d['roofline'].get('frac'), d.get('e2e',{}).get('value'))"
done
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/batch_cl_timeline.py > $OUT/batch_cl_timeline.txt 2>&1; cp gpurun_out/batch_cl_timeline.json $OUT/ 2>/dev/null; head -40 $OUT/batch_cl_timeline.txt
for ab in 0 4; do RAC_FUSED_AB=$ab AB_SET=fused timeout 300 python tools/ab_perf.py ab$ab >> $OUT/ab_fused.log 2>&1; done
cat $OUT/ab_fused.log
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/timeline.py > $OUT/timeline.txt 2>&1; grep -A3 c3-prop $OUT/timeline.txt | head -30
