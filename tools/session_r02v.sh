#!/bin/bash
# r02 session v: per-pass change lists on small dense passes (RAC_LIST_MAX A/B), C5 staging by coalesced loads, fences reverted
OUT=gpurun_out/r02v
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
for r in 1 2; do
  for lm in 0 16 64 256; do RAC_LIST_MAX=$lm AB_SET=fused timeout 300 python tools/ab_perf.py lm$lm >> $OUT/ab_list.log 2>&1; done
done
cat $OUT/ab_list.log
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/timeline.py > $OUT/timeline.txt 2>&1; grep -A2 "c3-prop\|c3-seed" $OUT/timeline.txt | head -12
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_certify.py -q -x --timeout 900 > $OUT/pytest_parity.log 2>&1; tail -3 $OUT/pytest_parity.log
for w in c5-batch c1-seed c3-prop c3-seed; do
  timeout 300 python bench.py --workload $w --steps 400 --warmup 10 --cpu-budget 3 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python -c "import json;d=json.load(open('$OUT/bench_$w.json'));print('$w', d['ms_per_step'], d['value'], d['roofline'] and d['roofline'].get('frac'), d['e2e']['value'])"
done
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/batch_cl_timeline.py > $OUT/batch_cl_timeline.txt 2>&1; head -12 $OUT/batch_cl_timeline.txt
timeout 600 python tools/e2e_probe.py > $OUT/e2e_probe.jsonl 2>&1; cat $OUT/e2e_probe.jsonl
