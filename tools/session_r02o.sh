#!/bin/bash
# r02 session o: wide tensor-core batch (f16 / fp8), pass A/B with fp8, wide tests
OUT=gpurun_out/r02o
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 1200 python -m pytest tests/test_gpu_wide.py -q -x --timeout 600 -k "batched or pass_eval" > $OUT/pytest_wide.log 2>&1; tail -3 $OUT/pytest_wide.log
timeout 900 python tools/wide_tc_ab.py > $OUT/wide_tc_ab.jsonl 2>&1; cat $OUT/wide_tc_ab.jsonl
RAC_WIDE_TC=fp8 timeout 900 python tools/wide_tc_ab.py > $OUT/wide_tc_ab_fp8.jsonl 2>&1; tail -1 $OUT/wide_tc_ab_fp8.jsonl
for v in "" "RAC_WIDE_TC=fp8" "RAC_WIDE_BATCH=state"; do
  env $v timeout 900 python bench.py --workload w128-batch --steps 10 --warmup 3 --cpu-budget 10 > $OUT/bench_w128-batch$(echo $v | tr '=' '_').json 2> $OUT/bench_w128-batch.err
  python -c "import json,glob;f=sorted(glob.glob('$OUT/bench_w128-batch*.json'),key=lambda p: __import__('os').path.getmtime(p))[-1];d=json.load(open(f));print('[$v]', d['ms_per_step'], d['value'], d['roofline'] and d['roofline'].get('frac'), d['roofline'] and d['roofline'].get('achieved'), d['enforcement'], d['cpu_baseline']['value'])"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wide_tc_pass -c 2 -o $OUT/prof_wide_tc \
   python tools/wide_tc_ab.py > $OUT/ncu_wide_tc.log 2>&1
ncu -i $OUT/prof_wide_tc.ncu-rep --page raw --csv > $OUT/prof_wide_tc_raw.csv 2>/dev/null
