#!/bin/bash
# r02 session e: batched cluster kernel (session d's content), wide tcgen05 A/B,
# graph-captured bench, e2e probe, GPU suite (wide search budget fix).
OUT=gpurun_out/r02e
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 300 python tools/e2e_probe.py > $OUT/e2e_probe.jsonl 2>&1; cat $OUT/e2e_probe.jsonl
for v in "" "RAC_BATCH_CL=1" "RAC_BATCH_CL=2" "RAC_BATCH_CL=8" "RAC_BATCH_IMPL=bs"; do
  env $v AB_SET=batch timeout 300 python tools/ab_perf.py "[$v]" >> $OUT/ab_batch.log 2>&1
done
cat $OUT/ab_batch.log
timeout 600 python tools/wide_tc_ab.py > $OUT/wide_tc_ab.jsonl 2>&1; cat $OUT/wide_tc_ab.jsonl
for w in c1-seed c2-root c3-stream c3-prop c5-batch; do
  timeout 600 python bench.py --workload $w --steps 500 --warmup 10 --cpu-budget 6 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python -c "import json;d=json.load(open('$OUT/bench_$w.json'));r=d['roofline'] or {};print('$w', 'ms', round(d['ms_per_step'],5), 'val', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'frac', r.get('frac'), r.get('kernel'), d['setup']['launch'][:40], 'cpu', round(d['cpu_baseline']['value'],2), d['cpu_baseline']['cores'], d.get('roofline_l2',{}).get('frac') if d.get('roofline_l2') else None)"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wide_tc_pass -c 1 -o $OUT/prof_wide_tc \
   python tools/wide_tc_ab.py > $OUT/ncu_wide_tc.log 2>&1
ncu -i $OUT/prof_wide_tc.ncu-rep --page raw --csv > $OUT/prof_wide_tc_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wide_bs_pass -c 1 -o $OUT/prof_wide_bs \
   python tools/wide_tc_ab.py > $OUT/ncu_wide_bs.log 2>&1
ncu -i $OUT/prof_wide_bs.ncu-rep --page raw --csv > $OUT/prof_wide_bs_raw.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rac_batch_cl -s 3 -c 1 -o $OUT/prof_c5_batch_cl \
   python bench.py --workload c5-batch --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ncu_c5.log 2>&1
ncu -i $OUT/prof_c5_batch_cl.ncu-rep --page raw --csv > $OUT/prof_c5_batch_cl_raw.csv 2>/dev/null
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/pytest_gpu.log 2>&1; tail -15 $OUT/pytest_gpu.log
