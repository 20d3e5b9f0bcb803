#!/bin/bash
# r02 session ap: create-time calibration of the full-pass sweep (rows vs columns) -- bench lines, parity
OUT=gpurun_out/r02ap
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
for r in 1 2; do
  AB_SET=fused timeout 300 python tools/ab_perf.py calib >> $OUT/ab_calib.log 2>&1
  RAC_NO_TIE_CALIB=1 AB_SET=fused timeout 300 python tools/ab_perf.py rows >> $OUT/ab_calib.log 2>&1
  RAC_FORCE_LAYOUT=tiecols AB_SET=fused timeout 300 python tools/ab_perf.py cols >> $OUT/ab_calib.log 2>&1
done
cat $OUT/ab_calib.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
python -c "import json;d=json.load(open('$OUT/bench_default.json'));print('default', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline'].get('box_copy_gbs'), d['setup'].get('full_pass_sweep'), d['e2e']['value'])"
for w in c3-prop c4-stream; do
  timeout 600 python bench.py --workload $w --steps 200 --warmup 5 --cpu-budget 3 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python -c "import json;d=json.load(open('$OUT/bench_$w.json'));print('$w', d['ms_per_step'], d['value'], d['roofline'] and d['roofline'].get('frac'), d['setup'].get('full_pass_sweep'))"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_certify.py -q -x --timeout 900 > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
