#!/bin/bash
# r02 session h: fused regression check vs the r02e library, rac_tiny (C1 one
# warp), rac_batch_cl inner-loop rework; the tests those touch.
OUT=gpurun_out/r02h
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
for i in 1 2; do
  RAC_LIB_PATH=$PWD/ablibs_e.so AB_SET=fused timeout 300 python tools/ab_perf.py "[r02e-lib]" >> $OUT/ab_lib.log 2>&1
  AB_SET=fused timeout 300 python tools/ab_perf.py "[current]" >> $OUT/ab_lib.log 2>&1
done
cat $OUT/ab_lib.log
for v in "" "RAC_NO_TINY=1"; do env $v AB_SET=small timeout 300 python tools/ab_perf.py "[$v]" >> $OUT/ab_small.log 2>&1; done
for v in "" "RAC_BATCH_CL=8" "RAC_BATCH_CL=2"; do env $v AB_SET=batch timeout 300 python tools/ab_perf.py "[$v]" >> $OUT/ab_batch.log 2>&1; done
cat $OUT/ab_small.log $OUT/ab_batch.log
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/timeline.py > $OUT/timeline.txt 2>&1; head -3 $OUT/timeline.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -k "spec_corpus or c5 or batched or golden or c1 or nonuniform" tests/test_gpu_certify.py -k "batched or seeded" -q > $OUT/pytest_sel.log 2>&1; tail -3 $OUT/pytest_sel.log
for w in c1-seed c5-batch; do
  timeout 600 python bench.py --workload $w --steps 500 --warmup 10 --cpu-budget 4 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python -c "import json;d=json.load(open('$OUT/bench_$w.json'));r=d['roofline'] or {};print('$w', 'ms', round(d['ms_per_step'],5), 'val', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'frac', r.get('frac'), r.get('kernel'))"
done
