#!/bin/bash
# r02 session i: bulk-copy staging of the mask tensor in the one-warp / one-block kernels (C1)
OUT=gpurun_out/r02i
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -k "spec_corpus or golden or c1 or nonuniform or seeded or async" tests/test_gpu_certify.py -k "seeded or batched" -q > $OUT/pytest_sel.log 2>&1; tail -3 $OUT/pytest_sel.log
for w in c1-seed c5-batch; do
  timeout 600 python bench.py --workload $w --steps 500 --warmup 10 --cpu-budget 4 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python -c "import json;d=json.load(open('$OUT/bench_$w.json'));r=d['roofline'] or {};print('$w', 'ms', round(d['ms_per_step'],5), 'val', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'frac', r.get('frac'), r.get('kernel'))"
done
timeout 300 python tools/e2e_probe.py > $OUT/e2e_probe.jsonl 2>&1; cat $OUT/e2e_probe.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rac_batch_cl -s 3 -c 1 -o $OUT/prof_c5_batch_cl \
   python bench.py --workload c5-batch --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ncu_c5.log 2>&1
ncu -i $OUT/prof_c5_batch_cl.ncu-rep --page raw --csv > $OUT/prof_c5_batch_cl_raw.csv 2>/dev/null
ncu -i $OUT/prof_c5_batch_cl.ncu-rep --page source --csv --print-source sass > $OUT/prof_c5_batch_cl_sass.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:rac_tiny -s 3 -c 1 -o $OUT/prof_c1_tiny \
   python bench.py --workload c1-seed --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ncu_c1.log 2>&1
ncu -i $OUT/prof_c1_tiny.ncu-rep --page raw --csv > $OUT/prof_c1_tiny_raw.csv 2>/dev/null
