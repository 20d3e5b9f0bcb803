#!/bin/bash
# r02 session bb: final committed state (after the staging tweak) -- smoke, full GPU suite, default bench, C5 bench
OUT=gpurun_out/r02bb
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
python -c "import json;d=json.load(open('$OUT/bench_default.json'));print('default', d['ms_per_step'], d['value'], d['roofline']['frac'], d['setup'].get('full_pass_sweep',{}).get('sweep'), d['e2e']['value'], d['clocks'])"
timeout 300 python bench.py --workload c5-batch --steps 400 --warmup 10 --cpu-budget 3 > $OUT/bench_c5-batch.json 2> $OUT/bench_c5.err
python -c "import json;d=json.load(open('$OUT/bench_c5-batch.json'));print('c5', d['ms_per_step'], d['value'], d['roofline']['frac'])"
