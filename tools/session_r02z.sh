#!/bin/bash
# r02 session x: C5 warp-per-column tables, staging without per-variable global loads; (z) pipelined list sweep, 800-thread CTAs
OUT=gpurun_out/r02z
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "batch" > $OUT/pytest_batch.log 2>&1; tail -3 $OUT/pytest_batch.log
timeout 300 python bench.py --workload c5-batch --steps 400 --warmup 10 --cpu-budget 3 > $OUT/bench_c5-batch.json 2> $OUT/bench_c5-batch.err
python -c "import json;d=json.load(open('$OUT/bench_c5-batch.json'));print('c5', d['ms_per_step'], d['value'], d['roofline'] and d['roofline'].get('frac'), d['e2e']['value'], d['clocks'])"
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/batch_cl_timeline.py > $OUT/batch_cl_timeline.txt 2>&1; head -30 $OUT/batch_cl_timeline.txt
