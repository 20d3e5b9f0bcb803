#!/bin/bash
# r02 session w: C5 kernel (quad table build, list-only, no full-row code), fused list mode t>1, box reference numbers
OUT=gpurun_out/r02w
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,clocks.max.mem,power.limit --format=csv > $OUT/gpu.txt; cat $OUT/gpu.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "batch" > $OUT/pytest_batch.log 2>&1; tail -3 $OUT/pytest_batch.log
for lm in 0 16; do RAC_LIST_MAX=$lm AB_SET=fused timeout 300 python tools/ab_perf.py lm$lm >> $OUT/ab_list.log 2>&1; done; cat $OUT/ab_list.log
timeout 300 python bench.py --workload c5-batch --steps 400 --warmup 10 --cpu-budget 3 > $OUT/bench_c5-batch.json 2> $OUT/bench_c5-batch.err
python -c "import json;d=json.load(open('$OUT/bench_c5-batch.json'));print('c5', d['ms_per_step'], d['value'], d['roofline'] and d['roofline'].get('frac'), d['e2e']['value'], d['clocks'])"
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/batch_cl_timeline.py > $OUT/batch_cl_timeline.txt 2>&1; head -30 $OUT/batch_cl_timeline.txt
