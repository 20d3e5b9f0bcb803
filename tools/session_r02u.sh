#!/bin/bash
# r02 session u: blocking calls poll the mapped status word; grid-barrier probe; C5 list-mode default
OUT=gpurun_out/r02u
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 120 ./tools/probes/grid_barrier > $OUT/grid_barrier.jsonl 2>&1; cat $OUT/grid_barrier.jsonl
timeout 600 python tools/e2e_probe.py > $OUT/e2e_probe.jsonl 2>&1; cat $OUT/e2e_probe.jsonl
RAC_NO_STATUS_POLL=1 timeout 600 python tools/e2e_probe.py > $OUT/e2e_probe_nopoll.jsonl 2>&1; cat $OUT/e2e_probe_nopoll.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_certify.py -q -x --timeout 900 > $OUT/pytest_parity.log 2>&1; tail -3 $OUT/pytest_parity.log
for w in c5-batch c1-seed c3-stream; do
  timeout 300 python bench.py --workload $w --steps 400 --warmup 10 --cpu-budget 3 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python -c "import json;d=json.load(open('$OUT/bench_$w.json'));print('$w', d['ms_per_step'], d['value'], d['roofline'] and d['roofline'].get('frac'), d['e2e'])"
done
