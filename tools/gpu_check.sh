#!/bin/bash
# GPU session: build, smoke, GPU parity tests, and bench lines for the given workloads.
OUT=gpurun_out/${TAG:-chk}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
for w in ${WORKLOADS:-c3-stream}; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-500} --warmup 10 --cpu-budget ${CPU_BUDGET:-5} > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python - $OUT/bench_$w.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r=d.get('roofline') or {}
    print(sys.argv[1].split('/')[-1], 'value=%.1f %s ms=%.4f frac=%s ach=%s e2e=%.1f cpu=%s iters=%s clk=%s' % (d['value'], d['unit'], d['ms_per_step'], r.get('frac'), r.get('achieved'), (d.get('e2e') or {}).get('value') or 0, (d.get('cpu_baseline') or {}).get('value'), d.get('enforcement'), d.get('clocks',{}).get('sm_mhz')))
except Exception as e:
    print('bench parse failed', sys.argv[1], e)
PY
done
