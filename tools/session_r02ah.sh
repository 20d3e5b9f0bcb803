#!/bin/bash
# r02 session ah: faster Python marshalling of the blocking calls (e2e), parity of the blocking paths
OUT=gpurun_out/r02ah
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 600 python tools/e2e_probe.py > $OUT/e2e_probe.jsonl 2>&1; cat $OUT/e2e_probe.jsonl
for w in c1-seed c3-stream c2-root; do
  timeout 300 python bench.py --workload $w --steps 2000 --warmup 10 --cpu-budget 3 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python -c "import json;d=json.load(open('$OUT/bench_$w.json'));print('$w', d['ms_per_step'], d['value'], d['roofline'] and d['roofline'].get('frac'), 'e2e', d['e2e']['value'], 1e6/d['e2e']['value'], 'us')"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py -q -x --timeout 900 > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
