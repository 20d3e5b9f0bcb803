#!/bin/bash
# Seeded wide timing; bench lines under the kept/removed roofline byte rule.
OUT=gpurun_out/${TAG:-r01n}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build3.log 2>&1
timeout 600 python tools/wide_seeded_perf.py > $OUT/wide_seeded_perf.jsonl 2> $OUT/wide_seeded_perf.err; cat $OUT/wide_seeded_perf.jsonl
timeout 600 python bench.py > $OUT/bench2_default.json 2> $OUT/bench2_default.err
for w in w128-prop w128-stream c3-prop c3s-prop; do
  timeout 600 python bench.py --workload $w --steps 30 --warmup 3 --cpu-budget 8 > $OUT/bench2_$w.json 2> $OUT/bench2_$w.err
done
for f in $OUT/bench2_*.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['value'], d.get('roofline'))"; done
