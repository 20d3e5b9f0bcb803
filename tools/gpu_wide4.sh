#!/bin/bash
# Thread-per-row mode for few tested columns: wide parity, seeded timing, wide bench lines.
OUT=gpurun_out/${TAG:-r01n}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_wide.py -q > $OUT/pytest_gpu_wide4.log 2>&1; tail -2 $OUT/pytest_gpu_wide4.log
timeout 600 python tools/wide_seeded_perf.py > $OUT/wide_seeded_perf4.jsonl 2> $OUT/wide_seeded_perf4.err; cat $OUT/wide_seeded_perf4.jsonl
for w in w128-prop w128-stream w256-stream; do
  timeout 600 python bench.py --workload $w --steps 30 --warmup 3 --cpu-budget 8 > $OUT/bench4_$w.json 2> $OUT/bench4_$w.err
done
for f in $OUT/bench4_*.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['value'], d['roofline']['frac'], d['roofline']['launch_ms_median'])"; done
