#!/bin/bash
# r02 session k: native 32-bit shared atomics in the one-warp / one-block / wide
# per-state kernels (the 64-bit ones were CAS spin loops); 32-bit table
# addressing in rac_batch_cl.
OUT=gpurun_out/r02k
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 300 python tools/c1_probe.py > $OUT/c1_probe.jsonl 2>&1; cat $OUT/c1_probe.jsonl
for v in "" "RAC_BATCH_IMPL=state"; do env $v AB_SET=batch timeout 300 python tools/ab_perf.py "[$v]" >> $OUT/ab_batch.log 2>&1; done
cat $OUT/ab_batch.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -k "spec_corpus or golden or c1 or nonuniform or seeded or async or c5 or batched" tests/test_gpu_certify.py -k "seeded or batched" tests/test_gpu_wide.py -k "batched or corpus or seeded" -q > $OUT/pytest_sel.log 2>&1; tail -3 $OUT/pytest_sel.log
for w in c1-seed c5-batch; do
  timeout 600 python bench.py --workload $w --steps 500 --warmup 10 --cpu-budget 4 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python -c "import json;d=json.load(open('$OUT/bench_$w.json'));r=d['roofline'] or {};print('$w', 'ms', round(d['ms_per_step'],5), 'val', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'frac', r.get('frac'), r.get('kernel'))"
done
