#!/bin/bash
# r02 session ao: full passes on HBM-resident tensors tie-break to the row sweep (default) vs the column sweep (tiecols)
OUT=gpurun_out/r02ao
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
python - <<'PY' > $OUT/copy_bw.txt 2>&1
import torch
a = torch.empty(1 << 29, dtype=torch.bfloat16, device='cuda'); b = torch.empty_like(a)
for _ in range(3): b.copy_(a)
torch.cuda.synchronize(); best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print("copy 1 GiB: %.1f GB/s" % (2 * (1 << 29) * 2 / (best / 1e3) / 1e9))
PY
cat $OUT/copy_bw.txt
for r in 1 2; do
  AB_SET=fused timeout 300 python tools/ab_perf.py tierows >> $OUT/ab_tie.log 2>&1
  RAC_FORCE_LAYOUT=tiecols AB_SET=fused timeout 300 python tools/ab_perf.py tiecols >> $OUT/ab_tie.log 2>&1
  AB_SET=sparse timeout 300 python tools/ab_perf.py sparse >> $OUT/ab_tie.log 2>&1
done
cat $OUT/ab_tie.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
python -c "import json;d=json.load(open('$OUT/bench_default.json'));print('default', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline'].get('box_copy_gbs'), d['e2e']['value'], d['clocks'])"
for w in c3-prop c3-seed c4-stream; do
  timeout 600 python bench.py --workload $w --steps 200 --warmup 5 --cpu-budget 3 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python -c "import json;d=json.load(open('$OUT/bench_$w.json'));print('$w', d['ms_per_step'], d['value'], d['roofline'] and d['roofline'].get('frac'))"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_certify.py -q -x --timeout 900 > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
