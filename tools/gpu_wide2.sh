#!/bin/bash
# Wide seeded calls: GPU parity tests of rac_wide.cu, timing sweeps.
OUT=gpurun_out/${TAG:-r01n}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_wide.py -q > $OUT/pytest_gpu_wide.log 2>&1; tail -2 $OUT/pytest_gpu_wide.log
timeout 600 python tools/wide_seeded_perf.py > $OUT/wide_seeded_perf.jsonl 2> $OUT/wide_seeded_perf.err; cat $OUT/wide_seeded_perf.jsonl
timeout 900 python tools/wide_perf.py > $OUT/wide_perf.jsonl 2> $OUT/wide_perf.err; cat $OUT/wide_perf.jsonl
ls $OUT
