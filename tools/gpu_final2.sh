#!/bin/bash
# End-of-session check: smoke, whole GPU suite, default bench line.
OUT=gpurun_out/${TAG:-r01n}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_final.log 2>&1; tail -1 $OUT/smoke_final.log
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_final.log 2>&1; tail -2 $OUT/pytest_gpu_final.log
timeout 600 python bench.py > $OUT/bench_final_default.json 2> $OUT/bench_final_default.err; cut -c1-200 $OUT/bench_final_default.json
