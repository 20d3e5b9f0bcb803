#!/bin/bash
# r02 session m: rac_tiny as a 256-thread block (row per thread, 4 masks in flight)
OUT=gpurun_out/r02m
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 300 python tools/c1_probe.py > $OUT/c1_probe.jsonl 2>&1; cat $OUT/c1_probe.jsonl
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/timeline.py > $OUT/timeline.txt 2>&1; head -1 $OUT/timeline.txt
timeout 300 python tools/e2e_probe.py > $OUT/e2e_probe.jsonl 2>&1; head -1 $OUT/e2e_probe.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py -k "spec_corpus or golden or c1 or seeded or async or search or nonuniform" tests/test_gpu_certify.py -k "seeded_empty or seeded_lists" -q > $OUT/pytest_sel.log 2>&1; tail -2 $OUT/pytest_sel.log
