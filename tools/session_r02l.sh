#!/bin/bash
# r02 session l: rac_tiny phase stamps; blocking-call CUDA graph (e2e)
OUT=gpurun_out/r02l
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/timeline.py > $OUT/timeline.txt 2>&1; head -2 $OUT/timeline.txt
timeout 300 python tools/e2e_probe.py > $OUT/e2e_probe.jsonl 2>&1; cat $OUT/e2e_probe.jsonl
RAC_NO_BLOCKING_GRAPH=1 timeout 300 python tools/e2e_probe.py > $OUT/e2e_probe_nograph.jsonl 2>&1; cat $OUT/e2e_probe_nograph.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py -k "spec_corpus or golden or c1 or seeded or async or search" -q > $OUT/pytest_sel.log 2>&1; tail -2 $OUT/pytest_sel.log
