#!/bin/bash
# r02 session aj: blocking-call input staging by a one-block kernel reading pinned host memory vs the copy engine (e2e A/B)
OUT=gpurun_out/r02aj
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
for r in 1 2; do
  timeout 300 python tools/e2e_probe.py >> $OUT/e2e_copyengine.jsonl 2>&1
  RAC_BLOCKING_STAGE_KERNEL=1 timeout 300 python tools/e2e_probe.py >> $OUT/e2e_stagekernel.jsonl 2>&1
done
cat $OUT/e2e_copyengine.jsonl $OUT/e2e_stagekernel.jsonl
RAC_BLOCKING_STAGE_KERNEL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "c3 or seeded or corpus" > $OUT/pytest_stagekernel.log 2>&1; tail -2 $OUT/pytest_stagekernel.log
