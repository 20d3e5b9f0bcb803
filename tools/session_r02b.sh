#!/bin/bash
# r02 session b: one-block kernel (rac_state) for batches and small instances,
# certification tests, A/B of block sizes, sanitizers on the new kernel.
OUT=gpurun_out/r02b
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python -m pytest tests/test_gpu_certify.py -q > $OUT/pytest_certify.log 2>&1; tail -3 $OUT/pytest_certify.log
for v in "" "RAC_STATE_T=32" "RAC_STATE_T=256" "RAC_BATCH_IMPL=bs" "RAC_SMALL_BYTES=3e7"; do
  env $v timeout 300 python tools/ab_perf.py "[$v]" >> $OUT/ab_state.log 2>&1
done
cat $OUT/ab_state.log
OUT=$OUT CASES="state batch" SAN_TIMEOUT=400 PEER_TOOLS="" bash tools/gpu_sanitize.sh
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
