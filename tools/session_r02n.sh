#!/bin/bash
# r02 session n: LUT-expanded tcgen05 wide pass A/B + wide enforcement for scale; test sweep of the small-instance and batched paths
OUT=gpurun_out/r02n
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python tools/wide_tc_ab.py > $OUT/wide_tc_ab.jsonl 2>&1; cat $OUT/wide_tc_ab.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wide_tc_pass -c 1 -o $OUT/prof_wide_tc \
   python tools/wide_tc_ab.py > $OUT/ncu_wide_tc.log 2>&1
ncu -i $OUT/prof_wide_tc.ncu-rep --page raw --csv > $OUT/prof_wide_tc_raw.csv 2>/dev/null
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_certify.py tests/test_gpu_wide.py -q -x --timeout 900 > $OUT/pytest_sel.log 2>&1; tail -3 $OUT/pytest_sel.log
