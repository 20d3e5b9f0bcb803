#!/bin/bash
OUT=gpurun_out/${TAG:-tc}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests -m gpu -x -q -k "batch_pass_eval" > $OUT/pytest_tc.log 2>&1; tail -2 $OUT/pytest_tc.log
timeout 300 python tools/tc_ab.py > $OUT/tc_ab.log 2>&1; cat $OUT/tc_ab.log
timeout 600 ncu --set full --clock-control none -k regex:"rac_batch_tc_pass|rac_batch_bs_pass" -s 2 -c 2 -o $OUT/prof_tc_ab python tools/tc_ab.py > $OUT/ncu_tc.log 2>&1
tail -2 $OUT/ncu_tc.log
