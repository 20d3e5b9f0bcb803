#!/bin/bash
# A/B of the column sweep's loads in flight (RAC_UNROLL_C) + the dense parity tests that exercise it.
P=$PWD/paper_2407_11388_b200
python -c "import __graft_entry__ as g; g.build()"
for v in "" uc8; do
  RAC_LIB_PATH=$P/librac${v:+_$v}.so AB_SET=cols timeout 300 python tools/ab_perf.py "${v:-uc16}"
  RAC_LIB_PATH=$P/librac${v:+_$v}.so timeout 300 python tools/ab_perf.py "${v:-uc16}"
done
timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py -x -k "forced_layouts or c3 or c2 or back_to_back or corpus or c1 or golden or seeded" 2>&1 | tail -2
