#!/bin/bash
# A/B: chunked dynamic claiming (RAC_CLAIM_K items per atomic) in the column / sparse sweeps.
P=$PWD/paper_2407_11388_b200
python -c "import __graft_entry__ as g; g.build()"
for k in 1 2; do for v in "" k4 k8; do
  RAC_LIB_PATH=$P/librac${v:+_$v}.so timeout 300 python tools/ab_perf.py "${v:-static}"
  RAC_LIB_PATH=$P/librac${v:+_$v}.so AB_SET=sparse timeout 300 python tools/ab_perf.py "${v:-static}"
done; done
