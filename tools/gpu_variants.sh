#!/bin/bash
# Build librac variants (compile-time knobs) and compare device times.
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
P=$PWD/paper_2407_11388_b200
python $P/build.py -DRAC_MIN_BLOCKS=2 -DRAC_UNROLL_R=4 --out=$P/librac_v2.so > /dev/null
python $P/build.py -DRAC_MIN_BLOCKS=1 -DRAC_UNROLL_R=4 --out=$P/librac_v3.so > /dev/null
timeout 300 python tools/ab_perf.py "V1:minb1-ur8"
RAC_LIB_PATH=$P/librac_v2.so timeout 300 python tools/ab_perf.py "V2:minb2-ur4"
RAC_LIB_PATH=$P/librac_v3.so timeout 300 python tools/ab_perf.py "V3:minb1-ur4"
RAC_FORCE_LAYOUT=cols timeout 300 python tools/ab_perf.py "V1-cols"
RAC_FORCE_LAYOUT=rows timeout 300 python tools/ab_perf.py "V1-rows"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
