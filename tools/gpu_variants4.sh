#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
P=$PWD/paper_2407_11388_b200
python $P/build.py -DRAC_UNROLL_R=16 --out=$P/librac_ur16.so > /dev/null
python $P/build.py -DRAC_UNROLL_R=12 --out=$P/librac_ur12.so > /dev/null
python $P/build.py -DRAC_UNROLL_R=16 -DRAC_UNROLL_C=16 --out=$P/librac_ur16c16.so > /dev/null
timeout 300 python tools/ab_perf.py "V1:ur8"
RAC_LIB_PATH=$P/librac_ur16.so timeout 300 python tools/ab_perf.py "ur16"
RAC_LIB_PATH=$P/librac_ur12.so timeout 300 python tools/ab_perf.py "ur12"
RAC_LIB_PATH=$P/librac_ur16c16.so timeout 300 python tools/ab_perf.py "ur16c16"
