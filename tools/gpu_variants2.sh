#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
P=$PWD/paper_2407_11388_b200
python $P/build.py -DRAC_MIN_BLOCKS=2 -DRAC_UNROLL_R=4 -DRAC_UNROLL_C=4 -DRAC_UNROLL_L=4 --out=$P/librac_v6.so > /dev/null
python $P/build.py -DRAC_MIN_BLOCKS=2 -DRAC_UNROLL_R=4 -DRAC_UNROLL_C=8 -DRAC_UNROLL_L=4 --out=$P/librac_v7.so > /dev/null
python $P/build.py -DRAC_MIN_BLOCKS=1 -DRAC_UNROLL_R=8 -DRAC_UNROLL_C=8 -DRAC_UNROLL_L=4 --out=$P/librac_v8.so > /dev/null
timeout 300 python tools/ab_perf.py "V1-default"
RAC_LIB_PATH=$P/librac_v6.so timeout 300 python tools/ab_perf.py "V6:mb2-r4-c4-l4"
RAC_LIB_PATH=$P/librac_v7.so timeout 300 python tools/ab_perf.py "V7:mb2-r4-c8-l4"
RAC_LIB_PATH=$P/librac_v8.so timeout 300 python tools/ab_perf.py "V8:mb1-r8-c8-l4"
RAC_LIB_PATH=$P/librac_v6.so RAC_FORCE_LAYOUT=cols timeout 300 python tools/ab_perf.py "V6-cols"
RAC_LIB_PATH=$P/librac_v7.so RAC_FORCE_LAYOUT=cols timeout 300 python tools/ab_perf.py "V7-cols"
