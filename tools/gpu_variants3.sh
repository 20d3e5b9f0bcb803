#!/bin/bash
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
P=$PWD/paper_2407_11388_b200
python $P/build.py -DRAC_RING_COLS=4 -DRAC_RING_STAGES=4 --out=$P/librac_r44.so > /dev/null
python $P/build.py -DRAC_RING_COLS=6 -DRAC_RING_STAGES=3 --out=$P/librac_r63.so > /dev/null
timeout 300 python tools/ab_perf.py "ring8x2"
RAC_NO_RING=1 timeout 300 python tools/ab_perf.py "no-ring"
RAC_LIB_PATH=$P/librac_r44.so timeout 300 python tools/ab_perf.py "ring4x4"
RAC_LIB_PATH=$P/librac_r63.so timeout 300 python tools/ab_perf.py "ring6x3"
RAC_FORCE_LAYOUT=cols timeout 300 python tools/ab_perf.py "ring8x2-cols"
RAC_LIB_PATH=$P/librac_r44.so RAC_FORCE_LAYOUT=cols timeout 300 python tools/ab_perf.py "ring4x4-cols"
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
