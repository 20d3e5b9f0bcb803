#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
python paper_2407_11388_b200/build.py -DRAC_THREADS=1024 --out=$PWD/paper_2407_11388_b200/librac_t1024.so > /dev/null
timeout 300 python tools/ab_perf.py "A:512-coop"
RAC_NO_COOP=1 timeout 300 python tools/ab_perf.py "B:512-nocoop"
RAC_LIB_PATH=$PWD/paper_2407_11388_b200/librac_t1024.so timeout 300 python tools/ab_perf.py "C:1024-coop"
RAC_LIB_PATH=$PWD/paper_2407_11388_b200/librac_t1024.so RAC_NO_COOP=1 timeout 300 python tools/ab_perf.py "D:1024-nocoop"
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/timeline.py 2>&1 | tail -5
