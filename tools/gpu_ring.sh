#!/bin/bash
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 300 python tools/ab_perf.py "ring"
RAC_NO_RING=1 timeout 300 python tools/ab_perf.py "no-ring"
RAC_FORCE_LAYOUT=cols timeout 300 python tools/ab_perf.py "ring-cols"
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
