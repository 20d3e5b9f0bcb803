#!/bin/bash
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 300 python tools/ab_perf.py "default"
RAC_FORCE_LAYOUT=cols timeout 300 python tools/ab_perf.py "cols-only"
RAC_FORCE_LAYOUT=rows timeout 300 python tools/ab_perf.py "rows-only"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
