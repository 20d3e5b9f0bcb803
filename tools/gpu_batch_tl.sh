#!/bin/bash
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/batch_timeline.py
timeout 300 python tools/ab_perf.py "single-cta-batchpath"
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
