#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python tools/table1.py 2000 100,250,500,750,1000 --ac3 > gpurun_out/table1.log 2>&1
tail -3 gpurun_out/table1.log
