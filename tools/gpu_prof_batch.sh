#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rac_batch_bs -s 3 -c 1 -o gpurun_out/prof_batch_bs \
   python bench.py --workload c5-batch --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_batch.log 2>&1
tail -3 gpurun_out/ncu_batch.log
