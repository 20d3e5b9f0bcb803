#!/bin/bash
# r02 session a: host facts, GPU suite after the seeded-call fixes, C4 W-prop
# tightness scan + O7 cost, sanitizers over every enforcement kernel.
OUT=gpurun_out/r02a
mkdir -p $OUT
(nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; nproc; lscpu | head -20; free -g) > $OUT/host.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
timeout 900 python tools/c4_scan.py > $OUT/c4_scan.jsonl 2> $OUT/c4_scan.err; cat $OUT/c4_scan.jsonl
OUT=$OUT SAN_TIMEOUT=500 bash tools/gpu_sanitize.sh
