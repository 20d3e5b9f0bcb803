#!/bin/bash
# r02 session s: ncu source-level profile of the rewritten rac_batch_cl (C5), e2e probe with graph-captured blocking calls
OUT=gpurun_out/r02s
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 600 python tools/e2e_probe.py > $OUT/e2e_probe.jsonl 2>&1; cat $OUT/e2e_probe.jsonl
RAC_BLOCKING_GRAPH=small timeout 600 python tools/e2e_probe.py > $OUT/e2e_probe_small.jsonl 2>&1; cat $OUT/e2e_probe_small.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rac_batch_cl -s 3 -c 1 -o $OUT/prof_c5 \
   python bench.py --workload c5-batch --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ncu_c5.log 2>&1
ncu -i $OUT/prof_c5.ncu-rep --page raw --csv > $OUT/prof_c5_raw.csv 2>/dev/null
ncu -i $OUT/prof_c5.ncu-rep --page source --csv --print-source sass > $OUT/prof_c5_source_sass.csv 2>/dev/null
ncu -i $OUT/prof_c5.ncu-rep --page source --csv > $OUT/prof_c5_source.csv 2>/dev/null
ncu -i $OUT/prof_c5.ncu-rep --page details --csv > $OUT/prof_c5_details.csv 2>/dev/null
ls -la $OUT
