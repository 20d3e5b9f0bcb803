#!/bin/bash
# r02 session d: batched kernel with one 32-state word per cluster (rac_batch_cl)
OUT=gpurun_out/r02d
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python -m pytest tests/test_gpu_certify.py -q -k "batched" tests/test_gpu_parity.py -k "c5 or batched or batch" > $OUT/pytest_batch.log 2>&1; tail -3 $OUT/pytest_batch.log
for v in "" "RAC_BATCH_CL=1" "RAC_BATCH_CL=2" "RAC_BATCH_CL=8" "RAC_BATCH_IMPL=bs"; do
  env $v AB_SET=batch timeout 300 python tools/ab_perf.py "[$v]" >> $OUT/ab_batch.log 2>&1
done
cat $OUT/ab_batch.log
timeout 600 python bench.py --workload c5-batch --steps 200 --warmup 10 --cpu-budget 8 > $OUT/bench_c5-batch.json 2> $OUT/bench_c5-batch.err
python -c "import json;d=json.load(open('$OUT/bench_c5-batch.json'));print('c5', d['value'], d['ms_per_step'], d['roofline'], d['cpu_baseline']['value'], d['cpu_baseline']['cores'])"
OUT=$OUT CASES="batch" SAN_TIMEOUT=400 PEER_TOOLS="" bash tools/gpu_sanitize.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rac_batch_cl -s 3 -c 1 -o $OUT/prof_c5_batch_cl \
   python bench.py --workload c5-batch --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ncu_c5.log 2>&1
ncu -i $OUT/prof_c5_batch_cl.ncu-rep --page raw --csv > $OUT/prof_c5_batch_cl_raw.csv 2>/dev/null
