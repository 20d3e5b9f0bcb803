#!/bin/bash
# r02 session t: rac_batch_cl with st.async DSMEM pushes + mbarrier (no per-pass MEMBAR.GPU); coop+cluster barrier probe
OUT=gpurun_out/r02t
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "batch" > $OUT/pytest_batch.log 2>&1; tail -3 $OUT/pytest_batch.log
for v in "" "RAC_BATCH_FULL=0"; do
  env $v timeout 300 python bench.py --workload c5-batch --steps 200 --warmup 10 --no-cpu-baseline > $OUT/bench_c5$(echo $v | tr '=/' '__').json 2> $OUT/bench_c5.err
  python -c "import json,glob,os;f=sorted(glob.glob('$OUT/bench_c5*.json'),key=os.path.getmtime)[-1];d=json.load(open(f));print('[$v]', d['ms_per_step'], d['value'], d['roofline'] and d['roofline'].get('frac'))"
done
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/batch_cl_timeline.py > $OUT/batch_cl_timeline.txt 2>&1; head -30 $OUT/batch_cl_timeline.txt
timeout 120 ./tools/probes/coop_cluster > $OUT/coop_cluster.jsonl 2>&1; cat $OUT/coop_cluster.jsonl
