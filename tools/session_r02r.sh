#!/bin/bash
# r02 session r: rac_batch_cl rewrite (chunk tables 6+5+5, full-row sweep, exact per-state columns, split cluster barrier + DSMEM push)
OUT=gpurun_out/r02r
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "batch" > $OUT/pytest_batch.log 2>&1; tail -3 $OUT/pytest_batch.log
for v in "" "RAC_BATCH_FULL=0" "RAC_BATCH_FULL=1/2" "RAC_BATCH_FULL=19/20"; do
  env $v timeout 300 python bench.py --workload c5-batch --steps 200 --warmup 10 --no-cpu-baseline > $OUT/bench_c5$(echo $v | tr '=/' '__').json 2> $OUT/bench_c5.err
  python -c "import json,glob,os;f=sorted(glob.glob('$OUT/bench_c5*.json'),key=os.path.getmtime)[-1];d=json.load(open(f));print('[$v]', d['ms_per_step'], d['value'], d['roofline'] and d['roofline'].get('frac'))"
done
RAC_DEBUG_TIMELINE=1 timeout 300 python tools/batch_cl_timeline.py > $OUT/batch_cl_timeline.txt 2>&1; head -45 $OUT/batch_cl_timeline.txt
CASES=batch TOOLS="memcheck racecheck synccheck" OUT=$OUT bash tools/gpu_sanitize.sh 2>&1 | grep -v peer | head -5
