#!/bin/bash
OUT=gpurun_out/${TAG:-prof}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
for w in ${WORKLOADS:-c1-seed c2-root}; do
  timeout 600 python bench.py --workload $w --steps 300 --warmup 10 --no-cpu-baseline > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python -c "
import json,sys
d=json.loads(open('$OUT/bench_$w.json').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$w', 'value=%.1f ms=%.4f frac=%s launches=%s' % (d['value'], d['ms_per_step'], r.get('frac'), d.get('gpu_launches')), d.get('enforcement'))
"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 40 --csv --log-file $OUT/launches_$w.csv \
     python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
  python - $OUT/launches_$w.csv <<'PY'
import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
h=None
for i,r in enumerate(rows):
    if 'Kernel Name' in r: h=i; break
if h is None: print('no launches'); sys.exit()
H=rows[h]; ki=H.index('Kernel Name'); vi=H.index('Metric Value')
from collections import defaultdict
agg=defaultdict(list)
for r in rows[h+1:]:
    if len(r)>vi: agg[r[ki][:50]].append(float(r[vi].replace(',','')))
for k,v in agg.items(): print('   ', len(v), k, 'mean ns', int(sum(v)/len(v)))
PY
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rac_fused|rac_batch" -s 10 -c 1 -o $OUT/prof_$w \
     python bench.py --workload $w --steps 12 --warmup 5 --no-cpu-baseline > $OUT/ncu_$w.log 2>&1
done
ls $OUT
