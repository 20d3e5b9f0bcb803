#!/bin/bash
# r02 final session: smoke, full GPU suite, every bench line, the reference arm, launch list, ncu captures of the
# default bench kernel (C3 W-stream) and the batched kernel (C5)
OUT=gpurun_out/r02final
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > $OUT/gpu.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
python -c "import json;d=json.load(open('$OUT/bench_default.json'));print('default', d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline'].get('box_copy_gbs'), d['setup'].get('full_pass_sweep',{}).get('sweep'), d['e2e']['value'], d['clocks'])"
for w in c3-prop c3-seed c2-root c1-seed c5-batch c3s-stream c3s-prop w128-prop w128-batch; do
  timeout 600 python bench.py --workload $w --steps 400 --warmup 10 --cpu-budget 4 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python -c "import json;d=json.load(open('$OUT/bench_$w.json'));print('$w', d['ms_per_step'], d['value'], d['unit'], d['roofline'] and d['roofline'].get('frac'), d['e2e']['value'])"
done
timeout 900 python bench.py --workload c4-stream --steps 30 --warmup 3 --cpu-budget 20 > $OUT/bench_c4-stream.json 2> $OUT/bench_c4-stream.err
python -c "import json;d=json.load(open('$OUT/bench_c4-stream.json'));print('c4-stream', d['ms_per_step'], d['value'], d['roofline'].get('frac'))"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; tail -c 300 $OUT/bench_reference.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
   python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_bench.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rac_fused -s 12 -c 1 -o $OUT/prof_c3_stream \
   python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/ncu_c3_stream.log 2>&1
ncu -i $OUT/prof_c3_stream.ncu-rep --page raw --csv > $OUT/prof_c3_stream_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rac_batch_cl -s 3 -c 1 -o $OUT/prof_c5 \
   python bench.py --workload c5-batch --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ncu_c5.log 2>&1
ncu -i $OUT/prof_c5.ncu-rep --page raw --csv > $OUT/prof_c5_raw.csv 2>/dev/null
ls $OUT
