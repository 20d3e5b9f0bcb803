#!/bin/bash
# One GPU session: bench lines for every workload, the reference arm, the ncu
# launch list of the default bench command and one full ncu capture of the
# dominant kernel.  Outputs under gpurun_out/ (scratch); summaries get copied
# into profiles/ by hand.
set -x
OUT=gpurun_out/${TAG:-r01}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for w in c3-prop c2-root c1-seed c5-batch; do
  timeout 600 python bench.py --workload $w --steps 500 --warmup 10 --cpu-budget 8 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
done
timeout 900 python bench.py --workload c4-stream --steps 50 --warmup 3 --cpu-budget 20 > $OUT/bench_c4-stream.json 2> $OUT/bench_c4-stream.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
   python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_bench.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rac_fused -s 5 -c 2 -o $OUT/prof_c3_stream \
   python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rac_fused -s 5 -c 1 -o $OUT/prof_c3_prop \
   python bench.py --workload c3-prop --steps 6 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_prop.log 2>&1
ls -la $OUT
