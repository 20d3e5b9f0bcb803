#!/bin/bash
# NEXT-4 evidence session: smoke, GPU tests, wide-domain bench lines + default line,
# launch list and one ncu --set full capture of wide_fused, memcheck of the wide tests.
OUT=gpurun_out/${TAG:-r01n}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for w in w128-stream w128-prop w256-stream; do
  timeout 600 python bench.py --workload $w --steps 30 --warmup 3 --cpu-budget 10 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches_w128.csv \
   python bench.py --workload w128-stream --steps 10 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_w128.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wide_fused -s 3 -c 1 -o $OUT/prof_w128_stream \
   python bench.py --workload w128-stream --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ncu_w128_stream.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wide_fused -s 3 -c 1 -o $OUT/prof_w128_prop \
   python bench.py --workload w128-prop --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ncu_w128_prop.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests -m gpu -q -k wide -x > $OUT/sanitizer_memcheck_wide.log 2>&1; echo "memcheck rc=$?" >> $OUT/sanitizer_memcheck_wide.log
tail -n 2 $OUT/sanitizer_memcheck_wide.log
ls $OUT
