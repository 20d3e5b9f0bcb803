#!/bin/bash
# Round-end style session: tests, bench lines, ncu evidence, sanitizers.
OUT=gpurun_out/${TAG:-final}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for w in c3-prop c3-seed c2-root c1-seed c5-batch c3s-stream c3s-prop; do
  timeout 600 python bench.py --workload $w --steps 1000 --warmup 10 --cpu-budget 8 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
done
timeout 900 python bench.py --workload c4-stream --steps 30 --warmup 3 --cpu-budget 20 > $OUT/bench_c4-stream.json 2> $OUT/bench_c4-stream.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
   python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_bench.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rac_fused -s 5 -c 1 -o $OUT/prof_c3_stream \
   python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/ncu_c3_stream.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rac_fused -s 5 -c 1 -o $OUT/prof_c3_prop \
   python bench.py --workload c3-prop --steps 6 --warmup 3 --no-cpu-baseline > $OUT/ncu_c3_prop.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rac_fused -s 3 -c 1 -o $OUT/prof_c3s_stream \
   python bench.py --workload c3s-stream --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ncu_c3s_stream.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rac_batch_bs -s 3 -c 1 -o $OUT/prof_c5_batch \
   python bench.py --workload c5-batch --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ncu_c5_batch.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/sanitizer_memcheck.log 2>&1; echo "memcheck rc=$?" >> $OUT/sanitizer_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/sanitizer_racecheck.log 2>&1; echo "racecheck rc=$?" >> $OUT/sanitizer_racecheck.log
for f in $OUT/sanitizer_memcheck.log $OUT/sanitizer_racecheck.log; do tail -n 2 $f; done
ls $OUT
