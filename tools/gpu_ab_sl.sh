#!/bin/bash
# A/B: column-sweep slabs per item (RAC_COL_SLABS) and an ncu capture of the sparse sweep.
OUT=gpurun_out/${TAG:-ab_sl}
mkdir -p $OUT
P=$PWD/paper_2407_11388_b200
python -c "import __graft_entry__ as g; g.build(); g.smoke()" | tail -1
for v in "" sl2 sl4; do
  lib=$P/librac${v:+_$v}.so
  RAC_LIB_PATH=$lib AB_SET=cols timeout 300 python tools/ab_perf.py "${v:-sl1}"
done 2>&1 | tee $OUT/ab_sl.log
for v in "" sl4; do RAC_LIB_PATH=$P/librac${v:+_$v}.so AB_SET=sparse timeout 300 python tools/ab_perf.py "sparse${v}"; done 2>&1 | tee -a $OUT/ab_sl.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rac_fused -s 3 -c 1 -o $OUT/prof_c3s_stream \
   python bench.py --workload c3s-stream --steps 5 --warmup 3 --no-cpu-baseline > $OUT/ncu_c3s.log 2>&1
ls $OUT
