#!/bin/bash
# r02 session ax: dense sweep variant tests
OUT=gpurun_out/r02ax
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "sweep_variants" > $OUT/pytest_variants.log 2>&1; tail -3 $OUT/pytest_variants.log
