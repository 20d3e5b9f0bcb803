#!/bin/bash
# A/B of the sparse sweep's loads in flight (RAC_UNROLL_S) + sparse parity tests.
P=$PWD/paper_2407_11388_b200
python -c "import __graft_entry__ as g; g.build()"
for v in "" us12 us16; do RAC_LIB_PATH=$P/librac${v:+_$v}.so AB_SET=sparse timeout 300 python tools/ab_perf.py "sparse${v:-_us8}"; done
timeout 600 python -m pytest -q -m gpu tests/test_gpu_parity.py -k sparse 2>&1 | tail -2
