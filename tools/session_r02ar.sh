#!/bin/bash
# r02 session ar: per-CTA stamps of the seeded C3 call (pass-1 skew)
OUT=gpurun_out/r02ar
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python tools/cta_stamps.py --seed > $OUT/cta_seed.txt 2>&1; cat $OUT/cta_seed.txt
timeout 300 python tools/cta_stamps.py > $OUT/cta_stream.txt 2>&1; cat $OUT/cta_stream.txt
