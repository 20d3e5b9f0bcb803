"""C4 (n=8000, d=64, density 1) tightness scan on one GPU for the W-prop
workload (t* = (-ln(1-f)/deg)^(1/d) ~ 0.82 predicts a consistent
10-20 pass enforcement), then the O7 certificate of the chosen enforcement on
this host's cores (its cost sets what the GPU test suite can afford)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2407_11388_b200 import rac  # noqa: E402

n, d = 8000, 64
dq = synth.quant_density(1.0)
root = synth.full_domains(np.full(n, d))
print(json.dumps({"nproc": os.cpu_count()}), flush=True)
best = None
for t in [float(a) for a in sys.argv[1:]] or (0.80, 0.81, 0.815, 0.82, 0.825, 0.83, 0.835, 0.84, 0.85):
    tq = synth.quant_tightness(t)
    ctx = rac.RacContext.create_random(n, d, dq, tq, 1)
    t0 = time.time()
    st, out, it, rem = ctx.enforce(root, removed_at=True)
    el = time.time() - t0
    removed = int((rem > 0).sum())
    print(json.dumps({"t": t, "status": int(st), "iters": int(it), "removed": removed, "s": round(el, 3)}), flush=True)
    if st == 0 and 8 <= it <= 25 and best is None:
        best = (t, tq, st, out, it, rem)
    ctx.close()
if best is not None:
    t, tq, st, out, it, rem = best
    t0 = time.time()
    r = oracle.certify_trajectory_synth(n, d, dq, tq, 1, root, out, rem, it, st, False, 0)
    print(json.dumps({"certify_t": t, "result": r, "seconds": round(time.time() - t0, 1)}), flush=True)
