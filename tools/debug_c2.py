"""Repeat the C2 W-seed parity case many times and report mismatches
(which (x,a), the oracle's removal epoch, the GPU's) -- debugging aid."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2407_11388_b200 import rac  # noqa: E402

t = float(os.environ.get("T", "0.0119"))
reps = int(os.environ.get("REPS", "20"))
dq, tq = synth.quant_density(1.0), synth.quant_tightness(t)
ctx = rac.RacContext.create_random(500, 20, dq, tq, 1)
orc = oracle.Oracle.from_synth(500, 20, dq, tq, 1)
root = synth.full_domains(np.full(500, 20))
o = orc.rac(root)
bad = 0
for k in range(3):
    ds, x0, v0 = synth.w_seed(o[1], 11, k)
    o2 = orc.rac(ds)
    for r in range(reps):
        g = ctx.enforce(ds, removed_at=True)
        diff = np.nonzero(g[1] != o2[1])[0]
        if g[0] != o2[0] or g[2] != o2[2] or len(diff):
            bad += 1
            xs, As = np.nonzero(g[3] != o2[3])
            info = [(int(x), int(a), int(o2[3][x, a]), int(g[3][x, a])) for x, a in zip(xs, As)]
            print("k=%d rep=%d status %s/%s iters %s/%s ndiff=%d (x,a,orc_epoch,gpu_epoch)=%s"
                  % (k, r, g[0], o2[0], g[2], o2[2], len(diff), info[:8]))
    print("k=%d seed var %d val %d iters %d removed/pass %s" % (
        k, x0, v0, o2[2], np.bincount(o2[3].ravel(), minlength=o2[2] + 1)[1:].tolist()))
print("bad runs:", bad, "of", 3 * reps, "env", {k: v for k, v in os.environ.items() if k.startswith("RAC_")})
