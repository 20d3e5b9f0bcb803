"""Device time per enforcement for a few workloads (A/B knobs come from the env:
RAC_LIB_PATH, RAC_NO_COOP, RAC_BATCH_IMPL)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import synth  # noqa: E402
from paper_2407_11388_b200 import rac  # noqa: E402


def timeit(fn, reps):
    import time
    t0 = time.time()
    while time.time() - t0 < 0.3:  # let the SM clock ramp up before timing
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def single(name, n, d, p, t, kind="root", reps=200):
    ctx = rac.RacContext.create_random(n, d, synth.quant_density(p), synth.quant_tightness(t), 1)
    full = synth.full_domains(np.full(n, d))
    d_in, sx = full, None
    if kind == "seed":
        _, root, _ = ctx.enforce(full)
        d_in, sx, _ = synth.w_seed(root, 1)
    din = torch.from_numpy(d_in.view(np.int64).copy()).cuda()
    dout = torch.zeros_like(din)
    it = torch.zeros(1, dtype=torch.int32, device='cuda')
    st = torch.zeros(1, dtype=torch.int32, device='cuda')
    if kind == "seed":
        sv = torch.tensor([sx], dtype=torch.int32, device='cuda')
        us = timeit(lambda: ctx.enforce_seeded_async(din, dout, it, st, sv, 1), reps)
    else:
        us = timeit(lambda: ctx.enforce_async(din, dout, it, st), reps)
    return f"{name}={us:.1f}us(it{it.item()})"


def batch(S=1024):
    n, d = 200, 16
    ctx = rac.RacContext.create_random(n, d, synth.quant_density(0.8), synth.quant_tightness(0.3), 1)
    _, root, _ = ctx.enforce(synth.full_domains(np.full(n, d)))
    states, seeds = synth.dive_states(root, lambda D: ctx.enforce(D)[:2], S, seed=1, return_seeds=True)
    din = torch.from_numpy(np.stack(states).view(np.int64)).cuda()
    dout = torch.zeros_like(din)
    its = torch.zeros(S, dtype=torch.int32, device='cuda')
    sts = torch.zeros(S, dtype=torch.int32, device='cuda')
    sv = torch.from_numpy(np.asarray(seeds, dtype=np.int32)).cuda()
    us1 = timeit(lambda: ctx.enforce_batch_seeded(S, din, dout, its, sts, sv), 20)
    us2 = timeit(lambda: ctx.enforce_batch(S, din, dout, its, sts), 20)
    return f"c5batch_seeded={us1:.0f}us c5batch={us2:.0f}us"


tag = sys.argv[1] if len(sys.argv) > 1 else ""
if os.environ.get("AB_SET") == "cols":  # column-sweep workloads only
    os.environ["RAC_FORCE_LAYOUT"] = "cols"
    print(tag, "cols:", single("c3stream", 2000, 32, 1.0, 0.5), single("c3prop", 2000, 32, 1.0, 0.70, reps=50),
          single("c3seed", 2000, 32, 1.0, 0.5, "seed", 100), flush=True)
    del os.environ["RAC_FORCE_LAYOUT"]
    print(tag, "auto:", single("c3prop", 2000, 32, 1.0, 0.70, reps=50), single("c3seed", 2000, 32, 1.0, 0.5, "seed", 100),
          single("c2", 500, 20, 1.0, 0.3, reps=1000), flush=True)
    sys.exit(0)
if os.environ.get("AB_SET") == "small":
    print(tag, single("c1seed", 20, 8, 0.5, 0.4, "seed", 2000), single("c1root", 20, 8, 0.5, 0.4, "root", 2000),
          flush=True)
    sys.exit(0)
if os.environ.get("AB_SET") == "fused":
    print(tag, single("c2", 500, 20, 1.0, 0.3, reps=1000), single("c3stream", 2000, 32, 1.0, 0.5, reps=200),
          single("c3prop", 2000, 32, 1.0, 0.70, reps=100), single("c3seed", 2000, 32, 1.0, 0.5, "seed", 200),
          single("c4stream", 8000, 64, 1.0, 0.5, reps=10), flush=True)
    sys.exit(0)
if os.environ.get("AB_SET") == "batch":
    print(tag, batch(), flush=True)
    sys.exit(0)
if os.environ.get("AB_SET") == "sparse":
    print(tag, single("c3s_stream", 4000, 32, 0.25, 0.5, reps=100), single("c3s_prop", 4000, 32, 0.25, 0.72, reps=50),
          flush=True)
    sys.exit(0)
print(tag, single("c1seed", 20, 8, 0.5, 0.4, "seed", 2000), single("c5single_seed", 200, 16, 0.8, 0.3, "seed", 1000),
      single("c2", 500, 20, 1.0, 0.3, reps=1000), single("c3stream", 2000, 32, 1.0, 0.5),
      single("c3prop", 2000, 32, 1.0, 0.70, reps=50), single("c3seed", 2000, 32, 1.0, 0.5, "seed", 100),
      batch(), flush=True)
