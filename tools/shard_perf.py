"""Device time per enforcement of the sharded per-pass path on one GPU: fused kernel vs
virtual shards (row blocks, gather = no-op) vs the real NCCL leg (one-rank communicator)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import synth  # noqa: E402
from paper_2407_11388_b200 import rac  # noqa: E402


def timeit(fn, reps):
    t0 = time.time()
    while time.time() - t0 < 0.3:
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for (n, d, t, reps) in [(2000, 32, 0.5, 100), (2000, 32, 0.70, 30)]:
    res = []
    for label, kw in [("fused", {}), ("vshard1-nccl", {"nccl_self": True}), ("vshard2", {"virtual_shards": 2}),
                      ("vshard8", {"virtual_shards": 8})]:
        ctx = rac.RacContext.create_random(n, d, synth.quant_density(1.0), synth.quant_tightness(t), 1, **kw)
        din = torch.from_numpy(synth.full_domains(np.full(n, d)).view(np.int64).copy()).cuda()
        dout = torch.zeros_like(din)
        it = torch.zeros(1, dtype=torch.int32, device='cuda')
        st = torch.zeros(1, dtype=torch.int32, device='cuda')
        us = timeit(lambda: ctx.enforce_async(din, dout, it, st), reps)
        res.append(f"{label}={us:.1f}us(it{it.item()},launches {ctx.last_launch_count})")
        ctx.close()
    print(f"n={n} d={d} t={t}: " + " ".join(res), flush=True)
