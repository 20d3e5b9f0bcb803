"""Wide-domain (NEXT-4) timing and tightness sweep on one GPU: per (n, d, t)
the status / iterations of the root enforcement and its CUDA-event time
(median of 5 after 2 warm-ups), with pass-1 algorithmic bytes / time."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2407_11388_b200 import rac  # noqa: E402

cases = [(2000, 128, t) for t in (0.5, 0.93, 0.94, 0.945, 0.95, 0.955)] + \
        [(1000, 256, t) for t in (0.5, 0.97, 0.973, 0.976)]
dev = torch.device("cuda", 0)
for n, d, t in cases:
    t0 = time.time()
    ctx = rac.RacContext.create_random(n, d, synth.quant_density(1.0), synth.quant_tightness(t), 1)
    torch.cuda.synchronize()
    gen = time.time() - t0
    full = synth.full_domains_wide(np.full(n, d))
    din = torch.from_numpy(full.view(np.int64).copy()).to(dev)
    dout = torch.zeros_like(din)
    its = torch.zeros(1, dtype=torch.int32, device=dev)
    sts = torch.zeros(1, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream()
    for _ in range(2):
        ctx.enforce_async(din, dout, its, sts, stream=s)
    ms = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        ctx.enforce_async(din, dout, its, sts, stream=s)
        b.record(s)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    out = dout.cpu().numpy().view(np.uint64)
    live = int(sum(bin(int(v)).count("1") for v in out))
    pass1 = n * d * (n - 1) * d / 8.0
    med = float(np.median(ms))
    print(json.dumps({"n": n, "d": d, "t": t, "gen_s": round(gen, 2), "status": int(sts.item()),
                      "iters": int(its.item()), "live_out": live, "ms": round(med, 4),
                      "pass1_GBps_if_1pass": round(pass1 / med / 1e6, 1)}), flush=True)
    del ctx
    torch.cuda.empty_cache()
