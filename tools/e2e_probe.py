"""Where the time of a blocking host-buffer call goes (C1 W-seed and C3 W-stream):
host wall clock per call of rac_enforce[_seeded] against its parts -- a bare
ctypes call, an empty stream round trip, the async call + synchronize -- and
the kernel's device time (CUDA events on back-to-back async calls)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2407_11388_b200 import rac  # noqa: E402


def wall(fn, reps):
    for _ in range(20):
        fn()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t) / reps * 1e6


for name, (n, d, p, t, kind) in {"c1-seed": (20, 8, 0.5, 0.4, "seed"), "c3-stream": (2000, 32, 1.0, 0.5, "root")}.items():
    ctx = rac.RacContext.create_random(n, d, synth.quant_density(p), synth.quant_tightness(t), 1)
    full = synth.full_domains(np.full(n, d))
    d_in, sx = full, None
    if kind == "seed":
        _, root, _ = ctx.enforce(full)
        d_in, sx, _ = synth.w_seed(root, 1)
    din = torch.from_numpy(d_in.view(np.int64).copy()).cuda()
    dout = torch.zeros_like(din)
    it = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    sv = torch.tensor([sx if sx is not None else 0], dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    if kind == "seed":
        def async_call():
            ctx.enforce_seeded_async(din, dout, it, st, sv, 1, stream=s)

        def host_call():
            ctx.enforce_seeded(d_in, [sx])
    else:
        def async_call():
            ctx.enforce_async(din, dout, it, st, stream=s)

        def host_call():
            ctx.enforce(d_in)
    reps = 2000 if n < 100 else 300
    out = {"workload": name, "path": ctx.path}
    out["ctypes_call_us"] = wall(lambda: rac.lib.rac_n_vars(ctx._h), 20000)
    out["empty_roundtrip_us"] = wall(lambda: (torch.cuda._sleep(0), torch.cuda.synchronize()), reps)
    out["async_enqueue_us"] = wall(async_call, reps)
    torch.cuda.synchronize()
    out["async_plus_sync_us"] = wall(lambda: (async_call(), torch.cuda.synchronize()), reps)
    out["blocking_call_us"] = wall(host_call, reps)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(s)
    try:
        with torch.cuda.graph(g, stream=cs):
            for _ in range(50):
                if kind == "seed":
                    ctx.enforce_seeded_async(din, dout, it, st, sv, 1, stream=cs)
                else:
                    ctx.enforce_async(din, dout, it, st, stream=cs)
        g.replay()
        torch.cuda.synchronize()
        a.record()
        for _ in range(20):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        out["device_us_graph_per_step"] = a.elapsed_time(b) * 1e3 / (20 * 50)
    except Exception as e:
        out["graph_error"] = repr(e)[:200]
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in out.items()}), flush=True)
