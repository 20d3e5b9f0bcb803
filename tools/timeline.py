"""Phase timeline of the fused kernel (CTA 0, %globaltimer) for a few workloads.
Run with RAC_DEBUG_TIMELINE=1 on a GPU box."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
os.environ.setdefault("RAC_DEBUG_TIMELINE", "1")
import synth  # noqa: E402
from paper_2407_11388_b200 import rac  # noqa: E402

lib = rac.lib
lib.rac_debug_timeline.restype = ctypes.c_int
lib.rac_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]


def run(name, n, d, p, t, kind="root"):
    ctx = rac.RacContext.create_random(n, d, synth.quant_density(p), synth.quant_tightness(t), 1)
    full = synth.full_domains(np.full(n, d))
    d_in = full
    sx = None
    if kind == "seed":
        _, root, _ = ctx.enforce(full)
        d_in, sx, _ = synth.w_seed(root, 1)
    din = torch.from_numpy(d_in.view(np.int64).copy()).cuda()
    dout = torch.zeros_like(din)
    it = torch.zeros(1, dtype=torch.int32, device='cuda')
    st = torch.zeros(1, dtype=torch.int32, device='cuda')
    sv = torch.tensor([sx if sx is not None else 0], dtype=torch.int32, device='cuda')
    for _ in range(5):
        if sx is not None:  # the seeded call (Alg. 1 tensorAC(Vars, [idx]), as bench.py times it)
            ctx.enforce_seeded_async(din, dout, it, st, sv, 1)
        else:
            ctx.enforce_async(din, dout, it, st)
    torch.cuda.synchronize()
    buf = (ctypes.c_uint64 * 256)()
    k = lib.rac_debug_timeline(ctx._h, buf, 256)
    ts = [buf[i] for i in range(k)]
    if len(ts) < 2:
        print(f"{name}: no timeline", flush=True)
        return
    d_ns = [ts[i + 1] - ts[i] for i in range(k - 1)]
    print(f"{name} [{ctx.path}]: iters={it.item()} total={ts[-1]-ts[0]} ns  phases(ns)={d_ns}", flush=True)


run("c1-seed", 20, 8, 0.5, 0.4, "seed")
run("c5-single", 200, 16, 0.8, 0.3, "seed")
run("c2-root", 500, 20, 1.0, 0.3)
run("c3-stream", 2000, 32, 1.0, 0.5)
run("c3-prop", 2000, 32, 1.0, 0.70)
run("c3-seed", 2000, 32, 1.0, 0.5, "seed")
run("c3s-prop", 4000, 32, 0.25, 0.72)
