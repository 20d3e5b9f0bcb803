"""Device time per C1 enforcement (CUDA graph of 50 calls, so no host launch
overhead is included) split into a fixed part (an empty seed list: staging and
output only, no pass) and the passes (root: 2 passes, seeded: 3), for the
one-warp kernel (rac_tiny) and the one-block kernel (rac_state, RAC_NO_TINY=1)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2407_11388_b200 import rac  # noqa: E402


def graph_us(fn, reps=20, per=50):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(per):
            fn(s)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / (reps * per)


for variant in ("tiny", "block"):
    if variant == "block":
        os.environ["RAC_NO_TINY"] = "1"
    ctx = rac.RacContext.create_random(20, 8, synth.quant_density(0.5), synth.quant_tightness(0.4), 1)
    full = synth.full_domains(np.full(20, 8))
    _, root, _ = ctx.enforce(full)
    ds, sx, _ = synth.w_seed(root, 1)
    din = torch.from_numpy(ds.view(np.int64).copy()).cuda()
    dfull = torch.from_numpy(full.view(np.int64).copy()).cuda()
    dout = torch.zeros_like(din)
    it = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    sv = torch.tensor([sx], dtype=torch.int32, device="cuda")
    out = {"variant": variant, "path": ctx.path}
    out["no_pass_us"] = graph_us(lambda s: ctx.enforce_seeded_async(din, dout, it, st, sv, 0, stream=s))
    out["seeded_us"] = graph_us(lambda s: ctx.enforce_seeded_async(din, dout, it, st, sv, 1, stream=s))
    out["seeded_iters"] = int(it.item())
    out["root_us"] = graph_us(lambda s: ctx.enforce_async(dfull, dout, it, st, stream=s))
    out["root_iters"] = int(it.item())
    x = torch.zeros(1, device="cuda")
    out["tiny_torch_kernel_us"] = graph_us(lambda s: x.add_(1))
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in out.items()}), flush=True)
    ctx.close()
