"""A/B of one batched Eq. 1 pass on wide domains (NEXT-4): bit-sliced byte
tables (impl 2) vs pipelined tcgen05 (impl 3), n=200, d=128, density 0.8,
1024 W-rand states; CUDA-event medians.  usage: python tools/wide_tc_ab.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2407_11388_b200 import rac  # noqa: E402

n, d, S = int(os.environ.get("AB_N", 200)), 128, int(os.environ.get("AB_S", 1024))
ctx = rac.RacContext.create_random(n, d, synth.quant_density(0.8), synth.quant_tightness(0.95), 1)
states = np.stack([synth.w_rand_wide(np.full(n, d), 0.8, seed=s) for s in range(S)])
din = torch.from_numpy(states.view(np.int64).copy()).cuda()
outs = {}
for impl in (2, 3, 4):
    dout = torch.zeros_like(din)
    for _ in range(3):
        ctx.batch_pass_eval(impl, S, din, dout)
    torch.cuda.synchronize()
    ms = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ctx.batch_pass_eval(impl, S, din, dout)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    outs[impl] = dout.cpu().numpy()
    tests = n * d * (n - 1) * 0.8 * S  # (x,a,y,state) support tests of one full pass
    flops = 2.0 * n * d * n * 128 * S  # the dense MMA work of impl 3 (every column, K = 128)
    med = float(np.median(ms))
    print(json.dumps({"impl": impl, "name": {2: "bit-sliced", 3: "tcgen05 f16", 4: "tcgen05 fp8"}[impl], "n": n, "d": d, "S": S,
                      "ms": round(med, 4), "T_tests_per_s": round(tests / med / 1e9, 3),
                      "mma_TFLOPs_if_tc": round(flops / med / 1e9, 1)}), flush=True)
print(json.dumps({"same_result": bool(np.array_equal(outs[2], outs[3]) and np.array_equal(outs[2], outs[4]))}))
# the product batched enforcement on the same states (wide_state, one block per
# state, every pass to each state's own fixpoint), for scale
dout = torch.zeros_like(din)
its = torch.zeros(S, dtype=torch.int32, device="cuda")
sts = torch.zeros(S, dtype=torch.int32, device="cuda")
for _ in range(2):
    ctx.enforce_batch(S, din, dout, its, sts)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    ctx.enforce_batch(S, din, dout, its, sts)
b.record()
torch.cuda.synchronize()
print(json.dumps({"wide_state_enforcement_ms": round(a.elapsed_time(b) / 3, 4),
                  "mean_iterations": float(its.float().mean().item()), "max_iterations": int(its.max().item())}))
