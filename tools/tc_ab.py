"""A/B of the batched contraction: one full Eq. 1 pass (all 200 columns) for 1024 C5 dive
states, bit-sliced ALU (impl 0) vs tcgen05 tensor cores (impl 1); CUDA-event time per pass."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import synth  # noqa: E402
from paper_2407_11388_b200 import rac  # noqa: E402

n, d, S = 200, 16, 1024
ctx = rac.RacContext.create_random(n, d, synth.quant_density(0.8), synth.quant_tightness(0.3), 1)
_, root, _ = ctx.enforce(synth.full_domains(np.full(n, d)))
states = np.stack(synth.dive_states(root, lambda D: ctx.enforce(D)[:2], S, seed=1))
din = torch.from_numpy(states.view(np.int64)).cuda()
outs = {}
for impl in (0, 1):
    dout = torch.zeros_like(din)
    for _ in range(5):
        ctx.batch_pass_eval(impl, S, din, dout)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        ctx.batch_pass_eval(impl, S, din, dout)
    e1.record()
    torch.cuda.synchronize()
    outs[impl] = dout.cpu().numpy()
    print(f"impl {impl} ({'bit-sliced ALU' if impl == 0 else 'tcgen05 f16'}): {e0.elapsed_time(e1) / 50 * 1e3:.1f} us per full pass "
          f"(incl. transpose in/out), S={S}, n={n}, d={d}", flush=True)
print("outputs identical:", bool(np.array_equal(outs[0], outs[1])))
