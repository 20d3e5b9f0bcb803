"""Per-word pass timeline of the bit-sliced batched kernel (RAC_DEBUG_TIMELINE=1)."""
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
lib.rac_debug_batch_timeline.restype = ctypes.c_int
lib.rac_debug_batch_timeline.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
n, d, S = 200, 16, 1024
ctx = rac.RacContext.create_random(n, d, synth.quant_density(0.8), synth.quant_tightness(0.3), 1)
_, root, _ = ctx.enforce(synth.full_domains(np.full(n, d)))
states, seeds = synth.dive_states(root, lambda D: ctx.enforce(D)[:2], S, seed=1, return_seeds=True)
din = torch.from_numpy(np.stack(states).view(np.int64)).cuda()
dout = torch.zeros_like(din)
its = torch.zeros(S, dtype=torch.int32, device='cuda')
sts = torch.zeros(S, dtype=torch.int32, device='cuda')
sv = torch.from_numpy(np.asarray(seeds, dtype=np.int32)).cuda()
for _ in range(5):
    ctx.enforce_batch_seeded(S, din, dout, its, sts, sv)
torch.cuda.synchronize()
buf = (ctypes.c_uint64 * (4096 * 64))()
k = lib.rac_debug_batch_timeline(ctx._h, buf, 4096 * 64)
T = np.frombuffer(buf, dtype=np.uint64)[:k].reshape(-1, 64).astype(np.int64)
t0 = T[:, 0][T[:, 0] > 0].min()
ends = []
for c in range(T.shape[0]):
    row = T[c]
    passes = int((row[1:] > 0).sum())
    ends.append((row[passes] - t0 if passes else 0, c, passes))
ends.sort()
print("ctas", T.shape[0], "first start offset spread (ns):", int(T[:, 0].max() - t0))
print("slowest CTAs (end ns, cta, passes):", ends[-5:])
c = ends[-1][1]
row = T[c]
p = int((row[1:] > 0).sum())
print("slowest CTA per-pass ns:", [int(row[i] - row[i - 1]) for i in range(1, p + 1)])
print("pass count histogram:", np.bincount([e[2] for e in ends]).tolist())
print("iterations of states:", np.bincount(its.cpu().numpy()).tolist())
