"""Per-word pass timeline of the cluster batch kernel rac_batch_cl at C5
(RAC_DEBUG_TIMELINE=1): for every cluster (one 32-state word), %globaltimer at
word start, after staging, and per pass after [prep (column list + tables),
sweep, push (split-barrier wait + DSMEM stores), full cluster barrier, loop
control]."""
import ctypes
import json
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
T = np.frombuffer(buf, dtype=np.uint64)[:k].reshape(-1, 256).astype(np.int64)
t0 = T[:, 0][T[:, 0] > 0].min()
iters = its.cpu().numpy().reshape(-1, 32)
words = []
for g in range(T.shape[0]):
    row = T[g]
    m = int((row > 0).sum())
    if m < 3:
        continue
    P = (m - 3) // 5
    ph = np.diff(row[:m])
    passes = ph[1:1 + 5 * P].reshape(P, 5) if P else np.zeros((0, 5))
    words.append({"g": g, "start": int(row[0] - t0), "end": int(row[m - 1] - t0), "stage": int(ph[0]),
                  "passes": P, "per_pass": passes.tolist(), "max_iters": int(iters[g].max())})
words.sort(key=lambda w: w["end"])
ends = [w["end"] for w in words]
print("words", len(words), "end ns min/median/max:", min(ends), int(np.median(ends)), max(ends))
print("start offset spread ns:", max(w["start"] for w in words))
print("passes histogram (words):", np.bincount([w["passes"] for w in words]).tolist())
print("state iterations histogram:", np.bincount(its.cpu().numpy()).tolist())
for w in words[-3:]:
    print("slow word g=%d passes=%d end=%d stage=%d" % (w["g"], w["passes"], w["end"], w["stage"]))
    for i, pp in enumerate(w["per_pass"]):
        print("   pass %2d  prep %5d sweep %6d push %5d sync %5d control %5d" % (i + 1, *pp))
allp = [pp for w in words for pp in w["per_pass"]]
print("phase totals over all passes of all words (ns): list %d tables %d sweep %d A %d B %d" %
      tuple(np.sum(allp, axis=0)))
json.dump(words, open("gpurun_out/batch_cl_timeline.json", "w"))
