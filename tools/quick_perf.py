"""Quick device-time probe of the enforcement on a few workloads (not the bench)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import synth  # noqa: E402
from paper_2407_11388_b200 import rac  # noqa: E402


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def single(n, d, p, t, kind="root", reps=50, vs=0):
    t0 = time.time()
    ctx = rac.RacContext.create_random(n, d, synth.quant_density(p), synth.quant_tightness(t), 1, virtual_shards=vs)
    torch.cuda.synchronize()
    tg = time.time() - t0
    full = synth.full_domains(np.full(n, d))
    d_in = full
    if kind == "seed":
        st, root, _ = ctx.enforce(full)
        d_in, _, _ = synth.w_seed(root, 1)
    din = torch.from_numpy(d_in.view(np.int64).copy()).cuda()
    dout = torch.zeros_like(din)
    it = torch.zeros(1, dtype=torch.int32, device='cuda')
    st = torch.zeros(1, dtype=torch.int32, device='cuda')
    ms = timeit(lambda: ctx.enforce_async(din, dout, it, st), reps)
    print(f"n={n} d={d} p={p} t={t} {kind} vs={vs} gen={tg:.2f}s iters={it.item()} status={st.item()} "
          f"ms/enf={ms:.4f} launches={ctx.last_launch_count} pass1 GB/s={n*d*(n-1)*p*d/8/ms/1e6:.0f}", flush=True)


def batch(S=1024):
    n, d = 200, 16
    ctx = rac.RacContext.create_random(n, d, synth.quant_density(0.8), synth.quant_tightness(0.3), 1)
    full = synth.full_domains(np.full(n, d))
    _, root, _ = ctx.enforce(full)
    states = np.stack(synth.dive_states(root, lambda D: ctx.enforce(D)[:2], S, seed=1))
    din = torch.from_numpy(states.view(np.int64)).cuda()
    dout = torch.zeros_like(din)
    its = torch.zeros(S, dtype=torch.int32, device='cuda')
    sts = torch.zeros(S, dtype=torch.int32, device='cuda')
    ms = timeit(lambda: ctx.enforce_batch(S, din, dout, its, sts), 20)
    print(f"C5 batch S={S} ms/batch={ms:.4f} states/s={S/ms*1e3:.0f} mean iters={its.float().mean().item():.2f}",
          flush=True)


if __name__ == "__main__":
    single(2000, 32, 1.0, 0.5)
    single(2000, 32, 1.0, 0.70, reps=20)
    single(2000, 32, 1.0, 0.70, reps=10, vs=4)
    single(2000, 32, 1.0, 0.5, kind="seed")
    single(500, 20, 1.0, 0.3, reps=200)
    single(20, 8, 0.5, 0.4, kind="seed", reps=500)
    batch()
