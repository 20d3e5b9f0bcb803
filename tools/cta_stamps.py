"""Per-CTA start / first-barrier / end stamps of the fused kernel (C3 W-stream; --seed: the seeded
C3 call, W-seed)."""
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
lib.rac_debug_cta_stamps.restype = ctypes.c_int
lib.rac_debug_cta_stamps.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
for (n, d, t) in [(2000, 32, 0.5), (8000, 64, 0.5)] if "--c4" in sys.argv else [(2000, 32, 0.5)]:
    ctx = rac.RacContext.create_random(n, d, synth.quant_density(1.0), synth.quant_tightness(t), 1)
    full = synth.full_domains(np.full(n, d))
    sx = None
    if "--seed" in sys.argv:
        _, root, _ = ctx.enforce(full)
        full, sx, _ = synth.w_seed(root, 1)
    din = torch.from_numpy(full.view(np.int64).copy()).cuda()
    dout = torch.zeros_like(din)
    it = torch.zeros(1, dtype=torch.int32, device='cuda')
    st = torch.zeros(1, dtype=torch.int32, device='cuda')
    sv = torch.tensor([sx or 0], dtype=torch.int32, device='cuda')
    call = (lambda: ctx.enforce_seeded_async(din, dout, it, st, sv, 1)) if sx is not None else \
        (lambda: ctx.enforce_async(din, dout, it, st))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(20):
        call()
    torch.cuda.synchronize()
    e0.record()
    call()
    e1.record()
    torch.cuda.synchronize()
    buf = (ctypes.c_uint64 * 3000)()
    k = lib.rac_debug_cta_stamps(ctx._h, buf, 3000)
    T = np.frombuffer(buf, dtype=np.uint64)[:k].reshape(-1, 3).astype(np.int64)
    t0 = T[:, 0].min()
    s, b, e = T[:, 0] - t0, T[:, 1] - t0, T[:, 2] - t0
    slow = np.argsort(b)[-8:]
    print("slowest first-barrier arrivals (cta, start, arrival):", [(int(i), int(s[i]), int(b[i])) for i in slow])
    print(f"n={n}: event {e0.elapsed_time(e1)*1e3:.1f} us; ctas {len(T)}; start spread {s.max()} ns; "
          f"barrier arrival min/median/max {b.min()}/{int(np.median(b))}/{b.max()} ns; end min/max {e.min()}/{e.max()} ns")
