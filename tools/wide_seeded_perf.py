"""Wide-domain seeded enforcement (NEXT-4 + NEXT-1) on one GPU: the paper's
per-assignment call tensorAC(Vars, [x]) after x := a on the root D_ac,
against the full enforcement of the same assigned state.  CUDA-event medians on
the launching stream; checks seeded == full (status, iterations, D_out; Prop. 2)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2407_11388_b200 import rac  # noqa: E402

dev = torch.device("cuda", 0)
for n, d, t in [(2000, 128, 0.9), (2000, 128, 0.92), (1000, 256, 0.95), (1000, 256, 0.96)]:
    ctx = rac.RacContext.create_random(n, d, synth.quant_density(1.0), synth.quant_tightness(t), 1)
    wq = ctx.wq
    full = synth.full_domains_wide(np.full(n, d))
    st, dac, it0 = ctx.enforce(full)[:3]
    if st != rac.RAC_OK:
        print(json.dumps({"n": n, "d": d, "t": t, "root_status": int(st)}), flush=True)
        continue
    rng = np.random.default_rng(0)
    D = dac.reshape(n, wq).copy()
    x = int(rng.integers(n))
    live = [a for a in range(d) if (int(D[x, a >> 6]) >> (a & 63)) & 1]
    a = live[len(live) // 2]
    D[x, :] = 0
    D[x, a >> 6] = np.uint64(1) << np.uint64(a & 63)
    din = torch.from_numpy(D.reshape(-1).view(np.int64).copy()).to(dev)
    seeds = torch.tensor([x], dtype=torch.int32, device=dev)
    res = {}
    for mode in ("seeded", "full"):
        dout = torch.zeros_like(din)
        its = torch.zeros(1, dtype=torch.int32, device=dev)
        sts = torch.zeros(1, dtype=torch.int32, device=dev)
        s = torch.cuda.current_stream()

        def call():
            if mode == "seeded":
                ctx.enforce_seeded_async(din, dout, its, sts, seeds, 1, stream=s)
            else:
                ctx.enforce_async(din, dout, its, sts, stream=s)
        for _ in range(3):
            call()
        ms = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            call()
            e1.record(s)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        res[mode] = (float(np.median(ms)), int(sts.item()), int(its.item()), dout.cpu().numpy().copy())
    same = res["seeded"][1:3] == res["full"][1:3] and np.array_equal(res["seeded"][3], res["full"][3])
    print(json.dumps({"n": n, "d": d, "t": t, "root_iters": int(it0), "x": x, "a": a,
                      "seeded_ms": round(res["seeded"][0], 4), "full_ms": round(res["full"][0], 4),
                      "status": res["seeded"][1], "iters": res["seeded"][2], "seeded_equals_full": bool(same)}),
          flush=True)
    del ctx
    torch.cuda.empty_cache()
