"""Debug helper: the nonuniform wide instance #5 of tests/test_gpu_wide.py, GPU vs oracle, listing differences."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
if "--torch" in sys.argv:
    import torch
    assert torch.cuda.is_available()
import oracle  # noqa: E402
import synth  # noqa: E402
from tests import _wide as WD  # noqa: E402
from paper_2407_11388_b200 import rac  # noqa: E402

if "--corpus-first" in sys.argv:
    from tests.test_oracle import _wide_corpus
    for j, inst in enumerate(_wide_corpus(40, 91)):
        c = rac.RacContext.from_instance(inst)
        c.enforce(synth.full_domains_wide(inst.dom), removed_at=True)
        del c
rng = np.random.default_rng(5)
for i in range(12):
    n = int(rng.integers(3, 40))
    dom = rng.integers(1, 257, size=n)
    dom[int(rng.integers(n))] = int(rng.integers(65, 257))
    cons = []
    for x in range(n):
        for y in range(x + 1, n):
            if rng.random() < 0.5:
                p = min(1.0, 3.0 / max(1, int(dom[y])))
                allowed = [(a, b) for a in range(int(dom[x])) for b in np.nonzero(rng.random(int(dom[y])) < p)[0]]
                cons.append((x, y, allowed))
    inst = synth.wide_from_constraints(n, dom.astype(np.int32), cons)
    mc = int([a for a in sys.argv if a.startswith('--max-ctas=')][0].split('=')[1]) if any(a.startswith('--max-ctas=') for a in sys.argv) else 0
    ctx = rac.RacContext.from_instance(inst, max_ctas=mc)
    wo = oracle.WideOracle.from_instance(inst)
    if "--dump" in sys.argv and i in (5, 8):
        import ctypes
        dmax, WS = int(dom.max()), (2 if int(dom.max()) <= 128 else 4)
        wq = wo.wq
        Mg = np.zeros(n * dmax * n * WS, dtype=np.uint64)
        pw = (n + 31) // 32
        Pg = np.zeros(n * pw, dtype=np.uint32)
        f = rac.lib.rac_debug_wide_dump
        f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        assert f(ctx._h, Mg.ctypes.data, Pg.ctypes.data) == 0
        M = np.full(n * dmax * n * WS, np.uint64(2**64 - 1), dtype=np.uint64)
        P = np.zeros(n * pw, dtype=np.uint32)
        rows = np.asarray(inst.rows)
        for r in range(inst.n_rel):
            x, y = int(inst.xs[r]), int(inst.ys[r])
            dx, dy = int(dom[x]), int(dom[y])
            for a in range(dx):
                for w in range(WS):
                    M[((x * dmax + a) * n + y) * WS + w] = rows[r, a, w] if w < wq else 0
            for b in range(dy):
                for w in range(WS):
                    v = 0
                    for k in range(64):
                        a = 64 * w + k
                        if a < dx and (int(rows[r, a, b >> 6]) >> (b & 63)) & 1:
                            v |= 1 << k
                    M[((y * dmax + b) * n + x) * WS + w] = v
            P[x * pw + (y >> 5)] |= np.uint32(1 << (y & 31))
            P[y * pw + (x >> 5)] |= np.uint32(1 << (x & 31))
        bad = np.nonzero(Mg != M)[0]
        print("inst", i, "M mismatches", bad.size, "P mismatches", int((Pg != P).sum()))
        if bad.size:
            idx = bad[:8]
            print("  first", [(int(j // WS // n // dmax), int(j // WS // n % dmax), int(j // WS % n), int(j % WS)) for j in idx],
                  [hex(int(v)) for v in Mg[idx]], [hex(int(v)) for v in M[idx]])
    for name, d_in in (("full", synth.full_domains_wide(inst.dom)), ("rand", synth.w_rand_wide(inst.dom, 0.7, seed=i))):
        for full in (False, True):
            for rep in range(3):
                g = ctx.enforce(d_in, full=full, removed_at=True)
                o = wo.rac(d_in, full=full)
                gb, ob = WD.bits_of(g[1], n, wo.wq), WD.bits_of(o[1], n, wo.wq)
                diff = np.argwhere(gb != ob)
                if len(diff) or g[0] != o[0] or g[2] != o[2]:
                    print("inst", i, "n", n, "dmax", int(dom.max()), name, "full", full, "rep", rep, "st", g[0], o[0],
                          "it", g[2], o[2], "diff", diff[:10].tolist(), "gpu", gb[diff[:, 0], diff[:, 1]][:10].tolist())
print("done")
