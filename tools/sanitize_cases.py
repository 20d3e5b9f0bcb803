"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck) over every enforcement kernel, each checked against the CPU oracle:

  fused   -- multi-CTA rac_fused (C2 shape n=500 d=20 t=0.3: root, seeded, W-rand,
             full mode) and a small C3-shaped propagating instance (n=600 d=32)
  sparse  -- rac_fused<W,0> over the sparse arc-block layout (density 0.25)
  vshard  -- rac_pass + rac_shard_{init,seed,slice,update,finalize} (3 row blocks)
  wide    -- wide_fused (d=128, propagating), wide_state (batched), wide_bs_pass / wide_tc_pass
             (tcgen05), the wide search
  state   -- rac_state (one block per state) on single instances up to C2 size
  batch   -- rac_batch_cl (clusters), rac_batch_bs and rac_state on 64 W-dive states, and C1
             (one warp: rac_tiny)
  peer    -- one rank of a 2-process RAC_OPT_PEER group (run under torchrun)

Exit status 0 iff every result equals the oracle's.
usage: python tools/sanitize_cases.py CASE
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2407_11388_b200 import rac  # noqa: E402


def same(g, o, what):
    ok = g[0] == o[0] and g[2] == o[2] and np.array_equal(np.asarray(g[1]).reshape(-1), np.asarray(o[1]).reshape(-1))
    if len(g) > 3 and g[3] is not None and o[3] is not None:
        ok = ok and np.array_equal(np.asarray(g[3]), np.asarray(o[3]))
    print(what, "OK" if ok else "MISMATCH", (g[0], g[2]), (o[0], o[2]), flush=True)
    return ok


def gen_case(n, d, p, t, seed, **kw):
    dq, tq = synth.quant_density(p), synth.quant_tightness(t)
    return rac.RacContext.create_random(n, d, dq, tq, seed, **kw), oracle.Oracle.from_synth(n, d, dq, tq, seed)


def run_common(ctx, orc, n, d, tag):
    ok = True
    root = synth.full_domains(np.full(n, d))
    o = orc.rac(root)
    ok &= same(ctx.enforce(root, removed_at=True), o, tag + " root")
    if o[0] == oracle.OK:
        ds, x, _ = synth.w_seed(o[1], 5)
        ok &= same(ctx.enforce_seeded(ds, [x]), orc.rac(ds, with_epochs=False), tag + " seeded")
        ok &= same(ctx.enforce_seeded(ds, []), (0 if all(int(v) for v in ds) else 1, ds, 0), tag + " seeded-empty")
    dr = synth.w_rand(np.full(n, d), 0.9, 3)
    ok &= same(ctx.enforce(dr, removed_at=True), orc.rac(dr), tag + " rand")
    ok &= same(ctx.enforce(dr, full=True, removed_at=True), orc.rac(dr, full=True), tag + " rand-full")
    return ok


def main(case):
    import torch
    torch.cuda.set_device(0)
    ok = True
    if case == "fused":
        for (n, d, p, t) in ((500, 20, 1.0, 0.3), (600, 32, 1.0, 0.66)):
            ctx, orc = gen_case(n, d, p, t, 1)
            ok &= run_common(ctx, orc, n, d, "fused n=%d" % n)
        # many passes (the rotating per-pass buffers, hundreds of grid barriers):
        # an equality chain inside a complete graph takes exactly n passes
        from tests import _instances as I
        inst = I.equality_chain(300, 8, embed_complete=True)
        ctx, orc = rac.RacContext.from_instance(inst), oracle.Oracle.from_instance(inst)
        assert ctx.path == "fused"
        d_in = inst.full_domains()
        d_in[0] = np.uint64(1)
        ok &= same(ctx.enforce(d_in, removed_at=True), orc.rac(d_in), "fused chain n=300")
    elif case == "state":
        # the one-block kernel (rac_state) on instances beyond its default size
        os.environ["RAC_SMALL_BYTES"] = "1e12"
        for (n, d, p, t) in ((500, 20, 1.0, 0.3), (150, 7, 0.6, 0.5)):
            ctx, orc = gen_case(n, d, p, t, 1)
            assert ctx.path == "one_block"
            ok &= run_common(ctx, orc, n, d, "state n=%d" % n)
    elif case == "sparse":
        ctx, orc = gen_case(800, 32, 0.25, 0.6, 2, layout="sparse")
        assert ctx.layout == "sparse"
        ok &= run_common(ctx, orc, 800, 32, "sparse")
    elif case == "vshard":
        ctx, orc = gen_case(500, 20, 1.0, 0.3, 1, virtual_shards=3)
        ok &= run_common(ctx, orc, 500, 20, "vshard")
    elif case == "wide":
        n, d = 200, 128
        dq, tq = synth.quant_density(1.0), synth.quant_tightness(0.93)
        ctx = rac.RacContext.create_random(n, d, dq, tq, 1)
        wo = oracle.WideOracle.from_synth(n, d, dq, tq, 1)
        full = synth.full_domains_wide(np.full(n, d))
        o = wo.rac(full)
        g = ctx.enforce(full, removed_at=True)
        ok &= same(g, o, "wide root")
        dr = synth.w_rand_wide(np.full(n, d), 0.9, 3)
        ok &= same(ctx.enforce(dr, removed_at=True), wo.rac(dr), "wide rand")
        # batched (wide_state) and the batched-pass A/B kernels (bit-sliced, tcgen05)
        S = 40
        states = np.stack([synth.w_rand_wide(np.full(n, d), 0.8, seed=100 + k) for k in range(S)])
        din = torch.from_numpy(states.view(np.int64).copy()).cuda()
        dout = torch.zeros_like(din)
        its = torch.zeros(S, dtype=torch.int32, device="cuda")
        sts = torch.zeros(S, dtype=torch.int32, device="cuda")
        ctx.enforce_batch(S, din, dout, its, sts)
        torch.cuda.synchronize()
        out = dout.cpu().numpy().view(np.uint64)
        for k in range(S):
            o = wo.rac(states[k], with_epochs=False)
            ok &= (int(sts[k]), int(its[k])) == (o[0], o[2]) and np.array_equal(out[k], o[1])
        print("wide batched", "OK" if ok else "MISMATCH", flush=True)
        from tests import _wide as WD
        for impl in (2, 3):
            ctx.batch_pass_eval(impl, S, din, dout)
            torch.cuda.synchronize()
            out = dout.cpu().numpy().view(np.uint64)
            for k in range(S):
                _, _, _, rem = wo.rac(states[k])
                ok &= np.array_equal(out[k], WD.words_of(WD.bits_of(states[k], n, wo.wq) & (rem != 1)))
            print("wide pass impl %d" % impl, "OK" if ok else "MISMATCH", flush=True)
        r, sol, st = ctx.search(full, max_assignments=200)
        ro, solo, sto = wo.search(full, max_assignments=200)
        ok &= all(st[k] == sto[k] for k in ("assignments", "recurrences", "wipeouts", "solutions"))
        print("wide search", "OK" if ok else "MISMATCH", flush=True)
    elif case == "batch":
        n, d, S = 200, 16, 64
        inst = synth.random_csp(n, d, 0.8, 0.3, 1)
        orc = oracle.Oracle.from_instance(inst)
        _, root, _, _ = orc.rac(inst.full_domains())
        states, svars = synth.dive_states(root, lambda D: orc.rac(D, with_epochs=False)[:2], S, seed=1,
                                          return_seeds=True)
        states = np.stack(states)
        ctx = rac.RacContext.from_instance(inst)
        din = torch.from_numpy(states.view(np.int64).copy()).cuda()
        dout = torch.zeros_like(din)
        its = torch.zeros(S, dtype=torch.int32, device="cuda")
        sts = torch.zeros(S, dtype=torch.int32, device="cuda")
        sv = torch.from_numpy(np.asarray(svars, dtype=np.int32)).cuda()
        for impl, seeded in (("cluster", False), ("cluster", True), ("bs", False), ("bs", True), ("state", True)):
            if impl in ("bs", "state"):
                os.environ["RAC_BATCH_IMPL"] = impl
            if seeded:
                ctx.enforce_batch_seeded(S, din, dout, its, sts, sv)
            else:
                ctx.enforce_batch(S, din, dout, its, sts)
            torch.cuda.synchronize()
            out = dout.cpu().numpy().view(np.uint64)
            for s in range(S):
                o = orc.rac(states[s], with_epochs=False)
                ok &= (int(sts[s]), int(its[s])) == (o[0], o[2]) and np.array_equal(out[s], o[1])
            print("batch %s seeded=%s" % (impl, seeded), "OK" if ok else "MISMATCH", flush=True)
        os.environ.pop("RAC_BATCH_IMPL", None)
        c1 = synth.random_csp(20, 8, 0.5, 0.4, 1)
        ctx1, orc1 = rac.RacContext.from_instance(c1), oracle.Oracle.from_instance(c1)
        ok &= same(ctx1.enforce(c1.full_domains(), removed_at=True), orc1.rac(c1.full_domains()), "single-cta C1")
    elif case == "peer":
        import torch.distributed as dist
        from paper_2407_11388_b200 import dist as rdist
        os.environ.setdefault("RAC_PEER_TIMEOUT_MS", "120000")
        dist.init_process_group("gloo")
        rank, world = dist.get_rank(), dist.get_world_size()
        n, d, p, t = 300, 16, 0.5, 0.5
        dq, tq = synth.quant_density(p), synth.quant_tightness(t)
        ctx = rac.RacContext.create_random(n, d, dq, tq, 3, device=0, rank=rank, world=world, peer=True, max_ctas=8)
        rdist.connect_peers(ctx)
        orc = oracle.Oracle.from_synth(n, d, dq, tq, 3)
        for k in range(2):
            dr = synth.w_rand(np.full(n, d), 0.9, 10 + k)
            ok &= same(ctx.enforce(dr), orc.rac(dr, with_epochs=False), "peer rank %d k=%d" % (rank, k))
        dist.barrier()
        ctx.close()
        dist.destroy_process_group()
    else:
        raise SystemExit("unknown case " + case)
    print("CASE", case, "PASS" if ok else "FAIL", flush=True)
    return 0 if ok else 3


if __name__ == "__main__":
    sys.exit(main(sys.argv[1]))
