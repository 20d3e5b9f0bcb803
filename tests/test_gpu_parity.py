"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Everything integer: the bar is bit-exact equality of
status, D_out, iteration count and (where requested) the per-value removal
epochs.  Expected values come only from oracle/ (never from the CUDA path).

Configs C1..C5 are BASELINE.json configs[0..4]; workloads W-root / W-seed /
W-rand / W-stream / W-prop / W-dive are defined in DESIGN.md "Input recipe".
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from tests import _instances as I

pytestmark = pytest.mark.gpu

U64 = np.uint64


@pytest.fixture(scope="module")
def rac():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2407_11388_b200 import rac as r
    return r


def assert_same(g, o, what=""):
    """g = (status, d_out, iters[, removed_at]) from the GPU, o from the oracle."""
    assert g[0] == o[0], (what, "status", g[0], o[0])
    assert g[2] == o[2], (what, "iterations", g[2], o[2])
    assert np.array_equal(g[1], o[1]), (what, "d_out")
    if len(g) > 3 and len(o) > 3 and o[3] is not None:
        assert np.array_equal(g[3], o[3]), (what, "removed_at")


def both(ctx, orc, d_in, full=False):
    g = ctx.enforce(d_in, full=full, removed_at=True)
    o = orc.rac(d_in, full=full)
    return g, o


# ----------------------------------------------------------------------------- hand traces
@pytest.mark.parametrize("name", I.golden_names())
def test_golden(rac, name):
    doc, inst = I.load_golden(name)
    exp = doc["expect"]
    ctx = rac.RacContext.from_instance(inst)
    st, d_out, it, rem = ctx.enforce(np.asarray(doc["d_in"], dtype=U64), removed_at=True)
    assert st == (rac.RAC_OK if exp["status"] == "OK" else rac.RAC_WIPEOUT)
    assert [int(v) for v in d_out] == exp["d_out"] and it == exp["iterations"]
    trace = [set() for _ in range(it)]
    for x in range(inst.n):
        for a in range(64):
            if rem[x, a]:
                trace[rem[x, a] - 1].add((x, a))
    assert trace == [set(map(tuple, s)) for s in exp["trace"]]


# ----------------------------------------------------------------------------- packer
@pytest.mark.parametrize("n,d,p,t", [(9, 3, 0.5, 0.3), (33, 8, 0.7, 0.4), (70, 17, 0.3, 0.5), (40, 64, 0.9, 0.6),
                                     (17, 1, 1.0, 0.2)])
def test_packer_matches_oracle_layout(rac, n, d, p, t):
    """Packed masks M[x][a][·] and presence bits equal the oracle's support sets
    c_xy|(x,a) (both orientations), for host-packed (N1) and device-generated (N7)
    instances of the same seed."""
    inst = synth.random_csp(n, d, p, t, seed=5)
    orc = oracle.Oracle.from_instance(inst)
    for ctx in (rac.RacContext.from_instance(inst),
                rac.RacContext.create_random(n, d, synth.quant_density(p), synth.quant_tightness(t), 5)):
        allones = U64((1 << (8 * ctx.mask_bytes)) - 1)
        for x in range(n):
            for a in range(d):
                masks, pres = ctx.read_row(x, a)
                for y in range(n):
                    present, s = orc.support(x, y, a)
                    assert bool(pres[y]) == present
                    if present:
                        assert int(masks[y]) == s, (x, a, y)
                    else:
                        assert masks[y] == allones


# ----------------------------------------------------------------------------- corpora
@pytest.mark.parametrize("path", ["one-warp", "one-block", "fused"])
def test_spec_corpus(rac, path, monkeypatch):
    """SPEC.md acceptance corpus shape: 1000 instances, n 2..20, d 1..6,
    density 0.1..1, tightness 0..0.9; W-root and W-rand; stop and full modes --
    through the one-warp kernel (rac_tiny, the default for n <= 64), the
    one-block kernel (rac_state, RAC_NO_TINY=1) and the cooperative rac_fused
    kernel (RAC_SMALL_BYTES=0)."""
    if path == "fused":
        monkeypatch.setenv("RAC_SMALL_BYTES", "0")
    if path == "one-block":
        monkeypatch.setenv("RAC_NO_TINY", "1")
    for k, inst in enumerate(I.random_corpus(1000)):
        ctx = rac.RacContext.from_instance(inst)
        orc = oracle.Oracle.from_instance(inst)
        d_in = inst.full_domains() if k % 2 == 0 else synth.w_rand(inst.dom, 0.9, seed=k)
        for full in (False, True):
            g, o = both(ctx, orc, d_in, full)
            assert_same(g, o, (k, full))


def test_nonuniform_domains_and_empty_rows(rac):
    """Per-variable domain sizes (padded to the max) and empty rows in D_in
    (reading R7: one pass, presence semantics, then WIPEOUT)."""
    rng = np.random.default_rng(3)
    for k in range(200):
        n = int(rng.integers(2, 14))
        dom = rng.integers(1, 9, size=n)
        cons = []
        for x in range(n):
            for y in range(x + 1, n):
                if rng.random() < 0.5:
                    allowed = [(a, b) for a in range(dom[x]) for b in range(dom[y]) if rng.random() > 0.35]
                    cons.append((x, y, allowed))
        inst = synth.from_constraints(n, dom, cons)
        ctx = rac.RacContext.from_instance(inst)
        orc = oracle.Oracle.from_instance(inst)
        d_in = synth.w_rand(inst.dom, 0.85, seed=k)
        if k % 3 == 0:
            d_in[int(rng.integers(n))] = U64(0)
        for full in (False, True):
            g, o = both(ctx, orc, d_in, full)
            assert_same(g, o, (k, full))


@pytest.mark.parametrize("d", [8, 16, 32, 64])
def test_equality_chain_many_passes(rac, d):
    """Closed form (equality chain embedded in a complete graph): exactly n passes;
    exercises the device-side loop and grid barrier over hundreds of passes."""
    n = 300
    inst = I.equality_chain(n, d, embed_complete=True)
    ctx = rac.RacContext.from_instance(inst)
    d_in = inst.full_domains()
    d_in[0] = U64(1)
    st, d_out, it = ctx.enforce(d_in)
    assert st == rac.RAC_OK and it == n and np.all(d_out == U64(1))
    st, d_out, it = ctx.enforce(d_in, full=True)
    assert st == rac.RAC_OK and it == n


# ----------------------------------------------------------------------------- C1
def test_c1_many_seeds(rac):
    """C1: n=20, d=8, density 0.5, t=0.4 (BASELINE configs[0]); 300 instance seeds,
    W-root, W-seed and W-rand; full removal-epoch parity."""
    for seed in range(1, 301):
        inst = synth.random_csp(20, 8, 0.5, 0.4, seed)
        ctx = rac.RacContext.from_instance(inst)
        orc = oracle.Oracle.from_instance(inst)
        root = inst.full_domains()
        g, o = both(ctx, orc, root)
        assert_same(g, o, ("root", seed))
        if o[0] == oracle.OK:
            ds, _, _ = synth.w_seed(o[1], seed)
            g, o2 = both(ctx, orc, ds)
            assert_same(g, o2, ("seed", seed))
        g, o = both(ctx, orc, synth.w_rand(inst.dom, 0.9, seed))
        assert_same(g, o, ("rand", seed))


# ----------------------------------------------------------------------------- C2
@pytest.mark.parametrize("t", [0.0119, 0.3])
def test_c2(rac, t):
    """C2: n=500, d=20, complete graph (configs[1]); t at the phase-transition
    estimate and a propagating t=0.3; W-root, W-seed, W-rand."""
    dq, tq = synth.quant_density(1.0), synth.quant_tightness(t)
    ctx = rac.RacContext.create_random(500, 20, dq, tq, 1)
    orc = oracle.Oracle.from_synth(500, 20, dq, tq, 1)
    root = synth.full_domains(np.full(500, 20))
    g, o = both(ctx, orc, root)
    assert_same(g, o, "root")
    if o[0] == oracle.OK:
        for k in range(3):
            ds, _, _ = synth.w_seed(o[1], 11, k)
            g, o2 = both(ctx, orc, ds)
            assert_same(g, o2, ("seed", k))
    g, o = both(ctx, orc, synth.w_rand(np.full(500, 20), 0.9, 2))
    assert_same(g, o, "rand")


# ----------------------------------------------------------------------------- C3
@pytest.mark.parametrize("t,workload", [(0.5, "stream"), (0.70, "prop")])
def test_c3(rac, t, workload):
    """C3: n=2000, d=32, density 1 (configs[2], 512 MB of masks); W-stream (1 pass,
    every byte read) and W-prop (about 10 passes).  Full parity incl. epochs, plus the
    O4 certificate on the GPU's own removal epochs."""
    dq, tq = synth.quant_density(1.0), synth.quant_tightness(t)
    ctx = rac.RacContext.create_random(2000, 32, dq, tq, 1)
    orc = oracle.Oracle.from_synth(2000, 32, dq, tq, 1)
    root = synth.full_domains(np.full(2000, 32))
    g, o = both(ctx, orc, root)
    assert_same(g, o, workload)
    if workload == "stream":
        assert g[2] == 1 and np.array_equal(g[1], root)
    else:
        assert g[2] > 3
    assert orc.certify(root, g[1], g[3], check_ac=(g[0] == rac.RAC_OK)) == 0


def test_c3_virtual_shards(rac):
    """The sharded per-pass path (row blocks, TMA-staged D, gather by device copy)
    at C3 shape (W-prop, 13 passes): every block count's (status, D_out, iterations,
    removal epochs) is certified by the oracle's exact-trajectory certificate O7
    (the recurrence's own output, pass by pass), and equals the fused path's."""
    dq, tq = synth.quant_density(1.0), synth.quant_tightness(0.70)
    ref = rac.RacContext.create_random(2000, 32, dq, tq, 1)
    root = synth.full_domains(np.full(2000, 32))
    r0 = ref.enforce(root, removed_at=True)
    for v in (2, 3, 8):
        ctx = rac.RacContext.create_random(2000, 32, dq, tq, 1, virtual_shards=v)
        r = ctx.enforce(root, removed_at=True)
        assert oracle.certify_trajectory_synth(2000, 32, dq, tq, 1, root, r[1], r[3], r[2], r[0]) == 0, v
        assert_same(r, r0, v)


def test_virtual_shards_corpus(rac):
    for k, inst in enumerate(I.random_corpus(200, seed0=31)):
        orc = oracle.Oracle.from_instance(inst)
        d_in = synth.w_rand(inst.dom, 0.9, seed=k)
        ctx = rac.RacContext.from_instance(inst, virtual_shards=1 + k % 5)
        for full in (False, True):
            g, o = both(ctx, orc, d_in, full)
            assert_same(g, o, (k, full))


# ----------------------------------------------------------------------------- C4
def test_c4_sampled(rac):
    """C4 shape on one GPU: n=8000, d=64, density 1 (32.8 GB of masks, generated on
    device).  W-stream (t=0.5): 1 pass, nothing removed.  A W-rand input at t=0.85
    removes about half the rows in pass 1; 200 sampled rows' pass-1 verdicts are
    checked one by one against the oracle computed straight from the generator."""
    import torch
    n, d = 8000, 64
    free, _ = torch.cuda.mem_get_info()
    if free < 36e9:
        pytest.skip("needs ~36 GB free device memory")
    dq = synth.quant_density(1.0)
    ctx = rac.RacContext.create_random(n, d, dq, synth.quant_tightness(0.5), 1)
    root = synth.full_domains(np.full(n, d))
    st, d_out, it = ctx.enforce(root)
    assert st == rac.RAC_OK and it == 1 and np.array_equal(d_out, root)
    rng = np.random.default_rng(1)
    for x, a in zip(rng.integers(0, n, 30), rng.integers(0, d, 30)):
        assert oracle.row_supported_synth(n, d, dq, synth.quant_tightness(0.5), 1, int(x), int(a), root)
    ctx.close()
    del ctx
    tq = synth.quant_tightness(0.85)
    ctx = rac.RacContext.create_random(n, d, dq, tq, 2)
    d_in = synth.w_rand(np.full(n, d), 0.9, 3)
    st, d_out, it, rem = ctx.enforce(d_in, removed_at=True)
    live = [(x, a) for x in range(n) for a in range(d) if (int(d_in[x]) >> a) & 1]
    pick = rng.choice(len(live), 200, replace=False)
    n_removed = 0
    for i in pick:
        x, a = live[i]
        sup = oracle.row_supported_synth(n, d, dq, tq, 2, x, a, d_in)
        assert sup == (rem[x, a] != 1), (x, a)
        n_removed += not sup
    assert 20 < n_removed < 180


# ----------------------------------------------------------------------------- C5 (batched)
def test_c5_batched(rac):
    """C5: 1024 W-dive states on n=200, d=16, density 0.8, t=0.3 (configs[4]).  Each
    state's (status, D_out, iterations) equals the oracle's single-state result; batch
    composition does not matter (a permuted batch gives permuted results)."""
    import torch
    n, d, S = 200, 16, 1024
    inst = synth.random_csp(n, d, 0.8, 0.3, 1)
    orc = oracle.Oracle.from_instance(inst)
    st0, root, _, _ = orc.rac(inst.full_domains())
    assert st0 == oracle.OK

    def enf(D):
        s, out, _, _ = orc.rac(D, with_epochs=False)
        return s, out

    states = np.stack(synth.dive_states(root, enf, S, seed=1))
    expect = [orc.rac(s, with_epochs=False) for s in states]
    ctx = rac.RacContext.from_instance(inst)
    for perm in (np.arange(S), np.random.default_rng(0).permutation(S)):
        din = torch.from_numpy(states[perm].view(np.int64)).cuda()
        dout = torch.zeros_like(din)
        its = torch.zeros(S, dtype=torch.int32, device="cuda")
        sts = torch.zeros(S, dtype=torch.int32, device="cuda")
        ctx.enforce_batch(S, din, dout, its, sts)
        torch.cuda.synchronize()
        out = dout.cpu().numpy().view(np.uint64)
        its, sts = its.cpu().numpy(), sts.cpu().numpy()
        for j, s in enumerate(perm):
            e = expect[s]
            assert (sts[j], its[j]) == (e[0], e[2]), (s, sts[j], its[j], e[0], e[2])
            assert np.array_equal(out[j], e[1]), s
    iters = np.array([e[2] for e in expect])
    assert iters.max() > 3 and any(e[0] == oracle.WIPEOUT for e in expect)


def test_async_api_and_in_place(rac):
    """rac_enforce_async on torch device buffers and a torch stream; d_out == d_in."""
    import torch
    inst = synth.random_csp(150, 12, 0.6, 0.45, 4)
    orc = oracle.Oracle.from_instance(inst)
    ctx = rac.RacContext.from_instance(inst)
    d_in = synth.w_rand(inst.dom, 0.9, 5)
    o = orc.rac(d_in)
    buf = torch.from_numpy(d_in.view(np.int64).copy()).cuda()
    it = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    rem = torch.zeros(150 * 64, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx.enforce_async(buf, buf, it, st, rem, stream=s)
    s.synchronize()
    assert int(st.item()) == o[0] and int(it.item()) == o[2]
    assert np.array_equal(buf.cpu().numpy().view(np.uint64), o[1])
    assert np.array_equal(rem.cpu().numpy().reshape(150, 64), o[3])
    assert ctx.last_launch_count >= 1


def test_input_padding_bits_rejected(rac):
    inst = synth.random_csp(5, 3, 1.0, 0.3, 1)
    ctx = rac.RacContext.from_instance(inst)
    bad = inst.full_domains()
    bad[2] |= U64(1 << 5)
    with pytest.raises(rac.RacError) as ei:
        ctx.enforce(bad)
    assert ei.value.code == rac.RAC_EINVAL
    # the context stays usable after EINVAL
    assert ctx.enforce(inst.full_domains())[0] in (rac.RAC_OK, rac.RAC_WIPEOUT)


# ----------------------------------------------------------------------------- seeded (NEXT-1)
def test_seeded_c1_and_corpus(rac):
    """Seeded enforcement (Alg. 1 tensorAC(Vars, [idx])) on W-seed inputs: equal to
    the oracle's full recurrence O1 and to the literal Alg. 1 O5 (status, D, iterations)."""
    n_checked = 0
    for seed in range(1, 201):
        inst = synth.random_csp(20, 8, 0.5, 0.4, seed) if seed % 2 else \
            I.random_corpus(1, seed0=seed, n_range=(3, 20))[0]
        orc = oracle.Oracle.from_instance(inst)
        st, root, _, _ = orc.rac(inst.full_domains())
        if st != oracle.OK:
            continue
        ctx = rac.RacContext.from_instance(inst)
        for j in range(2):
            s, x, v = synth.w_seed(root, seed, j)
            g = ctx.enforce_seeded(s, [x])
            o = orc.rac(s)
            o5 = orc.rac_seeded(s, [x])
            assert (g[0], g[2]) == (o[0], o[2]) == (o5[0], o5[2]), (seed, j)
            assert np.array_equal(g[1], o[1]) and np.array_equal(g[1], o5[1])
            n_checked += 1
        g = ctx.enforce_seeded(root, [])
        assert g[0] == rac.RAC_OK and g[2] == 0 and np.array_equal(g[1], root)
    assert n_checked > 100


def test_seeded_c3(rac):
    """C3 W-seed (n=2000, d=32, t=0.5): the seeded call reads only the assigned variable's
    masks in pass 1 and equals the oracle's full recurrence."""
    dq, tq = synth.quant_density(1.0), synth.quant_tightness(0.5)
    ctx = rac.RacContext.create_random(2000, 32, dq, tq, 1)
    orc = oracle.Oracle.from_synth(2000, 32, dq, tq, 1)
    root = synth.full_domains(np.full(2000, 32))
    st, droot, _, _ = orc.rac(root)
    assert st == oracle.OK
    for j in range(3):
        s, x, v = synth.w_seed(droot, 5, j)
        g = ctx.enforce_seeded(s, [x])
        o = orc.rac(s, with_epochs=False)
        assert (g[0], g[2]) == (o[0], o[2]) and np.array_equal(g[1], o[1])


def test_c5_batched_seeded(rac):
    """C5 dive states with their assigned variable as the per-state seed: equal to the
    oracle's single-state full recurrence."""
    import torch
    n, d, S = 200, 16, 1024
    inst = synth.random_csp(n, d, 0.8, 0.3, 1)
    orc = oracle.Oracle.from_instance(inst)
    _, root, _, _ = orc.rac(inst.full_domains())

    def enf(D):
        s, out, _, _ = orc.rac(D, with_epochs=False)
        return s, out

    states, seeds = synth.dive_states(root, enf, S, seed=2, return_seeds=True)
    states = np.stack(states)
    seeds = np.asarray(seeds, dtype=np.int32)
    seeds[::7] = -1  # some states as root calls
    ctx = rac.RacContext.from_instance(inst)
    din = torch.from_numpy(states.view(np.int64)).cuda()
    dout = torch.zeros_like(din)
    its = torch.zeros(S, dtype=torch.int32, device="cuda")
    sts = torch.zeros(S, dtype=torch.int32, device="cuda")
    sv = torch.from_numpy(seeds).cuda()
    ctx.enforce_batch_seeded(S, din, dout, its, sts, sv)
    torch.cuda.synchronize()
    out = dout.cpu().numpy().view(np.uint64)
    its, sts = its.cpu().numpy(), sts.cpu().numpy()
    for s in range(S):
        e = orc.rac(states[s], with_epochs=False)
        assert (sts[s], its[s]) == (e[0], e[2]) and np.array_equal(out[s], e[1]), s


# ----------------------------------------------------------------------------- layouts
@pytest.mark.parametrize("layout", ["rows", "cols"])
def test_forced_layouts(rac, layout, monkeypatch):
    """Every pass on the row-major copy only, or on the column-major tensor only
    (RAC_FORCE_LAYOUT), gives the oracle's results: both sweeps are exact."""
    monkeypatch.setenv("RAC_FORCE_LAYOUT", layout)
    monkeypatch.setenv("RAC_SMALL_BYTES", "0")  # tiny instances through rac_fused too (not the one-block path)
    for k, inst in enumerate(I.random_corpus(150, seed0=61)):
        ctx = rac.RacContext.from_instance(inst)
        orc = oracle.Oracle.from_instance(inst)
        d_in = synth.w_rand(inst.dom, 0.9, seed=k)
        if k % 4 == 0:
            d_in[k % inst.n] = U64(0)
        for full in (False, True):
            g, o = both(ctx, orc, d_in, full)
            assert_same(g, o, (layout, k, full))
    dq = synth.quant_density(1.0)
    for t, kind in ((0.70, "root"), (0.5, "seed")):
        tq = synth.quant_tightness(t)
        ctx = rac.RacContext.create_random(2000, 32, dq, tq, 1)
        orc = oracle.Oracle.from_synth(2000, 32, dq, tq, 1)
        root = synth.full_domains(np.full(2000, 32))
        if kind == "root":
            g, o = both(ctx, orc, root)
            assert_same(g, o, (layout, kind))
        else:
            _, droot, _, _ = orc.rac(root, with_epochs=False)
            s, x, v = synth.w_seed(droot, 7)
            g = ctx.enforce_seeded(s, [x])
            o = orc.rac(s, with_epochs=False)
            assert (g[0], g[2]) == (o[0], o[2]) and np.array_equal(g[1], o[1])


@pytest.mark.parametrize("layout", ["auto", "rows"])
def test_back_to_back_launches(rac, layout, monkeypatch):
    """Many enforcements in a row on ONE context with pass counts 1, 2 and 3 mixed:
    the per-pass buffers (removal vector, row-claim counter, removal flag) rotate
    through three copies across launches, so every residue of the global pass
    number mod 3 is exercised; every result keeps full epoch parity.  (A rotation
    bug once left a stale row-claim counter that skipped rows: C2 W-seed.)"""
    if layout != "auto":
        monkeypatch.setenv("RAC_FORCE_LAYOUT", layout)
    dq, tq = synth.quant_density(1.0), synth.quant_tightness(0.0119)
    ctx = rac.RacContext.create_random(500, 20, dq, tq, 1)
    orc = oracle.Oracle.from_synth(500, 20, dq, tq, 1)
    root = synth.full_domains(np.full(500, 20))
    o_root = orc.rac(root)
    inputs = [root] + [synth.w_seed(o_root[1], 11, k)[0] for k in range(3)] + \
        [synth.w_rand(np.full(500, 20), 0.9, 2)]
    expect = [orc.rac(d) for d in inputs]
    assert len({e[2] for e in expect}) >= 2
    order = [0, 1, 1, 2, 4, 1, 3, 3, 0, 2, 2, 4, 4, 1, 0, 3, 2, 1, 4, 0, 3]
    for i, k in enumerate(order):
        assert_same(ctx.enforce(inputs[k], removed_at=True), expect[k], (layout, i, k))


# ----------------------------------------------------------------------------- search (NEXT-2)
def test_search_parity(rac):
    """rac_search (Alg. 2 with seeded enforcement per assignment) explores the
    same tree as the oracle's O6: identical verdict, first solution, assignments, summed
    #Recurrence, wipeouts and depth -- on the tiny corpus (whole trees, all solutions),
    C1 instances and a C5-shaped instance under an assignment budget."""
    keys = ("assignments", "recurrences", "wipeouts", "solutions", "max_depth", "root_iterations")
    cases = [(inst, 0, True) for inst in I.random_corpus(120, seed0=81, n_range=(1, 8), d_range=(1, 4))]
    cases += [(synth.random_csp(20, 8, 0.5, 0.4, s), 3000, False) for s in range(1, 21)]
    cases += [(synth.random_csp(200, 16, 0.8, 0.3, 1), 1500, False), (synth.random_csp(100, 20, 0.25, 0.3, 2), 1500, False)]
    for k, (inst, budget, all_sol) in enumerate(cases):
        orc = oracle.Oracle.from_instance(inst)
        ctx = rac.RacContext.from_instance(inst)
        r_o, sol_o, st_o = orc.search(inst.full_domains(), max_assignments=budget, all_solutions=all_sol)
        r_g, sol_g, st_g = ctx.search(inst.full_domains(), max_assignments=budget, all_solutions=all_sol)
        assert r_g == r_o, (k, r_g, r_o)
        for key in keys:
            assert st_g[key] == st_o[key], (k, key, st_g[key], st_o[key])
        if r_o == 0:
            assert np.array_equal(sol_g, sol_o)


def test_batched_corpus(rac):
    """Batched enforcement (bit-sliced, and the per-state kernel via RAC_BATCH_IMPL=state) on
    random instances with odd row counts and non-uniform domains: every state equals the
    oracle's single-state result; seeded and unseeded; batch sizes not multiples of 32."""
    import os
    import torch
    rng = np.random.default_rng(5)
    for impl in ("bs", "state"):
        if impl == "state":
            os.environ["RAC_BATCH_IMPL"] = "state"
        try:
            for k, inst in enumerate(I.random_corpus(40, seed0=91, n_range=(2, 15), d_range=(1, 7))):
                orc = oracle.Oracle.from_instance(inst)
                S = int(rng.integers(1, 70))
                states = np.stack([synth.w_rand(inst.dom, 0.85, seed=1000 * k + s) for s in range(S)])
                seeds = np.full(S, -1, dtype=np.int32)
                st_root, root, _, _ = orc.rac(inst.full_domains(), with_epochs=False)
                if st_root == oracle.OK:  # some states as assignments on the root fixpoint (seeded)
                    for s in range(0, S, 2):
                        ds, x, v = synth.w_seed(root, k, s)
                        states[s], seeds[s] = ds, x
                ctx = rac.RacContext.from_instance(inst)
                din = torch.from_numpy(states.view(np.int64)).cuda()
                dout = torch.zeros_like(din)
                its = torch.zeros(S, dtype=torch.int32, device="cuda")
                sts = torch.zeros(S, dtype=torch.int32, device="cuda")
                for seeded in (False, True):
                    if seeded:
                        ctx.enforce_batch_seeded(S, din, dout, its, sts, torch.from_numpy(seeds).cuda())
                    else:
                        ctx.enforce_batch(S, din, dout, its, sts)
                    torch.cuda.synchronize()
                    out = dout.cpu().numpy().view(np.uint64)
                    it_h, st_h = its.cpu().numpy(), sts.cpu().numpy()
                    for s in range(S):
                        e = orc.rac(states[s], with_epochs=False)
                        assert (st_h[s], it_h[s]) == (e[0], e[2]) and np.array_equal(out[s], e[1]), (impl, k, s, seeded)
        finally:
            os.environ.pop("RAC_BATCH_IMPL", None)


def test_c5_batched_many_words(rac):
    """More words than co-resident clusters (C5 shape, 5000 states = 157 words, the last one
    partial): every cluster runs several words back to back (per-word re-staging, mbarrier
    phases continuing across words) -- each state equals the oracle's single-state result."""
    import torch
    n, d, S = 200, 16, 5000
    inst = synth.random_csp(n, d, 0.8, 0.3, 1)
    orc = oracle.Oracle.from_instance(inst)
    _, root, _, _ = orc.rac(inst.full_domains(), with_epochs=False)

    def enf(D):
        st, out, _, _ = orc.rac(D, with_epochs=False)
        return st, out

    states, seeds = synth.dive_states(root, enf, S, seed=4, return_seeds=True)
    states = np.stack(states)
    seeds = np.asarray(seeds, dtype=np.int32)
    seeds[::3] = -1
    ctx = rac.RacContext.from_instance(inst)
    din = torch.from_numpy(states.view(np.int64)).cuda()
    dout = torch.zeros_like(din)
    its = torch.zeros(S, dtype=torch.int32, device="cuda")
    sts = torch.zeros(S, dtype=torch.int32, device="cuda")
    ctx.enforce_batch_seeded(S, din, dout, its, sts, torch.from_numpy(seeds).cuda())
    torch.cuda.synchronize()
    out = dout.cpu().numpy().view(np.uint64)
    its, sts = its.cpu().numpy(), sts.cpu().numpy()
    for s in range(S):
        e = orc.rac(states[s], with_epochs=False)
        assert (sts[s], its[s]) == (e[0], e[2]) and np.array_equal(out[s], e[1]), s


@pytest.mark.parametrize("mode", ["default", "per_state", "groups"])
def test_batched_exact_columns(rac, mode, monkeypatch):
    """The cluster batch kernel tests, per state, only the columns that changed for
    that state (Alg. 1's Cons[:, @changed]): C5 dive states seeded with their
    assigned variable (O1, the seeded call's precondition holds), and seeded calls on
    W-rand states, where the precondition does not hold, against O5
    (tensorAC(Vars, @changed = seeds) as written) -- every state follows its own
    Alg. 1 trajectory, not the union of its word's columns; plus a corpus with every
    mask width (d up to 32, W = 1, 2, 4)."""
    import torch
    # sweeps: union columns through chunk tables (per-column masks, or the 8-byte column-group
    # A/B layout), and the per-state sweep for <= 8 active states (auto, or forced)
    monkeypatch.setenv("RAC_CL_GROUPS", "1" if mode == "groups" else "0")
    monkeypatch.setenv("RAC_CL_PS", {"default": "0", "per_state": "2", "union_only": "0", "groups": "0"}[mode])
    groups = mode
    n, d, S = 200, 16, 512
    inst = synth.random_csp(n, d, 0.8, 0.3, 1)
    orc = oracle.Oracle.from_instance(inst)
    _, root, _, _ = orc.rac(inst.full_domains())

    def enf(D):
        s, out, _, _ = orc.rac(D, with_epochs=False)
        return s, out

    states, seeds = synth.dive_states(root, enf, S, seed=3, return_seeds=True)
    states = np.stack(states)
    seeds = np.asarray(seeds, dtype=np.int32)
    seeds[::5] = -1
    # the second half: W-rand states (not arc consistent) with random seed lists of one variable
    rng = np.random.default_rng(11)
    for s in range(S // 2, S):
        states[s] = synth.w_rand(inst.dom, 0.9, seed=500 + s)
        seeds[s] = int(rng.integers(0, n))
    ctx = rac.RacContext.from_instance(inst)
    din = torch.from_numpy(states.view(np.int64)).cuda()
    dout = torch.zeros_like(din)
    its = torch.zeros(S, dtype=torch.int32, device="cuda")
    sts = torch.zeros(S, dtype=torch.int32, device="cuda")
    ctx.enforce_batch_seeded(S, din, dout, its, sts, torch.from_numpy(seeds).cuda())
    torch.cuda.synchronize()
    out = dout.cpu().numpy().view(np.uint64)
    its, sts = its.cpu().numpy(), sts.cpu().numpy()
    for s in range(S):
        if seeds[s] < 0:
            e = orc.rac(states[s], with_epochs=False)
        else:
            e = orc.rac_seeded(states[s], [int(seeds[s])], with_epochs=False)
        assert (sts[s], its[s]) == (e[0], e[2]) and np.array_equal(out[s], e[1]), (s, seeds[s], groups)
    for k, inst in enumerate(I.random_corpus(30, seed0=191, n_range=(2, 40), d_range=(1, 32))):
        orc = oracle.Oracle.from_instance(inst)
        S2 = int(rng.integers(1, 80))
        st2 = np.stack([synth.w_rand(inst.dom, 0.85, seed=1000 * k + s) for s in range(S2)])
        sd2 = rng.integers(-1, inst.n, size=S2).astype(np.int32)
        ctx = rac.RacContext.from_instance(inst)
        din = torch.from_numpy(st2.view(np.int64)).cuda()
        dout = torch.zeros_like(din)
        its = torch.zeros(S2, dtype=torch.int32, device="cuda")
        sts = torch.zeros(S2, dtype=torch.int32, device="cuda")
        ctx.enforce_batch_seeded(S2, din, dout, its, sts, torch.from_numpy(sd2).cuda())
        torch.cuda.synchronize()
        out = dout.cpu().numpy().view(np.uint64)
        it_h, st_h = its.cpu().numpy(), sts.cpu().numpy()
        for s in range(S2):
            e = (orc.rac(st2[s], with_epochs=False) if sd2[s] < 0
                 else orc.rac_seeded(st2[s], [int(sd2[s])], with_epochs=False))
            assert (st_h[s], it_h[s]) == (e[0], e[2]) and np.array_equal(out[s], e[1]), (k, s, groups)


@pytest.mark.parametrize("variant", ["row_agg", "tiecols", "rows"])
def test_dense_sweep_variants(rac, variant, monkeypatch):
    """The dense persistent kernel's A/B variants give the oracle's exact trajectory (O7 at C3
    W-prop and W-seed): per-CTA shared-memory aggregation of the row sweep's removals
    (RAC_ROW_AGG), full passes on the column sweep (tiecols) or the row sweep (rows); and the
    create-time calibration reports its choice."""
    env = {"row_agg": ("RAC_ROW_AGG", "1"), "tiecols": ("RAC_FORCE_LAYOUT", "tiecols"),
           "rows": ("RAC_FORCE_LAYOUT", "rows")}[variant]
    monkeypatch.setenv(*env)
    dq = synth.quant_density(1.0)
    for t in (0.70, 0.5):
        tq = synth.quant_tightness(t)
        ctx = rac.RacContext.create_random(2000, 32, dq, tq, 1)
        root = synth.full_domains(np.full(2000, 32))
        g = ctx.enforce(root, removed_at=True)
        assert oracle.certify_trajectory_synth(2000, 32, dq, tq, 1, root, g[1], g[3], g[2], g[0]) == 0, (variant, t)
        if g[0] == oracle.OK and t == 0.5:
            ds, x, _ = synth.w_seed(g[1], 1)
            gs = ctx.enforce(ds, removed_at=True)  # a root call on the W-seed state: multi-pass, removal-heavy
            assert oracle.certify_trajectory_synth(2000, 32, dq, tq, 1, ds, gs[1], gs[3], gs[2], gs[0]) == 0
        lay, ms_c, ms_r = ctx.full_pass_layout
        if variant == "row_agg":
            assert lay in ("rows", "columns") and ms_c > 0 and ms_r > 0
        else:
            assert lay == ("columns" if variant == "tiecols" else "rows")


def test_nccl_exchange_leg_single_rank(rac):
    """The multi-GPU path with its real NCCL all-gather (a one-rank communicator,
    RAC_OPT_NCCL_SELF) gives the oracle's results: exercises dlopen of libnccl, comm init,
    the in-place ncclAllGather on the enforcement stream and the chunked host loop."""
    for k, inst in enumerate(I.random_corpus(60, seed0=97)):
        orc = oracle.Oracle.from_instance(inst)
        ctx = rac.RacContext.from_instance(inst, nccl_self=True)
        d_in = synth.w_rand(inst.dom, 0.9, seed=k)
        for full in (False, True):
            g, o = both(ctx, orc, d_in, full)
            assert_same(g, o, (k, full))
    dq, tq = synth.quant_density(1.0), synth.quant_tightness(0.70)
    ctx = rac.RacContext.create_random(2000, 32, dq, tq, 1, nccl_self=True)
    orc = oracle.Oracle.from_synth(2000, 32, dq, tq, 1)
    root = synth.full_domains(np.full(2000, 32))
    g, o = both(ctx, orc, root)
    assert_same(g, o, "c3-prop nccl")


# ----------------------------------------------------------------------------- batched contraction A/B
def test_batch_pass_eval_tc_and_bitsliced(rac):
    """One Eq. 1 pass for many states by the bit-sliced ALU contraction (impl 0) and the
    tcgen05 tensor-core contraction (impl 1): both equal the oracle's first step (values
    with removal epoch 1), on C5 dive states and on random instances with d <= 16."""
    import torch
    cases = []
    inst = synth.random_csp(200, 16, 0.8, 0.3, 1)
    orc = oracle.Oracle.from_instance(inst)
    _, root, _, _ = orc.rac(inst.full_domains(), with_epochs=False)
    states = synth.dive_states(root, lambda D: orc.rac(D, with_epochs=False)[:2], 300, seed=3)
    cases.append((inst, np.stack(states)))
    for k, ins in enumerate(I.random_corpus(20, seed0=101, n_range=(2, 40), d_range=(1, 16))):
        cases.append((ins, np.stack([synth.w_rand(ins.dom, 0.8, seed=50 * k + s) for s in range(37)])))
    for ci, (ins, st) in enumerate(cases):
        orc = oracle.Oracle.from_instance(ins)
        ctx = rac.RacContext.from_instance(ins)
        S = st.shape[0]
        din = torch.from_numpy(st.view(np.int64)).cuda()
        expect = []
        for s in range(S):
            _, _, _, rem = orc.rac(st[s])
            one = st[s].copy()
            for x in range(ins.n):
                for a in range(64):
                    if rem[x, a] == 1:
                        one[x] &= ~U64(1 << a)
            expect.append(one)
        for impl in (0, 1):
            dout = torch.zeros_like(din)
            ctx.batch_pass_eval(impl, S, din, dout)
            torch.cuda.synchronize()
            out = dout.cpu().numpy().view(np.uint64)
            for s in range(S):
                assert np.array_equal(out[s], expect[s]), (ci, impl, s)


def test_scratch_growth_interleaved(rac):
    """Growing one scratch buffer (the seed list, the batch exchange buffers) must
    leave the others intact: batched calls of growing size interleaved with seeded
    calls of growing seed lists on ONE context, every result against the oracle,
    then destroy (regression for a growth path that freed unrelated buffers)."""
    import torch
    inst = synth.random_csp(80, 10, 0.7, 0.4, 9)
    orc = oracle.Oracle.from_instance(inst)
    st0, root, _, _ = orc.rac(inst.full_domains())
    assert st0 == oracle.OK
    ctx = rac.RacContext.from_instance(inst)
    rng = np.random.default_rng(4)
    for rnd, (S, ns) in enumerate(((32, 1), (200, 7), (96, 40), (700, 80))):
        states = np.stack([synth.w_rand(inst.dom, 0.8, seed=1000 * rnd + s) for s in range(S)])
        din = torch.from_numpy(states.view(np.int64).copy()).cuda()
        dout = torch.zeros_like(din)
        its = torch.zeros(S, dtype=torch.int32, device="cuda")
        sts = torch.zeros(S, dtype=torch.int32, device="cuda")
        ctx.enforce_batch(S, din, dout, its, sts)
        torch.cuda.synchronize()
        out, its, sts = dout.cpu().numpy().view(np.uint64), its.cpu().numpy(), sts.cpu().numpy()
        for s in range(0, S, 7):
            e = orc.rac(states[s], with_epochs=False)
            assert (sts[s], its[s]) == (e[0], e[2]) and np.array_equal(out[s], e[1]), (rnd, s)
        seeds = rng.choice(inst.n, size=ns, replace=False).astype(np.int32)
        # the seeded-call precondition (DESIGN R12): AC on every c_xy with y not a
        # seed -- an AC state whose seed variables lost some values
        st_ac, d_in, _, _ = orc.rac(synth.w_rand(inst.dom, 0.9, seed=rnd), with_epochs=False)
        if st_ac != oracle.OK:
            d_in = root.copy()
        for x in seeds:
            vals = [a for a in range(64) if (int(d_in[x]) >> a) & 1]
            keep = rng.choice(vals, size=max(1, len(vals) - 1), replace=False)
            d_in[x] = U64(sum(1 << int(a) for a in keep))
        assert orc.rac(d_in, with_epochs=False)[2] == orc.rac_seeded(d_in, seeds, with_epochs=False)[2]
        g = ctx.enforce_seeded(d_in, seeds)
        o = orc.rac_seeded(d_in, seeds, with_epochs=False)
        assert (g[0], g[2]) == (o[0], o[2]) and np.array_equal(g[1], o[1]), ("seeded", rnd)
    ctx.close()


# ----------------------------------------------------------------------------- sparse layout (NEXT-3)
@pytest.mark.parametrize("n,d,p,t", [(9, 3, 0.5, 0.3), (33, 8, 0.7, 0.4), (70, 17, 0.3, 0.5), (40, 64, 0.9, 0.6),
                                     (17, 1, 1.0, 0.2), (50, 32, 0.2, 0.6)])
def test_sparse_packer_matches_oracle(rac, n, d, p, t):
    """Sparse arc blocks (RAC_OPT_SPARSE): every stored mask equals the oracle's
    support set c_xy|(x,a), absent pairs read back as all ones, presence bits
    match -- host-packed and generated instances."""
    inst = synth.random_csp(n, d, p, t, seed=5)
    orc = oracle.Oracle.from_instance(inst)
    for ctx in (rac.RacContext.from_instance(inst, layout="sparse"),
                rac.RacContext.create_random(n, d, synth.quant_density(p), synth.quant_tightness(t), 5,
                                             layout="sparse")):
        assert ctx.layout == "sparse"
        allones = U64((1 << (8 * ctx.mask_bytes)) - 1)
        for x in range(n):
            for a in range(d):
                masks, pres = ctx.read_row(x, a)
                for y in range(n):
                    present, s = orc.support(x, y, a)
                    assert bool(pres[y]) == present
                    assert masks[y] == (U64(s) if present else allones), (x, a, y)


def test_sparse_corpus(rac):
    """SPEC-corpus shapes and non-uniform domains through the sparse layout: full
    epoch parity in stop and full-fixpoint modes, empty rows included."""
    for k, inst in enumerate(I.random_corpus(300, seed0=77)):
        ctx = rac.RacContext.from_instance(inst, layout="sparse")
        orc = oracle.Oracle.from_instance(inst)
        d_in = inst.full_domains() if k % 3 == 0 else synth.w_rand(inst.dom, 0.85, seed=k)
        if k % 7 == 0:
            d_in[k % inst.n] = U64(0)
        for full in (False, True):
            g, o = both(ctx, orc, d_in, full)
            assert_same(g, o, (k, full))


@pytest.mark.parametrize("t,workload", [(0.5, "stream"), (0.74, "prop")])
def test_sparse_c3_density(rac, t, workload):
    """n=2000, d=32 at density 0.25 (the paper's density grid): the library
    picks the sparse layout by itself; W-stream (1 pass) / W-prop (~23 passes) root,
    W-rand, a W-seed seeded call and back-to-back launches all match the oracle;
    the dense layout gives the same results."""
    n, d = 2000, 32
    dq, tq = synth.quant_density(0.25), synth.quant_tightness(t)
    ctx = rac.RacContext.create_random(n, d, dq, tq, 1)
    assert ctx.layout == "sparse"
    assert ctx.relation_bytes < 0.3 * n * n * d * 4
    orc = oracle.Oracle.from_synth(n, d, dq, tq, 1)
    root = synth.full_domains(np.full(n, d))
    o_root = orc.rac(root)
    for rep in range(2):
        assert_same(ctx.enforce(root, removed_at=True), o_root, (workload, "root", rep))
    rnd = synth.w_rand(np.full(n, d), 0.9, 3)
    assert_same(ctx.enforce(rnd, removed_at=True), orc.rac(rnd), (workload, "rand"))
    if o_root[0] == oracle.OK:
        s, x, v = synth.w_seed(o_root[1], 7)
        g = ctx.enforce_seeded(s, [x])
        o = orc.rac(s, with_epochs=False)
        assert (g[0], g[2]) == (o[0], o[2]) and np.array_equal(g[1], o[1])
    dense = rac.RacContext.create_random(n, d, dq, tq, 1, layout="dense")
    assert dense.layout == "dense"
    assert_same(dense.enforce(root, removed_at=True), o_root, (workload, "dense"))


def test_sparse_unsupported_and_invalid(rac):
    """Sparse contexts refuse the batched calls (RAC_EUNSUPPORTED) and sparse with
    virtual shards is rejected at create (RAC_EINVAL)."""
    import torch
    inst = synth.random_csp(30, 8, 0.5, 0.4, seed=2)
    ctx = rac.RacContext.from_instance(inst, layout="sparse")
    din = torch.zeros((4, 30), dtype=torch.int64, device="cuda")
    i32 = torch.zeros(4, dtype=torch.int32, device="cuda")
    with pytest.raises(rac.RacError) as e:
        ctx.enforce_batch(4, din, din.clone(), i32, i32.clone())
    assert e.value.code == rac.RAC_EUNSUPPORTED
    with pytest.raises(rac.RacError) as e:
        rac.RacContext.from_instance(inst, layout="sparse", virtual_shards=2)
    assert e.value.code == rac.RAC_EINVAL


@pytest.mark.parametrize("n,d,p,t", [(120, 16, 0.3, 0.6), (90, 40, 0.4, 0.8), (80, 64, 0.35, 0.9), (150, 5, 0.2, 0.2)])
def test_sparse_mask_widths(rac, n, d, p, t):
    """Sparse arc blocks at every mask width (W = 1, 2, 8 bytes; dpad padding at
    d = 40 and d = 5), generated instances: W-root, W-rand and full-fixpoint mode
    with epochs, seeded calls after an assignment -- all equal to the oracle."""
    dq, tq = synth.quant_density(p), synth.quant_tightness(t)
    ctx = rac.RacContext.create_random(n, d, dq, tq, 4, layout="sparse")
    assert ctx.layout == "sparse"
    orc = oracle.Oracle.from_synth(n, d, dq, tq, 4)
    root = synth.full_domains(np.full(n, d))
    o_root = orc.rac(root)
    assert_same(ctx.enforce(root, removed_at=True), o_root, "root")
    for k in range(4):
        d_in = synth.w_rand(np.full(n, d), 0.85, 20 + k)
        for full in (False, True):
            g, o = both(ctx, orc, d_in, full)
            assert_same(g, o, (k, full))
    if o_root[0] == oracle.OK:
        for k in range(4):
            s, x, v = synth.w_seed(o_root[1], 9, k)
            g = ctx.enforce_seeded(s, [x])
            o = orc.rac(s, with_epochs=False)
            assert (g[0], g[2]) == (o[0], o[2]) and np.array_equal(g[1], o[1]), k


def test_sparse_nonuniform_domains(rac):
    """Per-variable domain sizes through the sparse layout (rows a >= dom(x) are
    padding inside each block, never live)."""
    rng = np.random.default_rng(8)
    for k in range(60):
        n = int(rng.integers(2, 40))
        dom = rng.integers(1, 30, size=n)
        cons = []
        for x in range(n):
            for y in range(x + 1, n):
                if rng.random() < 0.4:
                    allowed = [(a, b) for a in range(dom[x]) for b in range(dom[y]) if rng.random() > 0.3]
                    cons.append((x, y, allowed))
        inst = synth.from_constraints(n, dom, cons)
        ctx = rac.RacContext.from_instance(inst, layout="sparse")
        orc = oracle.Oracle.from_instance(inst)
        d_in = synth.w_rand(inst.dom, 0.85, seed=k)
        for full in (False, True):
            g, o = both(ctx, orc, d_in, full)
            assert_same(g, o, (k, full))
