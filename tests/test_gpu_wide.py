"""GPU parity for wide domains (65..256 values per
variable): the CUDA path (rac_wide.cu through the C ABI) against the wide
oracle O1w (oracle.WideOracle, pinned in tests/test_oracle.py) on the same
seeded inputs.  Integer work: status, D_out, iteration count and removal
epochs must be bit-exact.  Expected values come only from oracle/."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from tests import _wide as WD
from tests.test_oracle import _narrow_cases, _wide_corpus

pytestmark = pytest.mark.gpu

U64 = np.uint64


@pytest.fixture(scope="module")
def rac():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2407_11388_b200 import rac as r
    return r


def same(ctx, wo, d_in, full=False, what=""):
    g = ctx.enforce(d_in, full=full, removed_at=True)
    o = wo.rac(d_in, full=full)
    assert g[0] == o[0], (what, "status", g[0], o[0])
    assert g[2] == o[2], (what, "iterations", g[2], o[2])
    assert np.array_equal(g[1], o[1]), (what, "d_out")
    assert np.array_equal(g[3], o[3]), (what, "removed_at")
    return g


def test_wide_corpus(rac):
    """Random wide instances (65..256 values, density 0.2..1, propagating
    tightness), W-root and W-rand, stop and FULL modes."""
    for i, inst in enumerate(_wide_corpus(40, 91)):
        ctx = rac.RacContext.from_instance(inst)
        wo = oracle.WideOracle.from_instance(inst)
        assert ctx.wq == wo.wq == synth.words_per_var(int(inst.dom.max()))
        for d_in in (synth.full_domains_wide(inst.dom), synth.w_rand_wide(inst.dom, 0.8, seed=i)):
            for full in (False, True):
                same(ctx, wo, d_in, full, "corpus %d" % i)


def test_wide_nonuniform_domains(rac):
    """Domain sizes mixed across the one-word boundary (1..256 in one instance)."""
    rng = np.random.default_rng(5)
    for i in range(12):
        n = int(rng.integers(3, 40))
        dom = rng.integers(1, 257, size=n)
        dom[int(rng.integers(n))] = int(rng.integers(65, 257))  # at least one wide domain
        cons = []
        for x in range(n):
            for y in range(x + 1, n):
                if rng.random() < 0.5:
                    p = min(1.0, 3.0 / max(1, int(dom[y])))
                    allowed = [(a, b) for a in range(int(dom[x])) for b in np.nonzero(rng.random(int(dom[y])) < p)[0]]
                    cons.append((x, y, allowed))
        inst = synth.wide_from_constraints(n, dom.astype(np.int32), cons)
        ctx = rac.RacContext.from_instance(inst)
        wo = oracle.WideOracle.from_instance(inst)
        for d_in in (synth.full_domains_wide(inst.dom), synth.w_rand_wide(inst.dom, 0.7, seed=i)):
            same(ctx, wo, d_in, False, "nonuniform %d" % i)
            same(ctx, wo, d_in, True, "nonuniform %d full" % i)


@pytest.mark.parametrize("k", [2, 4, 5])
def test_wide_duplication(rac, k):
    """Value-duplicated instances (tests/_wide.py) with random copy masks."""
    for case, narrow in enumerate(_narrow_cases()):
        if int(narrow.dom.max()) * k > 256 or int(narrow.dom.max()) * k <= 64:
            continue
        wide = WD.duplicate(narrow, k)
        ctx = rac.RacContext.from_instance(wide)
        wo = oracle.WideOracle.from_instance(wide)
        d_in = WD.duplicate_state(narrow, k, synth.w_rand(narrow.dom, 0.9, seed=case),
                                  np.random.default_rng(case))
        same(ctx, wo, d_in, False, "dup %d" % case)
        same(ctx, wo, d_in, True, "dup %d full" % case)


def test_wide_equality_chain(rac):
    n, d = 300, 200
    inst = synth.wide_from_constraints(n, d, [(i, i + 1, [(a, a) for a in range(d)]) for i in range(n - 1)])
    ctx = rac.RacContext.from_instance(inst)
    wo = oracle.WideOracle.from_instance(inst)
    D = WD.bits_of(synth.full_domains_wide(inst.dom), n, wo.wq)
    D[0, :] = False
    D[0, 150] = True
    g = same(ctx, wo, WD.words_of(D), False, "chain")
    assert g[0] == rac.RAC_OK and g[2] == n


def test_wide_edge_cases(rac):
    """Empty D_in row (reading R7: one pass, then WIPEOUT), all-empty D_in, no
    constraints, a single variable, d_in bits beyond the domains rejected."""
    inst = _wide_corpus(3, 17)[0]
    ctx = rac.RacContext.from_instance(inst)
    wo = oracle.WideOracle.from_instance(inst)
    d_in = synth.full_domains_wide(inst.dom).reshape(inst.n, -1)
    d_in[1, :] = 0
    g = same(ctx, wo, d_in.reshape(-1), False, "empty row")
    assert g[0] == rac.RAC_WIPEOUT and g[2] == 1
    same(ctx, wo, d_in.reshape(-1), True, "empty row full")
    same(ctx, wo, np.zeros_like(d_in).reshape(-1), False, "all empty")
    free = synth.wide_from_constraints(5, 130, [])
    cf, of = rac.RacContext.from_instance(free), oracle.WideOracle.from_instance(free)
    g = same(cf, of, synth.full_domains_wide(free.dom), False, "no constraints")
    assert g[0] == rac.RAC_OK and g[2] == 1
    one = synth.wide_from_constraints(1, 256, [])
    same(rac.RacContext.from_instance(one), oracle.WideOracle.from_instance(one),
         synth.full_domains_wide(one.dom), False, "n=1")
    bad = synth.full_domains_wide(free.dom).reshape(5, -1)
    bad[0, -1] |= U64(1) << U64(63)  # value 191 of a 130-value domain
    with pytest.raises(rac.RacError) as ei:
        cf.enforce(bad.reshape(-1))
    assert ei.value.code == rac.RAC_EINVAL
    with pytest.raises(rac.RacError) as ei:
        cf.enforce_seeded(bad.reshape(-1), [0])
    assert ei.value.code == rac.RAC_EINVAL


def _assignments(ctx, wo, n, wq, d_ac, rng, count):
    """Alg. 2's per-assignment call on a wide context: from
    the arc-consistent D_ac, x := a (D(x) = {a}), then tensorAC(Vars, [x]).  By
    Prop. 2 the seeded result equals the full enforcement of the
    assigned state, which the oracle computes from scratch."""
    bits = WD.bits_of(d_ac, n, wq)
    xs = [x for x in range(n) if bits[x].sum() >= 2]
    for _ in range(min(count, len(xs))):
        x = int(rng.choice(xs))
        a = int(rng.choice(np.flatnonzero(bits[x])))
        b2 = bits.copy()
        b2[x, :] = False
        b2[x, a] = True
        d_in = WD.words_of(b2)
        o = wo.rac(d_in)
        for seeds in ([x], [x, x]):
            g = ctx.enforce_seeded(d_in, seeds)
            assert g[0] == o[0], ("status", x, a, g[0], o[0])
            assert g[2] == o[2], ("iterations", x, a, g[2], o[2])
            assert np.array_equal(g[1], o[1]), ("d_out", x, a)


def test_wide_seeded(rac):
    """Seeded wide enforcement (NEXT-1 on NEXT-4 contexts) against O1w on the
    assigned state, on corpus instances and a generator instance; an empty
    seed list is no pass (iterations 0, D_out = D_in, status from emptiness)."""
    rng = np.random.default_rng(23)
    cases = [(inst, rac.RacContext.from_instance(inst), oracle.WideOracle.from_instance(inst))
             for inst in _wide_corpus(20, 57)]
    checked = 0
    for inst, ctx, wo in cases:
        st, d_ac, _, _ = wo.rac(synth.full_domains_wide(inst.dom))
        if st != rac.RAC_OK:
            continue
        _assignments(ctx, wo, inst.n, wo.wq, d_ac, rng, 4)
        checked += 1
        g = ctx.enforce_seeded(d_ac, [])
        assert g[0] == rac.RAC_OK and g[2] == 0 and np.array_equal(g[1], d_ac)
        e = d_ac.reshape(inst.n, -1).copy()
        e[0, :] = 0
        g = ctx.enforce_seeded(e.reshape(-1), [])
        assert g[0] == rac.RAC_WIPEOUT and g[2] == 0
    assert checked >= 5
    n, d = 200, 128  # t = 0.93: root D_ac is OK after 5 passes (0.94 wipes out)
    dq, tq = synth.quant_density(1.0), synth.quant_tightness(0.93)
    ctx = rac.RacContext.create_random(n, d, dq, tq, 7)
    wo = oracle.WideOracle.from_synth(n, d, dq, tq, 7)
    st, d_ac, _, _ = wo.rac(synth.full_domains_wide(np.full(n, d)))
    assert st == rac.RAC_OK
    _assignments(ctx, wo, n, wo.wq, d_ac, rng, 6)


@pytest.mark.parametrize("n,d,t", [(200, 128, 0.97), (120, 256, 0.985), (150, 100, 0.96), (90, 192, 0.98)])
def test_wide_generator(rac, n, d, t):
    """rac_create_random (device generator + packer) against the oracle's own
    build of the same seeded instance; W-root and W-rand, stop and FULL."""
    dq, tq = synth.quant_density(1.0 if d != 100 else 0.5), synth.quant_tightness(t)
    ctx = rac.RacContext.create_random(n, d, dq, tq, 7)
    wo = oracle.WideOracle.from_synth(n, d, dq, tq, 7)
    dom = np.full(n, d)
    for d_in in (synth.full_domains_wide(dom), synth.w_rand_wide(dom, 0.9, seed=3)):
        for full in (False, True):
            same(ctx, wo, d_in, full, "gen n=%d d=%d" % (n, d))


def _sample_supported(n, d, dq, tq, seed, x, a, Dbits):
    """Straight from the numpy generator: is (x,a) supported on every declared
    c_xy against D?  (one step of Eq. 1 for one row)."""
    px, py = synth.present_pairs(n, dq, seed)
    sel = (px == x) | (py == x)
    lo, hi = px[sel], py[sel]
    rows = synth.relation_rows_wide(n, d, lo, hi, tq, seed)  # [pairs, d, wq] of c_{lo hi}
    for k in range(lo.shape[0]):
        if int(lo[k]) == x:   # c_xy is the pair's own orientation: row a
            y = int(hi[k])
            sup = [b for b in range(d) if (int(rows[k, a, b >> 6]) >> (b & 63)) & 1]
        else:                 # c_xy = transpose of c_yx: column a
            y = int(lo[k])
            sup = [b for b in range(d) if (int(rows[k, b, a >> 6]) >> (a & 63)) & 1]
        if not any(Dbits[y, b] for b in sup):
            return False
    return True


@pytest.mark.parametrize("n,d", [(2000, 128), (1000, 256)])
def test_wide_bench_size_stream(rac, n, d):
    """The bench's W-stream configurations at full size, in the bench's launch
    configuration: every row supported -> one pass, D_out = D_in (checked on
    sampled rows straight from the generator), status OK."""
    import torch
    dq, tq = synth.quant_density(1.0), synth.quant_tightness(0.5)
    ctx = rac.RacContext.create_random(n, d, dq, tq, 1)
    full = synth.full_domains_wide(np.full(n, d))
    dev = torch.device("cuda", 0)
    din = torch.from_numpy(full.view(np.int64).copy()).to(dev)
    dout = torch.zeros_like(din)
    its = torch.zeros(1, dtype=torch.int32, device=dev)
    sts = torch.zeros(1, dtype=torch.int32, device=dev)
    ctx.enforce_async(din, dout, its, sts)
    torch.cuda.synchronize()
    out = dout.cpu().numpy().view(np.uint64)
    assert int(sts.item()) == rac.RAC_OK and int(its.item()) == 1
    assert np.array_equal(out, full)
    # the whole output certified by the oracle's O7 (every row's support on every
    # column regenerated from the generator), not a sample
    g = ctx.enforce(full, removed_at=True)
    assert oracle.certify_trajectory_synth(n, d, dq, tq, 1, full, g[1], g[3], g[2], g[0]) == 0


def test_wide_search_parity(rac):
    """rac_search on wide contexts (Alg. 2, seeded enforcement per
    assignment) explores the same tree as the wide oracle O6w: same verdict,
    first solution and statistics (assignments, #Recurrence, wipeouts,
    solutions, depth) -- whole trees on small wide instances (all solutions),
    and a budgeted search on a 60-variable generator instance."""
    checked = 0
    for k, inst in enumerate(_wide_corpus(12, 71)):
        ctx = rac.RacContext.from_instance(inst)
        wo = oracle.WideOracle.from_instance(inst)
        d_in = synth.full_domains_wide(inst.dom)
        # all solutions under an assignment budget (loose instances have up to
        # d^n leaves): the same budget cuts both trees at the same node
        r, sol, st = ctx.search(d_in, max_assignments=3000, all_solutions=True)
        ro, solo, sto = wo.search(d_in, max_assignments=3000, all_solutions=True)
        assert r == {0: rac.RAC_OK, 1: rac.RAC_WIPEOUT, 2: rac.RAC_BUDGET}[ro], (k, r, ro)
        for key in ("assignments", "recurrences", "wipeouts", "solutions", "max_depth"):
            assert st[key] == sto[key], (k, key, st[key], sto[key])
        if r == rac.RAC_OK:
            assert np.array_equal(sol, solo), k
        checked += 1
    assert checked >= 4
    n, d = 60, 100
    dq, tq = synth.quant_density(0.5), synth.quant_tightness(0.95)
    ctx = rac.RacContext.create_random(n, d, dq, tq, 3)
    wo = oracle.WideOracle.from_synth(n, d, dq, tq, 3)
    d_in = synth.full_domains_wide(np.full(n, d))
    r, sol, st = ctx.search(d_in, max_assignments=300)
    ro, solo, sto = wo.search(d_in, max_assignments=300)
    assert {0: rac.RAC_OK, 1: rac.RAC_WIPEOUT, 2: rac.RAC_BUDGET}[ro] == r
    for key in ("assignments", "recurrences", "wipeouts", "solutions", "max_depth"):
        assert st[key] == sto[key], (key, st[key], sto[key])


def test_wide_nonuniform_domains_at_scale(rac):
    """Non-uniform wide domains at n = 1000 (NEXT-4): domain sizes 16..200 drawn
    per variable (four words per variable; domains inside one word and across
    word boundaries), density 0.02, tightness 0.75 (3-4 removing passes);
    root and W-rand enforcements in stop and full mode equal O1w (status, D_out,
    iterations, epochs) and are accepted by the O7 certificate."""
    n, d = 1000, 200
    rng = np.random.default_rng(12)
    dom = rng.integers(16, d + 1, size=n).astype(np.int32)
    base = synth.random_csp_wide(n, d, 0.02, 0.75, seed=8)
    inst = WD.restrict_domains(base, dom)
    ctx = rac.RacContext.from_instance(inst)
    wo = oracle.WideOracle.from_instance(inst)
    assert ctx.wq == 4 or ctx.wq == wo.wq
    for k, d_in in enumerate((synth.full_domains_wide(inst.dom), synth.w_rand_wide(inst.dom, 0.8, seed=3))):
        for full in (False, True):
            g = same(ctx, wo, d_in, full, (k, full))
            assert wo.certify_trajectory(d_in, g[1], g[3], g[2], g[0], full) == 0


@pytest.mark.parametrize("impl", ["state", "tc-f16", "tc-fp8"])
def test_wide_batched(rac, impl, monkeypatch):
    """Batched enforcement on wide contexts -- one block per state (wide_state),
    and the tensor-core batch (every pass one dense tcgen05 contraction of all
    states, fp8 (default) or f16 operands, then per-state loop control; d <= 128, other
    instances fall back to wide_state): every state's (status, D_out,
    iterations) equals O1w on that state alone -- W-rand states in stop and full
    mode, and assigned states (x := a on the root D_ac) with their assigned
    variable as the per-state seed (Prop. 2)."""
    import torch
    monkeypatch.setenv("RAC_WIDE_BATCH", "state" if impl == "state" else "tc")
    monkeypatch.setenv("RAC_WIDE_TC", "f16" if impl == "tc-f16" else "fp8")
    rng = np.random.default_rng(31)
    for k, inst in enumerate(_wide_corpus(10, 91)):
        ctx = rac.RacContext.from_instance(inst)
        wo = oracle.WideOracle.from_instance(inst)
        S = 40 + k
        states = np.stack([synth.w_rand_wide(inst.dom, 0.85, seed=1000 * k + s) for s in range(S)])
        din = torch.from_numpy(states.view(np.int64).copy()).cuda()
        for full in (False, True):
            dout = torch.zeros_like(din)
            its = torch.zeros(S, dtype=torch.int32, device="cuda")
            sts = torch.zeros(S, dtype=torch.int32, device="cuda")
            ctx.enforce_batch(S, din, dout, its, sts, full=full)
            torch.cuda.synchronize()
            out = dout.cpu().numpy().view(np.uint64)
            for s in range(S):
                o = wo.rac(states[s], full=full, with_epochs=False)
                assert (int(sts[s]), int(its[s])) == (o[0], o[2]), (k, s, full)
                assert np.array_equal(out[s], o[1]), (k, s, full)
        st, root, _, _ = wo.rac(synth.full_domains_wide(inst.dom), with_epochs=False)
        if st != oracle.OK:
            continue
        bits = WD.bits_of(root, inst.n, wo.wq)
        xs = [x for x in range(inst.n) if bits[x].sum() >= 2]
        if not xs:
            continue
        seeds, sts_ = [], []
        for s in range(24):
            x = int(rng.choice(xs))
            a = int(rng.choice(np.flatnonzero(bits[x])))
            b2 = bits.copy()
            b2[x, :] = False
            b2[x, a] = True
            sts_.append(WD.words_of(b2))
            seeds.append(x)
        states = np.stack(sts_)
        din = torch.from_numpy(states.view(np.int64).copy()).cuda()
        dout = torch.zeros_like(din)
        its = torch.zeros(24, dtype=torch.int32, device="cuda")
        sts = torch.zeros(24, dtype=torch.int32, device="cuda")
        sv = torch.from_numpy(np.asarray(seeds, dtype=np.int32)).cuda()
        ctx.enforce_batch_seeded(24, din, dout, its, sts, sv)
        torch.cuda.synchronize()
        out = dout.cpu().numpy().view(np.uint64)
        for s in range(24):
            o = wo.rac(states[s], with_epochs=False)
            assert (int(sts[s]), int(its[s])) == (o[0], o[2]) and np.array_equal(out[s], o[1]), (k, s, "seeded")


@pytest.mark.parametrize("impl", [2, 3, 4])
def test_wide_pass_eval_bitsliced_and_tcgen05(rac, impl):
    """The wide batched-pass A/B kernels (rac_batch_pass_eval impl 2 = bit-sliced
    byte tables, impl 3 = pipelined tcgen05 f16 MMA with TMEM accumulators,
    impl 4 = the same with fp8 e4m3 0/1 operands, kind::f8f6f4):
    ONE step of Eq. 1 for every state, D_1 = D_0 minus the values O1w removes
    in its first pass (removal epoch 1), on instances with 65..128 values
    (non-uniform included) and 300 states spanning several 256-state tiles."""
    import torch
    cases = [synth.random_csp_wide(40, 128, 0.6, 1.0 - 3.0 / 128, 7),
             synth.random_csp_wide(33, 100, 0.9, 0.95, 8)]
    rng = np.random.default_rng(2)
    dom = rng.integers(65, 129, size=50).astype(np.int32)
    cases.append(WD.restrict_domains(synth.random_csp_wide(50, 128, 0.5, 0.9, 9), dom))
    for k, inst in enumerate(cases):
        ctx = rac.RacContext.from_instance(inst)
        wo = oracle.WideOracle.from_instance(inst)
        S = 300
        states = np.stack([synth.w_rand_wide(inst.dom, 0.7, seed=50 * k + s) for s in range(S)])
        din = torch.from_numpy(states.view(np.int64).copy()).cuda()
        dout = torch.zeros_like(din)
        ctx.batch_pass_eval(impl, S, din, dout)
        torch.cuda.synchronize()
        out = dout.cpu().numpy().view(np.uint64)
        for s in range(S):
            _, _, _, rem = wo.rac(states[s])
            exp = WD.words_of(WD.bits_of(states[s], inst.n, wo.wq) & (rem != 1))
            assert np.array_equal(out[s], exp), (k, s)
