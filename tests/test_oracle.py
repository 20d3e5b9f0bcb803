"""Pins for the CPU oracle (oracle/): each check ties the oracle to something
other than itself -- the paper's definitions, closed forms, hand traces,
brute force, an independent algorithm (AC-3), or a textbook routine (BFS).

Citations: PAPER.md line numbers (P:n), SPEC.md line numbers (S:n).
"""
from __future__ import annotations

import collections
import itertools

import numpy as np
import pytest

import oracle
import synth
from tests import _instances as I

U64 = np.uint64


def epochs_to_trace(rem, n, iters):
    trace = [set() for _ in range(iters)]
    for x in range(n):
        for a in range(64):
            t = int(rem[x, a])
            if t:
                trace[t - 1].add((x, a))
    return trace


# ----------------------------------------------------------------------------- hand traces
@pytest.mark.parametrize("name", I.golden_names())
def test_golden_hand_traces(name):
    """EQ2 / PATH3 / WIPE2 / SINGLE hand traces."""
    doc, inst = I.load_golden(name)
    exp = doc["expect"]
    orc = oracle.Oracle.from_instance(inst)
    d_in = np.asarray(doc["d_in"], dtype=U64)
    st, d_out, it, rem = orc.rac(d_in)
    assert st == (oracle.OK if exp["status"] == "OK" else oracle.WIPEOUT)
    assert [int(v) for v in d_out] == exp["d_out"]
    assert it == exp["iterations"]
    trace = epochs_to_trace(rem, inst.n, it)
    assert trace == [set(map(tuple, s)) for s in exp["trace"]]
    # the pure-Python transcription agrees
    st2, d2, it2, tr2 = oracle.rac_python(inst, d_in)
    assert (st2, [int(v) for v in d2], it2) == (st, [int(v) for v in d_out], it)
    assert tr2 == trace
    # AC-3 reaches the same verdict (and D when consistent)
    st3, d3, _ = orc.ac3(d_in)
    assert st3 == st
    if st == oracle.OK:
        assert np.array_equal(d3, d_out)


# ----------------------------------------------------------------------------- brute force
def test_bruteforce_union_of_ac_subsets():
    """O3 (union of all AC subsets) == O1 full mode on 300 tiny instances.
    Inputs: W-root and W-rand domain states."""
    for k, inst in enumerate(I.tiny_corpus(300)):
        orc = oracle.Oracle.from_instance(inst)
        for d_in in (inst.full_domains(), synth.w_rand(inst.dom, 0.8, seed=k)):
            bf = oracle.brute_force_dac(inst, d_in)
            st, d_out, it, rem = orc.rac(d_in, full=True)
            assert np.array_equal(bf, d_out), (k, inst.to_json())
            assert (st == oracle.WIPEOUT) == bool(np.any(bf == 0))


def test_bruteforce_is_ac_definition():
    """The brute-force AC predicate and the C audit agree on every subset of tiny instances."""
    for k, inst in enumerate(I.tiny_corpus(40, seed0=3)):
        if int(inst.dom.sum()) > 10:
            continue
        orc = oracle.Oracle.from_instance(inst)
        sup = oracle._support_sets(inst)
        elems = sorted(oracle._to_set(inst.full_domains()))
        for mask in range(1 << len(elems)):
            S = {elems[i] for i in range(len(elems)) if (mask >> i) & 1}
            assert oracle._is_ac_set(sup, S) == orc.is_ac(oracle._from_set(S, inst.n))


# ----------------------------------------------------------------------------- AC-3 agreement
def test_rac_agrees_with_ac3_corpus():
    """S:528 corpus (>=1000 instances, n 2..20, d 1..6): O1 ≡ O2 on verdict, and on D when
    consistent; O1 full mode has an empty row iff stop mode reports WIPEOUT; stop and full
    modes coincide when no wipeout happens."""
    corpus = I.random_corpus(1000)
    n_wipe = 0
    for k, inst in enumerate(corpus):
        orc = oracle.Oracle.from_instance(inst)
        d_in = inst.full_domains() if k % 2 == 0 else synth.w_rand(inst.dom, 0.9, seed=k)
        st, d_out, it, _ = orc.rac(d_in)
        st3, d3, _ = orc.ac3(d_in)
        stf, dfull, itf, _ = orc.rac(d_in, full=True)
        assert st == st3, k
        assert (st == oracle.WIPEOUT) == bool(np.any(dfull == 0)), k
        if st == oracle.OK:
            assert np.array_equal(d_out, d3), k
            assert np.array_equal(d_out, dfull) and it == itf, k
        n_wipe += st == oracle.WIPEOUT
    assert 50 < n_wipe < 950  # the corpus exercises both outcomes


def test_c_and_python_transcriptions_agree():
    """Two transcriptions of Eq. 1 (C over bitsets, Python over sets) give the same
    trajectory (per-step removal sets) on 300 random instances, stop and full modes."""
    for k, inst in enumerate(I.random_corpus(300, seed0=5, n_range=(2, 9), d_range=(1, 5))):
        orc = oracle.Oracle.from_instance(inst)
        d_in = synth.w_rand(inst.dom, 0.85, seed=k)
        for full in (False, True):
            st, d_out, it, rem = orc.rac(d_in, full=full)
            st2, d2, it2, tr2 = oracle.rac_python(inst, d_in, full=full)
            assert (st, it) == (st2, it2)
            assert np.array_equal(d_out, d2)
            assert epochs_to_trace(rem, inst.n, it) == tr2


# ----------------------------------------------------------------------------- certificate
def test_certificate_accepts_and_rejects():
    """O4 accepts every correct full-mode result; rejects over-pruned results (a kept value
    marked removed) and under-pruned ones (a removed value put back)."""
    rng = np.random.default_rng(11)
    rejected_over = rejected_under = 0
    for k, inst in enumerate(I.random_corpus(300, seed0=9)):
        orc = oracle.Oracle.from_instance(inst)
        d_in = inst.full_domains()
        st, d_out, it, rem = orc.rac(d_in, full=True)
        assert orc.certify(d_in, d_out, rem) == 0
        kept = [(x, a) for x in range(inst.n) for a in range(64) if (int(d_out[x]) >> a) & 1]
        if kept:
            x, a = kept[int(rng.integers(len(kept)))]
            bad = d_out.copy()
            bad[x] &= ~(U64(1) << U64(a))
            brem = rem.copy()
            brem[x, a] = int(rng.integers(1, it + 2))
            assert orc.certify(d_in, bad, brem) != 0
            rejected_over += 1
        removed = [(x, a) for x in range(inst.n) for a in range(64) if rem[x, a]]
        if removed:
            x, a = removed[int(rng.integers(len(removed)))]
            bad = d_out.copy()
            bad[x] |= U64(1) << U64(a)
            brem = rem.copy()
            brem[x, a] = 0
            assert orc.certify(d_in, bad, brem) != 0
            rejected_under += 1
    assert rejected_over > 100 and rejected_under > 100


def test_certificate_on_stop_mode_wipeouts():
    """Stop-mode WIPEOUT results: every removal is sound (Lemma 1 part only)."""
    seen = 0
    for k, inst in enumerate(I.random_corpus(400, seed0=13)):
        orc = oracle.Oracle.from_instance(inst)
        st, d_out, it, rem = orc.rac(inst.full_domains())
        if st == oracle.WIPEOUT:
            assert orc.certify(inst.full_domains(), d_out, rem, check_ac=False) == 0
            seen += 1
    assert seen > 20


# ----------------------------------------------------------------------------- closed forms
@pytest.mark.parametrize("n,d", [(1, 1), (5, 3), (17, 8), (40, 64)])
def test_tightness_zero_is_identity(n, d):
    """Tightness 0: every relation is universal, nothing is removed, 1 pass."""
    inst = synth.random_csp(n, d, 1.0, 0.0, seed=3)
    st, d_out, it, _ = oracle.Oracle.from_instance(inst).rac(inst.full_domains())
    assert st == oracle.OK and it == 1 and np.array_equal(d_out, inst.full_domains())


@pytest.mark.parametrize("n,d", [(2, 1), (3, 5), (4, 64), (9, 2)])
def test_empty_relation_wipes_in_one_pass(n, d):
    """An empty relation on a pair wipes both variables in pass 1 (WIPE2)."""
    cons = [(0, 1, [])] + [(i, i + 1, I.eq_rel(d)) for i in range(1, n - 1)]
    inst = synth.from_constraints(n, d, cons)
    st, d_out, it, _ = oracle.Oracle.from_instance(inst).rac(inst.full_domains())
    assert st == oracle.WIPEOUT and it == 1 and d_out[0] == 0 and d_out[1] == 0


@pytest.mark.parametrize("n,d,embed", [(2, 2, False), (7, 3, False), (30, 8, False), (12, 5, True), (25, 32, True)])
def test_equality_chain_takes_exactly_n_passes(n, d, embed):
    """Equality chain x_i = x_{i+1}, x_0 = {0}: step k of Eq. 1 removes the nonzero values
    of x_k only (its sole support chain runs through x_{k-1}), so D_ac = all {0}, reached
    after n-1 removing steps plus the final quiescent one: exactly n iterations."""
    inst = I.equality_chain(n, d, embed_complete=embed)
    d_in = inst.full_domains()
    d_in[0] = U64(1)
    st, d_out, it, rem = oracle.Oracle.from_instance(inst).rac(d_in)
    assert st == oracle.OK and it == n
    assert np.all(d_out == U64(1))
    for k in range(1, n):
        assert all(int(rem[k, a]) == k for a in range(1, d))


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8, 11, 20])
def test_two_ended_path(n):
    """x_0 = {0}, x_{n-1} = {1}, equality chain, d = 2: the left wave removes value 1 from
    x_k at step k, the right wave removes 0 from x_{n-1-k} at step k; they collide at step
    floor(n/2) -> stop mode WIPEOUT there.  Full mode keeps propagating: every domain
    ends empty and the n-th pass is the first quiescent one."""
    inst = I.equality_chain(n, 2)
    d_in = inst.full_domains()
    d_in[0] = U64(1)
    d_in[n - 1] = U64(2)
    orc = oracle.Oracle.from_instance(inst)
    st, d_out, it, _ = orc.rac(d_in)
    assert st == oracle.WIPEOUT and it == n // 2
    stf, dfull, itf, _ = orc.rac(d_in, full=True)
    assert stf == oracle.WIPEOUT and itf == n and np.all(dfull == 0)


def test_d1_full_mode_is_multisource_bfs():
    """d = 1: a constraint either allows (0,0) or forbids it.  Endpoints of forbidden
    constraints lose their only value at step 1; a variable adjacent (by any declared
    constraint) to a removed one loses its only support one step later.  So the removal
    epoch of x is 1 + BFS distance from the forbidden endpoints in the constraint graph,
    and iterations = max depth + 2 (or 1 if nothing is forbidden)."""
    rng = np.random.default_rng(21)
    for k in range(300):
        n = int(rng.integers(1, 30))
        p = float(rng.uniform(0.05, 0.5))
        t = float(rng.uniform(0.0, 0.15))
        inst = synth.random_csp(n, 1, p, t, seed=1000 + k)
        adj = collections.defaultdict(list)
        sources = set()
        for j in range(inst.n_rel):
            x, y = int(inst.xs[j]), int(inst.ys[j])
            adj[x].append(y)
            adj[y].append(x)
            if int(inst.rows[j, 0]) == 0:
                sources |= {x, y}
        dist = {s: 0 for s in sources}
        q = collections.deque(sources)
        while q:
            u = q.popleft()
            for v in adj[u]:
                if v not in dist:
                    dist[v] = dist[u] + 1
                    q.append(v)
        st, d_out, it, rem = oracle.Oracle.from_instance(inst).rac(inst.full_domains(), full=True)
        for x in range(n):
            if x in dist:
                assert d_out[x] == 0 and rem[x, 0] == dist[x] + 1
            else:
                assert d_out[x] == 1 and rem[x, 0] == 0
        assert it == (max(dist.values()) + 2 if dist else 1)


def test_empty_input_row():
    """Reading R7: an empty row in D_in -> one pass (only neighbours of the empty
    variable can lose values), then WIPEOUT with iterations = 1 (Alg. 1)."""
    inst = synth.from_constraints(4, 2, [(0, 1, [(0, 0), (1, 1)]), (2, 3, [(0, 0), (1, 1)])])
    d_in = inst.full_domains()
    d_in[0] = U64(0)
    st, d_out, it, _ = oracle.Oracle.from_instance(inst).rac(d_in)
    assert st == oracle.WIPEOUT and it == 1
    assert [int(v) for v in d_out] == [0, 0, 3, 3]
    # AC-3's upfront check gives the same verdict
    assert oracle.Oracle.from_instance(inst).ac3(d_in)[0] == oracle.WIPEOUT


# ----------------------------------------------------------------------------- invariants
def _solutions(inst):
    doms = [range(int(k)) for k in inst.dom]
    sols = []
    for assn in itertools.product(*doms):
        ok = all((int(inst.rows[j, assn[inst.xs[j]]]) >> assn[inst.ys[j]]) & 1 for j in range(inst.n_rel))
        if ok:
            sols.append(assn)
    return sols


def test_invariants_corpus():
    """Prop. 1/2 and SPEC invariants on 400 random instances:
    result AC; idempotent (re-enforce -> 1 pass, unchanged); subset of input; iterations
    <= |D_in| + 1; Prop. 2 cause check; solutions preserved; equivariant under
    relabelling variables."""
    rng = np.random.default_rng(17)
    for k, inst in enumerate(I.random_corpus(400, seed0=19, n_range=(2, 12), d_range=(1, 5))):
        orc = oracle.Oracle.from_instance(inst)
        d_in = synth.w_rand(inst.dom, 0.9, seed=k)
        st, d_out, it, rem = orc.rac(d_in, full=True)
        assert np.all((d_out & ~d_in) == 0)
        assert orc.is_ac(d_out)
        assert it <= sum(synth.popcount64(v) for v in d_in) + 1
        st2, d2, it2, _ = orc.rac(d_out, full=True)
        assert it2 == 1 and np.array_equal(d2, d_out)
        # Prop. 2 (2): every value removed at step k >= 2 has a c_xy whose supports
        # outside D~(k-2) all lie in V^(k-1).
        for x in range(inst.n):
            for a in range(64):
                t = int(rem[x, a])
                if t < 2:
                    continue
                ok = False
                for y in range(inst.n):
                    pres, s = orc.support(x, y, a)
                    if not pres:
                        continue
                    rest = [b for b in range(64) if (s >> b) & 1 and (int(d_in[y]) >> b) & 1
                            and not (1 <= rem[y, b] <= t - 2)]
                    if all(rem[y, b] == t - 1 for b in rest):
                        ok = True
                        break
                assert ok, (k, x, a)
        # solutions preserved (tiny only)
        if np.prod(inst.dom.astype(np.float64)) <= 2e4:
            for s in _solutions(inst):
                if all((int(d_in[x]) >> s[x]) & 1 for x in range(inst.n)):
                    assert all((int(d_out[x]) >> s[x]) & 1 for x in range(inst.n))
        # equivariance under a variable permutation
        perm = rng.permutation(inst.n)
        inv = np.argsort(perm)
        cons = [(int(perm[inst.xs[j]]), int(perm[inst.ys[j]]),
                 [(a, b) for a in range(int(inst.dom[inst.xs[j]])) for b in range(int(inst.dom[inst.ys[j]]))
                  if (int(inst.rows[j, a]) >> b) & 1]) for j in range(inst.n_rel)]
        pinst = synth.from_constraints(inst.n, inst.dom[inv], cons)
        pst, pd, pit, _ = oracle.Oracle.from_instance(pinst).rac(d_in[inv], full=True)
        assert pst == st and pit == it and np.array_equal(pd, d_out[inv])


def test_monotone():
    """D_in ⊆ D_in' => D_ac(D_in) ⊆ D_ac(D_in') (D_ac is the largest AC subset)."""
    for k, inst in enumerate(I.random_corpus(200, seed0=23, n_range=(2, 12))):
        orc = oracle.Oracle.from_instance(inst)
        big = synth.w_rand(inst.dom, 0.95, seed=k)
        small = big & synth.w_rand(inst.dom, 0.8, seed=k + 7)
        _, ds, _, _ = orc.rac(small, full=True)
        _, db, _, _ = orc.rac(big, full=True)
        assert np.all((ds & ~db) == 0)


# ----------------------------------------------------------------------------- generator
@pytest.mark.parametrize("n,d,p,t,seed", [(7, 5, 0.6, 0.3, 1), (20, 8, 0.5, 0.4, 2), (13, 64, 1.0, 0.5, 3),
                                          (31, 17, 0.3, 0.7, 4), (9, 1, 1.0, 0.2, 5)])
def test_generator_numpy_matches_c_header(n, d, p, t, seed):
    """synth/__init__.py (numpy) and synth/csp_synth.h (used by orc_build_synth) produce the
    same instance: compare every support set of both orientations."""
    inst = synth.random_csp(n, d, p, t, seed)
    a = oracle.Oracle.from_instance(inst)
    b = oracle.Oracle.from_synth(n, d, synth.quant_density(p), synth.quant_tightness(t), seed)
    for x in range(n):
        assert a.degree(x) == b.degree(x)
        for y in range(n):
            for v in range(d):
                assert a.support(x, y, v) == b.support(x, y, v)


def test_row_supported_synth_matches_one_step():
    """The on-the-fly row test equals membership in one step of O1 from D."""
    n, d, p, t, seed = 30, 12, 0.7, 0.55, 9
    inst = synth.random_csp(n, d, p, t, seed)
    orc = oracle.Oracle.from_instance(inst)
    D = synth.w_rand(inst.dom, 0.8, seed=4)
    st, d1, it, rem = orc.rac(D)
    for x in range(n):
        for a in range(d):
            if not (int(D[x]) >> a) & 1:
                continue
            sup = oracle.row_supported_synth(n, d, synth.quant_density(p), synth.quant_tightness(t), seed, x, a, D)
            assert sup == (rem[x, a] != 1)


def test_generator_statistics():
    """Constraint count ≈ density·n(n-1)/2 and allowed fraction ≈ 1 - tightness."""
    inst = synth.random_csp(200, 16, 0.3, 0.25, seed=77)
    m = inst.n_rel
    exp = 0.3 * 200 * 199 / 2
    assert abs(m - exp) < 4 * np.sqrt(exp * 0.7)
    bits = sum(bin(int(v)).count("1") for v in inst.rows.reshape(-1))
    cells = m * 16 * 16
    assert abs(bits / cells - 0.75) < 0.01
    assert synth.random_csp(3, 4, 1.0, 0.5, seed=1).n_rel == 3


def test_pass_block_matches_one_step():
    """The block-restricted step (used for sampled CPU timing) equals one O1 step."""
    n, d, p, t, seed = 40, 9, 0.8, 0.5, 12
    inst = synth.random_csp(n, d, p, t, seed)
    D = synth.w_rand(inst.dom, 0.85, seed=3)
    st, d1, it, rem = oracle.Oracle.from_instance(inst).rac(D)
    blk = oracle.Oracle.from_synth_block(n, d, synth.quant_density(p), synth.quant_tightness(t), seed, 7, 23)
    out, removed = blk.pass_block(D, 7, 23)
    for x in range(7, 23):
        expect = int(D[x]) & ~sum(1 << a for a in range(64) if rem[x, a] == 1)
        assert int(out[x - 7]) == expect
    assert removed == int(np.sum(rem[7:23] == 1))


# ----------------------------------------------------------------------------- Alg. 1 (seeded)
def test_seeded_all_equals_root():
    """tensorAC(Vars, all variables) is the root call: identical to O1."""
    for k, inst in enumerate(I.random_corpus(200, seed0=41)):
        orc = oracle.Oracle.from_instance(inst)
        d_in = synth.w_rand(inst.dom, 0.9, seed=k)
        for full in (False, True):
            a = orc.rac(d_in, full=full)
            b = orc.rac_seeded(d_in, np.arange(inst.n), full=full)
            assert a[0] == b[0] and a[2] == b[2] and np.array_equal(a[1], b[1]) and np.array_equal(a[3], b[3])


def test_seeded_after_assignment_matches_full_trajectory():
    """Prop. 2: after an assignment to x on an AC state (W-seed), Alg. 1 seeded
    with [x] follows exactly the same trajectory as the full recurrence: same
    status, D, iteration count and per-step removal sets.  Checked on W-seed and W-dive
    states (the precondition: D_in is AC on every c_xy with y not a seed)."""
    n_checked = 0
    for k, inst in enumerate(I.random_corpus(300, seed0=43, n_range=(3, 20))):
        orc = oracle.Oracle.from_instance(inst)
        st, root, _, _ = orc.rac(inst.full_domains())
        if st != oracle.OK:
            continue
        for j in range(3):
            s, x, v = synth.w_seed(root, k, j)
            a = orc.rac(s)
            b = orc.rac_seeded(s, [x])
            assert a[0] == b[0] and a[2] == b[2], (k, j)
            assert np.array_equal(a[1], b[1]) and np.array_equal(a[3], b[3])
            n_checked += 1
    assert n_checked > 200


def test_seeded_empty_and_precondition_violated():
    """Empty @changed: no pass.  Without the precondition the seeded call can keep
    values the full recurrence removes (it only looks at the changed columns)."""
    inst = synth.from_constraints(2, 2, [(0, 1, [(0, 0)])])
    orc = oracle.Oracle.from_instance(inst)
    st, d, it, _ = orc.rac_seeded(inst.full_domains(), [])
    assert it == 0 and st == oracle.OK and np.array_equal(d, inst.full_domains())
    # EQ2 seeded with [0] (precondition violated: full domains are not AC on c_01):
    # pass 1 tests only column x0 -> removes (1,1); pass 2 tests column x1 -> removes (0,1);
    # pass 3 tests column x0 -> nothing.  Same D as the full recurrence, 3 passes instead of 2.
    st, d, it, rem = orc.rac_seeded(inst.full_domains(), [0])
    assert (st, it, [int(v) for v in d]) == (oracle.OK, 3, [1, 1])
    assert rem[1, 1] == 1 and rem[0, 1] == 2
    assert orc.rac(inst.full_domains())[2] == 2


# ----------------------------------------------------------------------------- Alg. 2 search
def _enumerate(inst):
    return _solutions(inst)


def test_search_matches_enumeration():
    """O6 (Alg. 2) on 200 tiny instances: Solution iff the brute-force
    enumeration is non-empty; the solution satisfies every constraint and is one of the
    enumerated ones; with all_solutions the count equals the enumeration's (AC never
    removes a solution value, and every complete assignment reached is a solution)."""
    for k, inst in enumerate(I.random_corpus(200, seed0=71, n_range=(1, 7), d_range=(1, 4))):
        sols = _enumerate(inst)
        orc = oracle.Oracle.from_instance(inst)
        r, sol, st = orc.search(inst.full_domains())
        assert r == (0 if sols else 1), k
        if sols:
            assert tuple(int(v) for v in sol) in set(sols)
        r2, _, st2 = orc.search(inst.full_domains(), all_solutions=True)
        assert st2["solutions"] == len(sols)


def test_search_engines_agree():
    """The search tree depends only on D_ac at each node: O5 (seeded, the paper's call),
    O1 (full recurrence) and O2 (AC-3) explore identical trees (assignments, wipeouts,
    solution); O5 and O1 also give the same #Recurrence sum (Prop. 2 precondition holds
    at every node)."""
    for k, inst in enumerate(I.random_corpus(150, seed0=73, n_range=(3, 16), d_range=(2, 6))):
        orc = oracle.Oracle.from_instance(inst)
        res = {e: orc.search(inst.full_domains(), max_assignments=400, engine=e) for e in ("seeded", "full", "ac3")}
        for e in ("full", "ac3"):
            assert res[e][0] == res["seeded"][0]
            for key in ("assignments", "wipeouts", "solutions", "max_depth"):
                assert res[e][2][key] == res["seeded"][2][key], (k, e, key)
            assert np.array_equal(res[e][1], res["seeded"][1])
        assert res["full"][2]["recurrences"] == res["seeded"][2]["recurrences"]


def test_search_hand_cases():
    """SPEC mac_search examples: EQ2 -> x0=0, x1=0; WIPE2 -> unsat at the root;
    unconstrained n=3, d=2 -> (0,0,0)."""
    _, eq2 = I.load_golden("eq2.json")
    r, sol, st = oracle.Oracle.from_instance(eq2).search(eq2.full_domains())
    assert r == 0 and list(sol) == [0, 0]
    _, w2 = I.load_golden("wipe2.json")
    assert oracle.Oracle.from_instance(w2).search(w2.full_domains())[0] == 1
    free = synth.from_constraints(3, 2, [])
    r, sol, st = oracle.Oracle.from_instance(free).search(free.full_domains())
    assert r == 0 and list(sol) == [0, 0, 0] and st["assignments"] == 3


# ----------------------------------------------------------------------------- wide domains (NEXT-4)
from tests import _wide as WD  # noqa: E402


def _narrow_cases():
    inst = []
    for i, (n, d, p, t) in enumerate([(12, 20, 0.6, 0.8), (9, 40, 1.0, 0.91), (15, 33, 0.4, 0.88),
                                      (6, 50, 0.8, 0.93), (10, 7, 0.7, 0.45)]):
        inst.append(synth.random_csp(n, d, p, t, seed=501 + i))
    return inst


@pytest.mark.parametrize("case", range(5))
@pytest.mark.parametrize("k", [2, 4, 5])
@pytest.mark.parametrize("masked", [False, True])
def test_wide_value_duplication(case, k, masked):
    """O1w pinned to the (pinned) one-word O1 by value duplication: copy j of
    value a is value j*d + a and (a', b') is allowed iff (a' mod d, b' mod d) is.
    Eq. 1's support test depends on D(y) only through the set of values
    with a live copy, so the wide trajectory projects onto the narrow one run from
    the projected D_in: same status, same iteration count, a copy removed at
    epoch t iff its value is removed at t.  `masked` keeps random copies only, so
    copies of one value sit in different words with different liveness (a test
    that looked at one word of D(y) would fail)."""
    narrow = _narrow_cases()[case]
    if int(narrow.dom.max()) * k > 256:
        pytest.skip("beyond 256 values")
    rng = np.random.default_rng(case * 10 + k) if masked else None
    n = narrow.n
    d_in_n = synth.w_rand(narrow.dom, 0.9, seed=case + 3)
    wide = WD.duplicate(narrow, k)
    d_in_w = WD.duplicate_state(narrow, k, d_in_n, rng)
    proj = WD.project(narrow, k, d_in_w)
    for full in (False, True):
        st_n, out_n, it_n, rem_n = oracle.Oracle.from_instance(narrow).rac(proj, full=full)
        wo = oracle.WideOracle.from_instance(wide)
        st_w, out_w, it_w, rem_w = wo.rac(d_in_w, full=full)
        assert (st_w, it_w) == (st_n, it_n)
        assert np.array_equal(WD.project(narrow, k, out_w), out_n)
        win = WD.bits_of(d_in_w, n, wo.wq)
        wout = WD.bits_of(out_w, n, wo.wq)
        for x in range(n):
            dx = int(narrow.dom[x])
            for ap in range(dx * k):
                a = ap % dx
                if win[x, ap]:
                    assert wout[x, ap] == bool((int(out_n[x]) >> a) & 1)
                    assert rem_w[x, ap] == rem_n[x, a]
                else:
                    assert not wout[x, ap] and rem_w[x, ap] == 0


def test_wide_one_word_equals_o1():
    """With d <= 64 the wide oracle is O1 itself (wq = 1): identical outputs and epochs."""
    for i, inst in enumerate(I.random_corpus(40, seed0=77, n_range=(2, 14), d_range=(1, 64))):
        d_in = synth.w_rand(inst.dom, 0.8, seed=i)
        rows3 = np.asarray(inst.rows, dtype=U64).reshape(inst.n_rel, int(inst.dom.max()), 1)
        wi = synth.Instance(n=inst.n, dom=inst.dom, xs=inst.xs, ys=inst.ys, rows=rows3)
        a = oracle.Oracle.from_instance(inst).rac(d_in)
        b = oracle.WideOracle.from_instance(wi).rac(d_in)
        assert a[0] == b[0] and a[2] == b[2] and np.array_equal(a[1], b[1]) and np.array_equal(a[3], b[3])


def _wide_corpus(count, seed0):
    rng = np.random.default_rng(seed0)
    out = []
    for i in range(count):
        n = int(rng.integers(2, 12))
        d = int(rng.integers(65, 257))
        # tightness 1 - u/d: about u allowed values per row, so the recurrence propagates
        out.append(synth.random_csp_wide(n, d, float(rng.uniform(0.2, 1.0)), 1.0 - float(rng.uniform(1.0, 4.0)) / d,
                                         seed=seed0 * 1009 + i))
    return out


def _lemma1_certificate(wo, inst, d_in, d_out, rem):
    """Lemma 1 (proof P:304-308) for every removal in epoch order:
    (x,a) removed at epoch t has a declared c_xy whose supports in D_in were all
    removed before t.  Written here from the definitions (independent of oracle.c)."""
    n, wq = inst.n, wo.wq
    win, wout = WD.bits_of(d_in, n, wq), WD.bits_of(d_out, n, wq)
    arcs = {}
    for r in range(inst.n_rel):
        x, y = int(inst.xs[r]), int(inst.ys[r])
        arcs.setdefault(x, []).append((y, r, False))
        arcs.setdefault(y, []).append((x, r, True))
    for x in range(n):
        for a in range(int(inst.dom[x])):
            if not win[x, a] or wout[x, a]:
                continue
            t = int(rem[x, a])
            assert t >= 1
            ok = False
            for (y, r, rev) in arcs.get(x, []):
                sup = [b for b in range(int(inst.dom[y]))
                       if ((int(inst.rows[r, b, a >> 6]) >> (a & 63)) & 1 if rev
                           else (int(inst.rows[r, a, b >> 6]) >> (b & 63)) & 1) and win[y, b]]
                if all((not wout[y, b]) and 1 <= int(rem[y, b]) < t for b in sup):
                    ok = True
                    break
            assert ok, (x, a, t)


def test_wide_ac3_audit_certificate():
    """Random wide instances (65..256 values): O1w in FULL mode equals AC-3 at the
    fixpoint (AC-3 computes D_ac), the output passes the definitional AC
    audit unless a domain is empty, and every removal carries a Lemma-1
    certificate -- together D_out = D_ac."""
    for i, inst in enumerate(_wide_corpus(30, 31)):
        wo = oracle.WideOracle.from_instance(inst)
        d_in = synth.w_rand_wide(inst.dom, 0.85, seed=i)
        st, out, it, rem = wo.rac(d_in, full=True)
        st3, out3 = wo.ac3(d_in)
        assert np.array_equal(out, out3) and st == st3
        if st == oracle.OK:
            assert wo.is_ac(out)
        _lemma1_certificate(wo, inst, d_in, out, rem)


def test_wide_equality_chain_closed_form():
    """x_i = x_{i+1} with dom 200 and D_in(x_0) = {150} (word 2 of 4): pass t
    restricts x_t, so D_ac(x_i) = {150} for all i after n - 1 removing passes plus
    the final unchanged one (iterations = n; Prop. 1)."""
    n, d = 9, 200
    inst = synth.wide_from_constraints(n, d, [(i, i + 1, [(a, a) for a in range(d)]) for i in range(n - 1)])
    wo = oracle.WideOracle.from_instance(inst)
    D = WD.bits_of(synth.full_domains_wide(inst.dom), n, wo.wq)
    D[0, :] = False
    D[0, 150] = True
    st, out, it, rem = wo.rac(WD.words_of(D))
    ob = WD.bits_of(out, n, wo.wq)
    assert st == oracle.OK and it == n
    assert all(ob[x].sum() == 1 and ob[x, 150] for x in range(n))
    for x in range(1, n):
        assert all(int(rem[x, a]) == x for a in range(d) if a != 150)


def test_wide_synth_matches_numpy_generator():
    """orc_wbuild_synth (C, csp_synth.h) and random_csp_wide (numpy) are the same instance."""
    for (n, d, p, t, s) in [(14, 100, 0.5, 0.9, 3), (8, 256, 1.0, 0.97, 4), (20, 65, 0.3, 0.8, 5)]:
        inst = synth.random_csp_wide(n, d, p, t, s)
        a = oracle.WideOracle.from_instance(inst)
        b = oracle.WideOracle.from_synth(n, d, synth.quant_density(p), synth.quant_tightness(t), s)
        d_in = synth.w_rand_wide(inst.dom, 0.9, seed=s)
        ra, rb = a.rac(d_in, full=True), b.rac(d_in, full=True)
        assert ra[0] == rb[0] and ra[2] == rb[2] and np.array_equal(ra[1], rb[1])


def test_wide_pass_block_matches_o1w():
    """orc_wpass_block over every row block equals the first step of O1w (the
    removal epochs equal to 1), and the block build agrees with the full build."""
    n, d, dq, tq, seed = 24, 130, synth.quant_density(0.7), synth.quant_tightness(0.975), 9
    full = oracle.WideOracle.from_synth(n, d, dq, tq, seed)
    D = synth.w_rand_wide(np.full(n, d), 0.8, seed=1)
    st, out, it, rem = full.rac(D, full=True)
    exp = WD.bits_of(D, n, full.wq) & ~(rem == 1)
    got = np.zeros_like(exp)
    for lo in range(0, n, 5):
        hi = min(n, lo + 5)
        blk = oracle.WideOracle.from_synth_block(n, d, dq, tq, seed, lo, hi)
        o, _ = blk.pass_block(D, lo, hi)
        got[lo:hi] = WD.bits_of(o, n, full.wq)[lo:hi]
    assert np.array_equal(got, exp)


# ----------------------------------------------------------------------------- O7 exact-trajectory certificate
def _perturbations(d_in, d_out, rem, it, st, n, rng, wq=1):
    """Claims that differ from the recurrence's output (status, d_out, iterations,
    epochs) in one plausible way each: (kind, d_out', rem', it', st')."""
    out = []
    nb = 64 * wq
    din = np.asarray(d_in, dtype=U64).reshape(n, wq)
    dout = np.asarray(d_out, dtype=U64).reshape(n, wq)

    def bit(D, x, a):
        return (int(D[x, a >> 6]) >> (a & 63)) & 1

    def setb(D, x, a, v):
        D = D.copy()
        if v:
            D[x, a >> 6] |= U64(1) << U64(a & 63)
        else:
            D[x, a >> 6] &= ~(U64(1) << U64(a & 63))
        return D

    removed = [(x, a) for x in range(n) for a in range(nb) if rem[x, a]]
    kept = [(x, a) for x in range(n) for a in range(nb) if bit(dout, x, a)]
    if removed:
        x, a = removed[int(rng.integers(len(removed)))]
        e = int(rem[x, a])
        for de in (-1, +1):  # epoch one pass early / late, value still removed
            if 1 <= e + de <= it:
                r2 = rem.copy()
                r2[x, a] = e + de
                out.append(("epoch%+d" % de, dout.reshape(-1), r2, it, st))
        r2 = rem.copy()  # under-pruned: the value put back
        r2[x, a] = 0
        out.append(("under", setb(dout, x, a, 1).reshape(-1), r2, it, st))
    if kept:
        x, a = kept[int(rng.integers(len(kept)))]
        r2 = rem.copy()  # over-pruned: a kept value claimed removed
        r2[x, a] = int(rng.integers(1, it + 1))
        out.append(("over", setb(dout, x, a, 0).reshape(-1), r2, it, st))
    out.append(("iters+1", dout.reshape(-1), rem, it + 1, st))
    if it > 1:
        out.append(("iters-1", dout.reshape(-1), rem, it - 1, st))
    out.append(("status", dout.reshape(-1), rem, it, 1 - st))
    return out


def test_trajectory_certificate_accepts_recurrence_and_rejects_perturbations():
    """O7 (oracle.c orc_certify_trajectory) accepts O1's output (O1 is pinned by
    brute force, AC-3 and the hand traces above) in stop and full mode on W-root
    and W-rand inputs, and rejects every one-step perturbation: an epoch moved one
    pass (Prop. 2: a removal at k is caused at k-1), a value put back
    (fails the AC rule), a kept value claimed removed (fails Lemma 1), a
    wrong iteration count or status (Alg. 1 loop control).  O4 cannot
    see epoch shifts that keep Lemma 1 true; O7 must."""
    rng = np.random.default_rng(21)
    counts = collections.Counter()
    o4_blind = 0
    for k, inst in enumerate(I.random_corpus(400, seed0=17) +
                             [synth.random_csp(20, 8, 0.5, 0.4, s) for s in range(1, 101)]):
        orc = oracle.Oracle.from_instance(inst)
        d_in = inst.full_domains() if k % 2 == 0 else synth.w_rand(inst.dom, 0.85, seed=k)
        for full in (False, True):
            st, d_out, it, rem = orc.rac(d_in, full=full)
            assert orc.certify_trajectory(d_in, d_out, rem, it, st, full) == 0, (k, full)
            for kind, o2, r2, it2, st2 in _perturbations(d_in, d_out, rem, it, st, inst.n, rng):
                assert orc.certify_trajectory(d_in, o2, r2, it2, st2, full) != 0, (k, full, kind)
                counts[kind] += 1
                if kind.startswith("epoch") and orc.certify(d_in, o2, r2, check_ac=(st == oracle.OK)) == 0:
                    o4_blind += 1
    for kind in ("epoch-1", "epoch+1", "under", "over", "iters+1", "iters-1", "status"):
        assert counts[kind] > 40, counts
    assert o4_blind > 10, o4_blind


def test_trajectory_certificate_hand_traces():
    """The hand traces: EQ2 / PATH3 / WIPE2 outputs are accepted with
    their traced epochs and iteration counts; the PATH3 trace with its two
    epochs swapped is rejected."""
    for name in I.golden_names():
        doc, inst = I.load_golden(name)
        orc = oracle.Oracle.from_instance(inst)
        exp = doc["expect"]
        rem = np.zeros((inst.n, 64), dtype=np.int32)
        for t, s in enumerate(exp["trace"], start=1):
            for (x, a) in s:
                rem[x, a] = t
        st = oracle.OK if exp["status"] == "OK" else oracle.WIPEOUT
        d_in = np.asarray(doc["d_in"], dtype=U64)
        d_out = np.asarray(exp["d_out"], dtype=U64)
        assert orc.certify_trajectory(d_in, d_out, rem, exp["iterations"], st) == 0, name
        if name.startswith("path3"):
            sw = rem.copy()
            sw[rem == 1], sw[rem == 2] = 2, 1
            assert orc.certify_trajectory(d_in, d_out, sw, exp["iterations"], st) != 0


def test_trajectory_certificate_synth_streaming_matches():
    """orc_certify_trajectory_synth (support sets regenerated per variable from
    the generator, OpenMP over variables) gives the same verdicts as the
    in-memory O7 on the same seeded instances, for 1 and 4 threads, one-word
    and wide domains."""
    rng = np.random.default_rng(5)
    for (n, d, p, t, s) in [(60, 20, 1.0, 0.3, 1), (45, 64, 0.6, 0.75, 2), (30, 8, 0.5, 0.4, 3)]:
        dq, tq = synth.quant_density(p), synth.quant_tightness(t)
        orc = oracle.Oracle.from_synth(n, d, dq, tq, s)
        d_in = synth.w_rand(np.full(n, d), 0.9, seed=s)
        for full in (False, True):
            st, d_out, it, rem = orc.rac(d_in, full=full)
            for th in (1, 4):
                assert oracle.certify_trajectory_synth(n, d, dq, tq, s, d_in, d_out, rem, it, st, full, th) == 0
            for kind, o2, r2, it2, st2 in _perturbations(d_in, d_out, rem, it, st, n, rng):
                a = orc.certify_trajectory(d_in, o2, r2, it2, st2, full)
                b = oracle.certify_trajectory_synth(n, d, dq, tq, s, d_in, o2, r2, it2, st2, full, 4)
                assert a != 0 and b != 0, (kind, a, b)  # codes may differ: first failing variable vs any
    for (n, d, p, t, s) in [(24, 130, 0.7, 0.975, 9), (12, 256, 1.0, 0.985, 4)]:
        dq, tq = synth.quant_density(p), synth.quant_tightness(t)
        wo = oracle.WideOracle.from_synth(n, d, dq, tq, s)
        d_in = synth.w_rand_wide(np.full(n, d), 0.8, seed=s)
        for full in (False, True):
            st, d_out, it, rem = wo.rac(d_in, full=full)
            assert wo.certify_trajectory(d_in, d_out, rem, it, st, full) == 0
            assert oracle.certify_trajectory_synth(n, d, dq, tq, s, d_in, d_out, rem, it, st, full, 2) == 0
            for kind, o2, r2, it2, st2 in _perturbations(d_in, d_out, rem, it, st, n, rng, wo.wq):
                a = wo.certify_trajectory(d_in, o2, r2, it2, st2, full)
                b = oracle.certify_trajectory_synth(n, d, dq, tq, s, d_in, o2, r2, it2, st2, full, 2)
                assert a != 0 and b != 0, (kind, a, b)  # codes may differ: first failing variable vs any


def test_wide_trajectory_certificate_corpus():
    """O7 on wide domains (wcertify): accepts O1w (pinned above by value
    duplication and AC-3) on the random wide corpus, rejects the perturbations."""
    rng = np.random.default_rng(8)
    counts = collections.Counter()
    for i, inst in enumerate(_wide_corpus(30, 77)):
        wo = oracle.WideOracle.from_instance(inst)
        d_in = synth.w_rand_wide(inst.dom, 0.85, seed=i)
        for full in (False, True):
            st, out, it, rem = wo.rac(d_in, full=full)
            assert wo.certify_trajectory(d_in, out, rem, it, st, full) == 0
            for kind, o2, r2, it2, st2 in _perturbations(d_in, out, rem, it, st, inst.n, rng, wo.wq):
                assert wo.certify_trajectory(d_in, o2, r2, it2, st2, full) != 0, (i, kind)
                counts[kind] += 1
    assert counts["under"] > 10 and counts["over"] > 10 and counts["epoch+1"] + counts["epoch-1"] > 10


def test_wide_is_ac_negative():
    """orc_wis_ac is the AC definition plus "no empty domain": D_ac
    (AC) is accepted; D_ac plus any one removed value of D_in is rejected (D_ac is
    the largest AC subset, so a superset cannot be AC); emptying the
    domain of a variable without constraints keeps the set AC by definition but
    is rejected by the empty-domain clause."""
    checked = 0
    for i, inst in enumerate(_wide_corpus(30, 41)):
        wo = oracle.WideOracle.from_instance(inst)
        d_in = synth.w_rand_wide(inst.dom, 0.9, seed=i)
        st, out, it, rem = wo.rac(d_in, full=True)
        if st != oracle.OK:
            continue
        assert wo.is_ac(out)
        ob = WD.bits_of(out, inst.n, wo.wq)
        for (x, a) in list(zip(*np.nonzero(rem)))[:5]:
            b2 = ob.copy()
            b2[x, a] = True
            assert not wo.is_ac(WD.words_of(b2)), (i, x, a)
            checked += 1
    assert checked > 20
    # an isolated variable (no constraint): emptying it leaves an AC set with an empty domain
    n, d = 4, 100
    inst = synth.wide_from_constraints(n, d, [(0, 1, [(a, a) for a in range(d)]), (1, 2, [(a, a) for a in range(d)])])
    wo = oracle.WideOracle.from_instance(inst)
    D = synth.full_domains_wide(inst.dom)
    assert wo.is_ac(D)
    bits = WD.bits_of(D, n, wo.wq)
    bits[3, :] = False
    assert not wo.is_ac(WD.words_of(bits))


def test_parallel_o1_equals_o1():
    """orc_rac_par (the all-core CPU baseline) equals orc_rac for 1, 3 and 8 threads,
    stop and full mode, on the corpus and a C2-shaped instance."""
    insts = I.random_corpus(150, seed0=23)
    for k, inst in enumerate(insts):
        orc = oracle.Oracle.from_instance(inst)
        d_in = inst.full_domains() if k % 2 else synth.w_rand(inst.dom, 0.85, seed=k)
        for full in (False, True):
            st, out, it, _ = orc.rac(d_in, full=full, with_epochs=False)
            for th in (1, 3, 8):
                g = orc.rac_par(d_in, full=full, threads=th)
                assert g[0] == st and g[2] == it and np.array_equal(g[1], out), (k, full, th)
    dq, tq = synth.quant_density(1.0), synth.quant_tightness(0.3)
    orc = oracle.Oracle.from_synth(500, 20, dq, tq, 1)
    d_in = synth.w_rand(np.full(500, 20), 0.9, 2)
    st, out, it, _ = orc.rac(d_in, with_epochs=False)
    g = orc.rac_par(d_in, threads=4)
    assert (g[0], g[2]) == (st, it) and np.array_equal(g[1], out)
    assert oracle.max_threads() >= 1
    inst = synth.random_csp(60, 8, 0.5, 0.4, 3)
    orc = oracle.Oracle.from_instance(inst)
    states = np.stack([synth.w_rand(inst.dom, 0.8, seed=s) for s in range(40)])
    st, out, it = orc.rac_many(states, threads=4)
    for s in range(40):
        o = orc.rac(states[s], with_epochs=False)
        assert (st[s], it[s]) == (o[0], o[2]) and np.array_equal(out[s], o[1])


def test_wide_search_equals_one_word_search():
    """O6w on instances whose domains fit one word (wq = 1) explores exactly O6's
    tree with the full-recurrence engine (same verdict, first solution and
    statistics), on tiny corpus instances with all solutions counted."""
    for k, inst in enumerate(I.random_corpus(60, seed0=97, n_range=(2, 9), d_range=(1, 5))):
        orc = oracle.Oracle.from_instance(inst)
        cons = []
        for r in range(inst.n_rel):
            x, y = int(inst.xs[r]), int(inst.ys[r])
            cons.append((x, y, [(a, b) for a in range(int(inst.dom[x])) for b in range(int(inst.dom[y]))
                                if (int(inst.rows[r, a]) >> b) & 1]))
        wide = synth.wide_from_constraints(inst.n, np.asarray(inst.dom), cons)
        wo = oracle.WideOracle.from_instance(wide)
        assert wo.wq == 1
        d_in = inst.full_domains()
        a = orc.search(d_in, engine="full", all_solutions=True)
        b = wo.search(d_in, all_solutions=True)
        assert a[0] == b[0] and a[2] == b[2] and np.array_equal(a[1], b[1]), k


def test_wide_search_solution_counts_by_enumeration():
    """O6w with all solutions on tiny wide instances (n = 3, domains 65..100
    values, several words): the solution count equals brute-force enumeration of
    every complete assignment, and the first solution satisfies every
    constraint."""
    rng = np.random.default_rng(4)
    for k in range(6):
        n = 3
        dom = rng.integers(65, 101, size=n)
        cons = []
        for x in range(n):
            for y in range(x + 1, n):
                allowed = [(a, b) for a in range(int(dom[x])) for b in range(int(dom[y]))
                           if (a * 7 + b * 3 + k) % 11 == 0 or a == b]
                cons.append((x, y, allowed))
        inst = synth.wide_from_constraints(n, dom.astype(np.int32), cons)
        wo = oracle.WideOracle.from_instance(inst)
        rel = {(x, y): set(al) for (x, y, al) in cons}
        count = 0
        for a0 in range(int(dom[0])):
            for a1 in range(int(dom[1])):
                if (a0, a1) not in rel[(0, 1)]:
                    continue
                for a2 in range(int(dom[2])):
                    if (a0, a2) in rel[(0, 2)] and (a1, a2) in rel[(1, 2)]:
                        count += 1
        r, sol, stats = wo.search(synth.full_domains_wide(inst.dom), all_solutions=True)
        assert stats["solutions"] == count, (k, stats, count)
        assert (r == 0) == (count > 0)
        if count:
            assert (sol[0], sol[1]) in rel[(0, 1)] and (sol[0], sol[2]) in rel[(0, 2)] and \
                (sol[1], sol[2]) in rel[(1, 2)]
