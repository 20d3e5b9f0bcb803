"""Bench-size GPU results certified exactly, and the seeded-call edge cases.

* C4 (BASELINE configs[3]: n=8000, d=64, density 1, 32.8 GB of masks), the
  NEXT-4 bench instance w128-prop (n=2000, d=128) and the NEXT-3 bench instance
  c3s-prop (n=4000, density 0.25): the GPU's (status, D_out, iterations,
  removal epochs) are accepted by the oracle's exact-trajectory certificate O7
  (oracle.c orc_certify_trajectory*, pinned in tests/test_oracle.py), which
  accepts only the RAC recurrence's own output (Eq. 1; Lemma 1,
  P:79-82; Prop. 2; Alg. 1 loop control) -- at sizes
  where the oracle's own recurrence would not fit in host memory.
* The sharded per-pass path compared with the ORACLE (not with the fused path).
* Seeded calls with an empty seed list on fresh contexts of every path, and
  seed lists on the sharded path.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from tests import _instances as I

pytestmark = pytest.mark.gpu

U64 = np.uint64

# C4 W-prop: a consistent propagating root enforcement at C4 (tools/c4_scan.py,
# profiles/r02a/c4_scan.jsonl; SURVEY §8(d) predicted t ~ 0.82)
C4_PROP_T = 0.82  # 18 passes, consistent, 22 428 values removed


@pytest.fixture(scope="module")
def rac():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2407_11388_b200 import rac as r
    return r


def _need_free(nbytes):
    import torch
    free, _ = torch.cuda.mem_get_info()
    if free < nbytes:
        pytest.skip("needs %.0f GB free device memory" % (nbytes / 1e9))


def _certify(n, d, dq, tq, seed, d_in, g, full=False):
    st, d_out, it, rem = g
    return oracle.certify_trajectory_synth(n, d, dq, tq, seed, d_in, d_out, rem, it, st, full)


@pytest.mark.parametrize("kind", ["prop", "rand"])
def test_c4_certified(rac, kind):
    """C4 on one GPU: W-prop (root enforcement at C4_PROP_T, many passes) and
    W-rand (t=0.85, 10% of the values dropped: a removing, wiping run).  The
    GPU's full output is certified exactly by O7 streaming the instance from the
    generator."""
    _need_free(70e9)
    n, d = 8000, 64
    dq = synth.quant_density(1.0)
    if kind == "prop":
        seed, tq = 1, synth.quant_tightness(C4_PROP_T)
        d_in = synth.full_domains(np.full(n, d))
    else:
        seed, tq = 2, synth.quant_tightness(0.85)
        d_in = synth.w_rand(np.full(n, d), 0.9, 3)
    ctx = rac.RacContext.create_random(n, d, dq, tq, seed)
    g = ctx.enforce(d_in, removed_at=True)
    ctx.close()
    del ctx
    if kind == "prop":
        assert g[2] >= 5, g[2]
    assert int((g[3] > 0).sum()) > 0
    assert _certify(n, d, dq, tq, seed, d_in, g) == 0, (g[0], g[2])


def test_w128_prop_certified(rac):
    """NEXT-4 bench workload w128-prop (n=2000, d=128, t=0.93: a few removing
    passes ending in a wipeout) certified exactly, plus W-rand in full mode."""
    _need_free(20e9)
    n, d = 2000, 128
    dq, tq = synth.quant_density(1.0), synth.quant_tightness(0.93)
    ctx = rac.RacContext.create_random(n, d, dq, tq, 1)
    full = synth.full_domains_wide(np.full(n, d))
    g = ctx.enforce(full, removed_at=True)
    assert g[2] >= 2
    assert _certify(n, d, dq, tq, 1, full, g) == 0
    dr = synth.w_rand_wide(np.full(n, d), 0.97, 5)
    g = ctx.enforce(dr, full=True, removed_at=True)
    assert _certify(n, d, dq, tq, 1, dr, g, full=True) == 0


def test_c3s_prop_bench_config(rac):
    """The sparse bench configuration c3s-prop itself (n=4000, d=32, density 0.25,
    t=0.72): exact parity with the oracle's recurrence, epochs included."""
    n, d = 4000, 32
    dq, tq = synth.quant_density(0.25), synth.quant_tightness(0.72)
    ctx = rac.RacContext.create_random(n, d, dq, tq, 1)
    assert ctx.layout == "sparse"
    orc = oracle.Oracle.from_synth(n, d, dq, tq, 1)
    root = synth.full_domains(np.full(n, d))
    g = ctx.enforce(root, removed_at=True)
    o = orc.rac(root)
    assert g[0] == o[0] and g[2] == o[2] and g[2] > 5
    assert np.array_equal(g[1], o[1]) and np.array_equal(g[3], o[3])


def test_c3_virtual_shards_vs_oracle(rac):
    """The sharded per-pass path (row blocks, TMA-staged D, device copy standing in
    for the all-gather) at C3 W-prop against the oracle's recurrence, for 2, 3
    and 8 blocks, root and seeded calls."""
    n, d = 2000, 32
    dq, tq = synth.quant_density(1.0), synth.quant_tightness(0.70)
    orc = oracle.Oracle.from_synth(n, d, dq, tq, 1)
    root = synth.full_domains(np.full(n, d))
    o = orc.rac(root)
    assert o[2] > 5
    for v in (2, 3, 8):
        ctx = rac.RacContext.create_random(n, d, dq, tq, 1, virtual_shards=v)
        g = ctx.enforce(root, removed_at=True)
        assert g[0] == o[0] and g[2] == o[2], v
        assert np.array_equal(g[1], o[1]) and np.array_equal(g[3], o[3]), v
        if o[0] == oracle.OK:
            s, x, _ = synth.w_seed(o[1], 3, v)
            gs = ctx.enforce_seeded(s, [x])
            os_ = orc.rac(s, with_epochs=False)
            assert (gs[0], gs[2]) == (os_[0], os_[2]) and np.array_equal(gs[1], os_[1]), v


def test_seeded_empty_list_every_path(rac, monkeypatch):
    """an empty seed list is no pass -- iterations 0, D
    unchanged, status from D_in (include/rac.h) -- on a FRESH context (no seed
    buffer allocated yet) of every path: the one-block path, the multi-CTA fused
    kernel, virtual shards, the NCCL leg; host and device (seeds_dev = NULL) calls."""
    import torch
    inst = synth.random_csp(300, 16, 0.6, 0.45, 4)
    orc = oracle.Oracle.from_instance(inst)
    st, root, _, _ = orc.rac(inst.full_domains())
    assert st == oracle.OK
    bad = root.copy()
    bad[7] = U64(0)  # an empty domain: status WIPEOUT with no pass
    makers = [("small", {}, "1e12"), ("fused", {}, "0"), ("vshard", {"virtual_shards": 3}, None),
              ("nccl_self", {"nccl_self": True}, None)]
    for name, kw, small in makers:
        if small is not None:  # one-block path for any size / never (read at create)
            monkeypatch.setenv("RAC_SMALL_BYTES", small)
        for D, exp in ((root, rac.RAC_OK), (bad, rac.RAC_WIPEOUT)):
            ctx = rac.RacContext.from_instance(inst, **kw)
            g = ctx.enforce_seeded(D, [])
            assert g[0] == exp and g[2] == 0 and np.array_equal(g[1], D), (name, g[0], g[2])
            ctx.close()
            ctx = rac.RacContext.from_instance(inst, **kw)
            din = torch.from_numpy(D.view(np.int64).copy()).cuda()
            dout = torch.zeros_like(din)
            its = torch.full((1,), -5, dtype=torch.int32, device="cuda")
            sts = torch.full((1,), -5, dtype=torch.int32, device="cuda")
            ctx.enforce_seeded_async(din, dout, its, sts, None, 0)
            torch.cuda.synchronize()
            assert int(sts.item()) == exp and int(its.item()) == 0, (name, "async")
            assert np.array_equal(dout.cpu().numpy().view(np.uint64), D), (name, "async")
            ctx.close()


def test_seeded_lists_sharded_and_small(rac):
    """Seed lists (several assigned variables at once, so the precondition holds
    for every non-seed column) on the sharded path (virtual shards, NCCL leg) and
    the one-block path: equal to the oracle's full recurrence (Prop. 2)."""
    checked = 0
    for k, inst in enumerate([synth.random_csp(120, 12, 0.6, 0.35, s) for s in range(1, 9)]):
        orc = oracle.Oracle.from_instance(inst)
        st, root, _, _ = orc.rac(inst.full_domains())
        if st != oracle.OK:
            continue
        rng = np.random.default_rng(k)
        D = root.copy()
        seeds = sorted(rng.choice(inst.n, size=3 + k % 5, replace=False).tolist())
        for x in seeds:
            vals = [a for a in range(64) if (int(D[x]) >> a) & 1]
            D[x] = U64(1) << U64(int(rng.choice(vals)))
        o = orc.rac(D, with_epochs=False)
        for kw in ({}, {"virtual_shards": 3}, {"nccl_self": True}):
            ctx = rac.RacContext.from_instance(inst, **kw)
            g = ctx.enforce_seeded(D, seeds + [seeds[0]])  # a duplicate seed tests once
            assert (g[0], g[2]) == (o[0], o[2]) and np.array_equal(g[1], o[1]), (k, kw)
            ctx.close()
            checked += 1
    assert checked >= 12


def test_wide_seeded_many_seeds(rac):
    """Wide seeded calls with more than 8 seeds (pass 1 takes the warp-per-row
    branch of wide_fused) and an out-of-range seed on the device path (skipped,
    as in rac_fused), at n=300, d=100 (t=0.9: a 4-pass consistent root): equal
    to O1w's full recurrence on the assigned state (Prop. 2)."""
    import torch
    from tests import _wide as WD
    n, d = 300, 100
    dq, tq = synth.quant_density(0.5), synth.quant_tightness(0.9)
    ctx = rac.RacContext.create_random(n, d, dq, tq, 2)
    wo = oracle.WideOracle.from_synth(n, d, dq, tq, 2)
    full = synth.full_domains_wide(np.full(n, d))
    st, root, _, _ = wo.rac(full, with_epochs=False)
    assert st == oracle.OK
    rng = np.random.default_rng(3)
    for trial in range(3):
        bits = WD.bits_of(root, n, wo.wq)
        seeds = rng.choice(n, size=12, replace=False)
        for x in seeds:
            vals = np.nonzero(bits[x])[0]
            keep = rng.choice(vals, size=max(1, len(vals) // 3), replace=False)
            bits[x, :] = False
            bits[x, keep] = True
        D = WD.words_of(bits)
        o = wo.rac(D, with_epochs=False)
        g = ctx.enforce_seeded(D, seeds.tolist())
        assert (g[0], g[2]) == (o[0], o[2]) and np.array_equal(g[1], o[1]), trial
        din = torch.from_numpy(D.view(np.int64).copy()).cuda()
        dout = torch.zeros_like(din)
        its = torch.zeros(1, dtype=torch.int32, device="cuda")
        sts = torch.zeros(1, dtype=torch.int32, device="cuda")
        sd = torch.from_numpy(np.concatenate([seeds, [n + 5, -3]]).astype(np.int32)).cuda()
        ctx.enforce_seeded_async(din, dout, its, sts, sd, int(sd.numel()))
        torch.cuda.synchronize()
        assert (int(sts.item()), int(its.item())) == (o[0], o[2])
        assert np.array_equal(dout.cpu().numpy().view(np.uint64), o[1])


@pytest.mark.parametrize("impl", ["cluster", "cluster1", "bs", "state"])
def test_batched_impls_corpus(rac, impl, monkeypatch):
    """Every batched kernel -- one 32-state word per cluster (default, cluster
    sizes 4 and 1), the r01 bit-sliced kernel (RAC_BATCH_IMPL=bs) and one block
    per state (RAC_BATCH_IMPL=state) -- equals the oracle state by state on
    mixed corpora (W-rand states, stop and full modes, empty rows)."""
    import torch
    if impl in ("bs", "state"):
        monkeypatch.setenv("RAC_BATCH_IMPL", impl)
    if impl == "cluster1":
        monkeypatch.setenv("RAC_BATCH_CL", "1")
    for k, inst in enumerate(I.random_corpus(40, seed0=301, n_range=(5, 60), d_range=(1, 16))):
        orc = oracle.Oracle.from_instance(inst)
        ctx = rac.RacContext.from_instance(inst)
        S = 37 + k
        states = np.stack([synth.w_rand(inst.dom, 0.8, seed=1000 * k + s) for s in range(S)])
        states[::9, 0] = U64(0)
        din = torch.from_numpy(states.view(np.int64).copy()).cuda()
        for full in (False, True):
            dout = torch.zeros_like(din)
            its = torch.zeros(S, dtype=torch.int32, device="cuda")
            sts = torch.zeros(S, dtype=torch.int32, device="cuda")
            ctx.enforce_batch(S, din, dout, its, sts, full=full)
            torch.cuda.synchronize()
            out = dout.cpu().numpy().view(np.uint64)
            for s in range(S):
                o = orc.rac(states[s], full=full, with_epochs=False)
                assert (int(sts[s]), int(its[s])) == (o[0], o[2]), (k, s, full)
                assert np.array_equal(out[s], o[1]), (k, s, full)
