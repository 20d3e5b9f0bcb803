"""Row-sharded multi-GPU enforcement with the peer-memory exchange (RAC_OPT_PEER).

The gpurun box has one GPU, so the ranks here are driven by ONE process on ONE
device (rac_connect_peers_local): each rank is its own context holding only its
row block, its own stream and its own persistent kernel (max_ctas keeps the
ranks' grids co-resident).  Everything the multi-GPU protocol does runs for real
-- the removal words written into the peers' buffers, the system-scope
arrival words, the cross-rank barrier, the global pass counter across launches
-- only the transport is local memory instead of NVLink.  Every rank must return
the oracle's (status, D, iterations) (include/rac.h "Multi-GPU"; the exchange is
not in the paper, it is BASELINE.json north_star's sharding).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
import synth
from tests import _instances as I

pytestmark = pytest.mark.gpu

# a rank that never arrives must not hang the box: fail fast instead
os.environ.setdefault("RAC_PEER_TIMEOUT_MS", "5000")


@pytest.fixture(scope="module")
def rac():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2407_11388_b200 import rac as r
    return r


def make_group(rac, world, make, max_ctas):
    ctxs = [make(r, world, max_ctas) for r in range(world)]
    regions = [c.peer_region() for c in ctxs]
    for c in ctxs:
        c.connect_peers_local(regions, [0] * world)
    return ctxs


def run_group(ctxs, d_in, full=False, seeds=None):
    """Enqueue one enforcement per rank on its own stream, then wait for all."""
    import torch
    streams = [torch.cuda.Stream() for _ in ctxs]
    src = torch.from_numpy(np.ascontiguousarray(d_in, dtype=np.uint64).view(np.int64).copy()).cuda()
    ins = [src.clone() for _ in ctxs]
    outs = [torch.zeros_like(src) for _ in ctxs]
    its = [torch.full((1,), -9, dtype=torch.int32, device="cuda") for _ in ctxs]
    sts = [torch.full((1,), -9, dtype=torch.int32, device="cuda") for _ in ctxs]
    sd = None
    if seeds is not None:
        sd = torch.from_numpy(np.asarray(seeds, dtype=np.int32)).cuda()
    torch.cuda.synchronize()
    for r, c in enumerate(ctxs):
        if seeds is None:
            c.enforce_async(ins[r], outs[r], its[r], sts[r], full=full, stream=streams[r])
        else:
            c.enforce_seeded_async(ins[r], outs[r], its[r], sts[r], sd, int(sd.numel()), full=full,
                                   stream=streams[r])
    torch.cuda.synchronize()
    return [(int(sts[r].item()), outs[r].cpu().numpy().view(np.uint64).copy(), int(its[r].item()))
            for r in range(len(ctxs))]


def run_group_epochs(ctxs, d_in, full=False):
    """As run_group, with every rank asking for the removal epochs."""
    import torch
    n = ctxs[0].n
    streams = [torch.cuda.Stream() for _ in ctxs]
    src = torch.from_numpy(np.ascontiguousarray(d_in, dtype=np.uint64).view(np.int64).copy()).cuda()
    ins = [src.clone() for _ in ctxs]
    outs = [torch.zeros_like(src) for _ in ctxs]
    its = [torch.full((1,), -9, dtype=torch.int32, device="cuda") for _ in ctxs]
    sts = [torch.full((1,), -9, dtype=torch.int32, device="cuda") for _ in ctxs]
    rems = [torch.full((n * 64,), -9, dtype=torch.int32, device="cuda") for _ in ctxs]
    torch.cuda.synchronize()
    for r, c in enumerate(ctxs):
        c.enforce_async(ins[r], outs[r], its[r], sts[r], rems[r], full=full, stream=streams[r])
    torch.cuda.synchronize()
    return [(int(sts[r].item()), outs[r].cpu().numpy().view(np.uint64).copy(), int(its[r].item()),
             rems[r].cpu().numpy().reshape(n, 64)) for r in range(len(ctxs))]


def check(res, o, what):
    for r, g in enumerate(res):
        assert g[0] == o[0], (what, r, "status", g[0], o[0])
        assert g[2] == o[2], (what, r, "iterations", g[2], o[2])
        assert np.array_equal(g[1], o[1]), (what, r, "d_out")


def test_peer_corpus(rac):
    """SPEC-shaped random corpus over 2, 3 and 4 ranks (including ranks whose row
    block is empty when n < world), both stop modes, two inputs per instance."""
    for k, inst in enumerate(I.random_corpus(36, seed0=211)):
        world = 2 + k % 3
        orc = oracle.Oracle.from_instance(inst)
        ctxs = make_group(rac, world, lambda r, w, m: rac.RacContext.from_instance(
            inst, rank=r, world=w, peer=True, max_ctas=m), max_ctas=4)
        for j, d_in in enumerate((inst.full_domains(), synth.w_rand(inst.dom, 0.85, seed=k))):
            for full in (False, True):
                check(run_group(ctxs, d_in, full), orc.rac(d_in, full=full, with_epochs=False), (k, j, full))


@pytest.mark.parametrize("world", [2, 4])
def test_peer_c3_prop_repeated(rac, world):
    """C3 shape (n=2000, d=32, density 1) at t=0.70 (about 13 passes) sharded over
    2 and 4 ranks; three launches back to back with different inputs, so the
    global pass counter, the rotating buffers and the arrival words carry over
    between launches."""
    dq, tq = synth.quant_density(1.0), synth.quant_tightness(0.70)
    orc = oracle.Oracle.from_synth(2000, 32, dq, tq, 1)
    ctxs = make_group(rac, world, lambda r, w, m: rac.RacContext.create_random(
        2000, 32, dq, tq, 1, rank=r, world=w, peer=True, max_ctas=m), max_ctas=128 // world)
    root = synth.full_domains(np.full(2000, 32))
    inputs = [root, synth.w_rand(np.full(2000, 32), 0.9, seed=3), root]
    for j, d_in in enumerate(inputs):
        o = orc.rac(d_in, with_epochs=False)
        check(run_group(ctxs, d_in), o, (world, j))
    assert o[2] > 3


def test_peer_seeded(rac):
    """Seeded enforcement (Alg. 1 with @changed = seeds) through the peer
    path: equal to the oracle's O5 on W-seed inputs."""
    for k, inst in enumerate(I.random_corpus(12, seed0=223, n_range=(6, 40), d_range=(2, 9))):
        orc = oracle.Oracle.from_instance(inst)
        ctxs = make_group(rac, 2, lambda r, w, m: rac.RacContext.from_instance(
            inst, rank=r, world=w, peer=True, max_ctas=m), max_ctas=4)
        root = orc.rac(inst.full_domains(), with_epochs=False)
        if root[0] != oracle.OK:
            continue
        for j in range(3):
            ds, x, _ = synth.w_seed(root[1], k, j)
            o = orc.rac_seeded(ds, [x], with_epochs=False)
            check(run_group(ctxs, ds, seeds=[x]), o, (k, j))


def test_peer_api_errors(rac):
    inst = synth.random_csp(10, 4, 0.8, 0.3, 2)
    with pytest.raises(rac.RacError) as ei:  # peer exchange needs world >= 2
        rac.RacContext.from_instance(inst, peer=True)
    assert ei.value.code == rac.RAC_EINVAL
    c0 = rac.RacContext.from_instance(inst, rank=0, world=2, peer=True, max_ctas=2)
    with pytest.raises(rac.RacError) as ei:  # not connected yet
        c0.enforce(inst.full_domains())
    assert ei.value.code == rac.RAC_EINVAL
    with pytest.raises(rac.RacError) as ei:  # regions[rank] must be this context's
        c0.connect_peers_local([1234, 5678], [0, 0])
    assert ei.value.code == rac.RAC_EINVAL
    assert len(c0.peer_handle()) == rac.RAC_IPC_HANDLE_BYTES


def test_peer_timeout_reports_epeer(rac, monkeypatch):
    """A rank whose peer never launches gives up after RAC_PEER_TIMEOUT_MS and
    reports RAC_EPEER (no hang); the context is then unusable."""
    monkeypatch.setenv("RAC_PEER_TIMEOUT_MS", "300")
    inst = synth.random_csp(30, 6, 1.0, 0.5, 5)
    c0, c1 = make_group(rac, 2, lambda r, w, m: rac.RacContext.from_instance(
        inst, rank=r, world=w, peer=True, max_ctas=m), max_ctas=2)
    with pytest.raises(rac.RacError) as ei:
        c0.enforce(inst.full_domains())  # rank 1 never runs
    assert ei.value.code == rac.RAC_EPEER
    with pytest.raises(rac.RacError) as ei:
        c0.enforce(inst.full_domains())
    assert ei.value.code == rac.RAC_ESTATE


def test_peer_removal_epochs(rac):
    """Removal epochs on the peer path (include/rac.h rac_enforce_ex: with world > 1
    every rank receives all epochs): each rank's epochs equal the oracle's, for
    2, 3 and 4 ranks, stop and full modes, with calls that do and do not ask for
    epochs interleaved (the double-buffered epoch arrays switch parity only on
    calls that ask)."""
    for k, inst in enumerate(I.random_corpus(18, seed0=307, n_range=(8, 40), d_range=(2, 10))):
        world = 2 + k % 3
        orc = oracle.Oracle.from_instance(inst)
        ctxs = make_group(rac, world, lambda r, w, m: rac.RacContext.from_instance(
            inst, rank=r, world=w, peer=True, max_ctas=m), max_ctas=4)
        for j in range(3):
            d_in = synth.w_rand(inst.dom, 0.85, seed=100 * k + j)
            full = j == 1
            o = orc.rac(d_in, full=full)
            for r, g in enumerate(run_group_epochs(ctxs, d_in, full)):
                assert (g[0], g[2]) == (o[0], o[2]) and np.array_equal(g[1], o[1]), (k, j, r)
                assert np.array_equal(g[3], o[3]), (k, j, r, "epochs")
            check(run_group(ctxs, d_in), orc.rac(d_in, with_epochs=False), (k, j, "no epochs"))
    # C3 shape, 13 passes, 2 ranks: certified epochs on every rank
    dq, tq = synth.quant_density(1.0), synth.quant_tightness(0.70)
    ctxs = make_group(rac, 2, lambda r, w, m: rac.RacContext.create_random(
        2000, 32, dq, tq, 1, rank=r, world=w, peer=True, max_ctas=m), max_ctas=64)
    root = synth.full_domains(np.full(2000, 32))
    for g in run_group_epochs(ctxs, root):
        assert oracle.certify_trajectory_synth(2000, 32, dq, tq, 1, root, g[1], g[3], g[2], g[0]) == 0
