"""The multi-process peer-memory path (RAC_OPT_PEER over CUDA IPC): two processes,
a gloo process group for the setup tokens (dist.connect_peers all-gathers the
regions' IPC handles), both ranks on cuda:0 (the gpurun box has one GPU; the
two contexts are time-sliced, so each cross-rank barrier also waits for a
context switch).  Every rank must return the oracle's (status, D, iterations)
-- the path bench.py would take with --exchange peer on several GPUs.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RAC_PEER_TIMEOUT_MS="20000")
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_2407_11388_b200 import dist as rdist
        from paper_2407_11388_b200 import rac
        torch.cuda.set_device(0)
        res = []
        for (n, d, p, t) in ((60, 8, 0.6, 0.45), (300, 16, 0.5, 0.5)):
            dq, tq = synth.quant_density(p), synth.quant_tightness(t)
            ctx = rac.RacContext.create_random(n, d, dq, tq, 3, device=0, rank=rank, world=world, peer=True,
                                               max_ctas=8)
            rdist.connect_peers(ctx)
            for k in range(3):
                d_in = synth.w_rand(np.full(n, d), 0.9, 10 + k)
                st, d_out, it = ctx.enforce(d_in)
                res.append((n, k, int(st), [int(v) for v in d_out], int(it)))
            dist.barrier()
            ctx.close()
        q.put((rank, res))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, "error: %r" % (e,)))
    finally:
        dist.destroy_process_group()


def test_peer_ipc_two_processes():
    import torch.multiprocessing as mp

    import oracle
    import synth
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, res = q.get(timeout=600)
        out[r] = res
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(out[r], str), out[r]
    for (n, d, p, t) in ((60, 8, 0.6, 0.45), (300, 16, 0.5, 0.5)):
        orc = oracle.Oracle.from_synth(n, d, synth.quant_density(p), synth.quant_tightness(t), 3)
        for k in range(3):
            o = orc.rac(synth.w_rand(np.full(n, d), 0.9, 10 + k), with_epochs=False)
            for r in range(world):
                g = [x for x in out[r] if x[0] == n and x[1] == k][0]
                assert g[2] == o[0] and g[4] == o[2], (n, k, r, g[2], o[0], g[4], o[2])
                assert np.array_equal(np.array(g[3], dtype=np.uint64), o[1]), (n, k, r)
