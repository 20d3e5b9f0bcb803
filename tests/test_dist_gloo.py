"""N > 1 host logic on CPU with the gloo backend (world size 2).

* the NCCL unique id produced by librac on rank 0 reaches every rank intact;
* max-over-ranks reduction of timings;
* the row blocks of librac's rac_shard_range partition the variables;
* the sharded exchange protocol (each rank tests only its row block against the
  replicated D_{t-1}, writes its slice of D_t, all-gather with equal padded
  counts, every rank derives `changed`/`wipe` from the gathered vector) reaches
  the same (status, D, iterations) as the single-process oracle on every rank.
  The per-block pass is computed with the oracle's row test (test code); the
  CUDA implementation of the same protocol is checked on one GPU by the
  virtual-shard parity tests.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sharded_protocol(n, d, dq, tq, seed, d_in, rank, world, full=False):
    import oracle
    from paper_2407_11388_b200 import rac
    lo, hi = rac.rac_shard_range(n, world, rank)
    blk = (n + world - 1) // world
    cur = np.array(d_in, dtype=np.uint64)
    it = 0
    while True:
        it += 1
        mine = np.zeros(blk, dtype=np.uint64)
        for x in range(lo, hi):
            w = int(cur[x])
            for a in range(d):
                if (w >> a) & 1 and not oracle.row_supported_synth(n, d, dq, tq, seed, x, a, cur):
                    w &= ~(1 << a)
            mine[x - lo] = w
        gathered = [torch.zeros(blk, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(mine.view(np.int64)))
        nxt = torch.cat(gathered).numpy().view(np.uint64)[:n].copy()
        changed = bool(np.any(nxt != cur))
        wipe = bool(np.any(nxt == 0))
        cur = nxt
        if wipe and not full:
            return 1, cur, it
        if not changed:
            return (1 if wipe else 0), cur, it


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2407_11388_b200 import dist as rdist
        from paper_2407_11388_b200 import rac
        res = {}
        uid = rdist.nccl_unique_id()
        res["uid"] = uid
        res["max"] = rdist.max_over_ranks(float(rank + 1))
        res["range"] = rac.rac_shard_range(37, world, rank)
        runs = []
        for (n, d, p, t, seed, keep) in [(23, 6, 0.6, 0.45, 1, 1.0), (30, 5, 1.0, 0.5, 2, 0.9),
                                         (17, 4, 0.4, 0.6, 3, 0.85), (26, 8, 0.8, 0.55, 4, 0.9)]:
            dq, tq = synth.quant_density(p), synth.quant_tightness(t)
            d_in = synth.w_rand(np.full(n, d), keep, seed)
            for full in (False, True):
                st, dd, it = _sharded_protocol(n, d, dq, tq, seed, d_in, rank, world, full)
                o = oracle.Oracle.from_synth(n, d, dq, tq, seed).rac(d_in, full=full, with_epochs=False)
                runs.append((st == o[0], bool(np.array_equal(dd, o[1])), it == o[2], it))
        res["runs"] = runs
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0]["uid"] == out[1]["uid"] and len(out[0]["uid"]) == 128
    assert out[0]["max"] == out[1]["max"] == 2.0
    (a0, b0), (a1, b1) = out[0]["range"], out[1]["range"]
    assert a0 == 0 and b0 == a1 and b1 == 37
    for r in (0, 1):
        for ok_st, ok_d, ok_it, it in out[r]["runs"]:
            assert ok_st and ok_d and ok_it
    # every rank made the same decisions
    assert [x[3] for x in out[0]["runs"]] == [x[3] for x in out[1]["runs"]]
    assert max(x[3] for x in out[0]["runs"]) > 1
