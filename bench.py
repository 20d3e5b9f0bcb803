#!/usr/bin/env python
"""bench.py -- RAC enforcement throughput on B200 (BASELINE.json metric:
"AC enforcements/sec and relation-tensor GB/s/iter vs HBM peak at 1/2/4/8 B200").

One step = one full enforcement D_in -> D_ac (every §8(a) row: D staged in
smem, support test over the packed relation masks, AND over C_x, device-side
loop control to the fixpoint; with N > 1 the per-pass all-gather over NCCL).
The instance is packed once before timing (rac_create is not per step).

Default workload (configs[2], C3): random binary CSP n=2000, d=32, density
1.0, tightness 0.5, root enforcement (W-stream: one pass reads every byte of
the 512 MB mask tensor; inputs larger than the 126 MB L2, so no flush).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3-stream|c3-prop|c2-root|c1-seed|c4-stream|c5-batch]
  python bench.py --impl reference ...   # the CPU oracle on the same workload

Prints ONE JSON line (rank 0).  Timing: CUDA events on the launching stream,
barrier + synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402  (input generation only)

METRIC = "AC enforcements/sec"
UNIT = "enforcements/s"
FALLBACK_HBM = 6650.0

WORKLOADS = {
    # name: (n, d, density, tightness, seed, D_in kind, description)
    "c3-stream": (2000, 32, 1.0, 0.5, 1, "root",
                  "C3 W-stream: random binary CSP n=2000, d=32, density 1.0, tightness 0.5; root enforcement "
                  "(full domains; 1 pass over all 512 MB of masks)"),
    "c3-prop": (2000, 32, 1.0, 0.70, 1, "root",
                "C3 W-prop: n=2000, d=32, density 1.0, tightness 0.70; root enforcement (~10 passes, consistent)"),
    "c2-root": (500, 20, 1.0, 0.3, 1, "root",
                "C2: n=500, d=20, complete graph, tightness 0.3; root enforcement (20 MB, L2-resident)"),
    "c1-seed": (20, 8, 0.5, 0.4, 1, "seed",
                "C1 W-seed: n=20, d=8, density 0.5, tightness 0.4; D_ac(root) with one seeded assignment, "
                "seeded enforcement (Alg. 1 tensorAC(Vars, [idx]), P:392)"),
    "c3-seed": (2000, 32, 1.0, 0.5, 1, "seed",
                "C3 W-seed: n=2000, d=32, density 1.0, tightness 0.5; D_ac(root) with one seeded assignment, "
                "seeded enforcement (Alg. 1 tensorAC(Vars, [idx]), P:392)"),
    "c3s-stream": (4000, 32, 0.25, 0.5, 1, "root",
                   "NEXT-3 sparse: n=4000, d=32, density 0.25 (paper's density grid P:236), tightness 0.5; root "
                   "enforcement (1 pass; sparse arc blocks, 512 MB of declared masks vs 2 GB dense)"),
    "c3s-prop": (4000, 32, 0.25, 0.72, 1, "root",
                 "NEXT-3 sparse: n=4000, d=32, density 0.25, tightness 0.72; root enforcement (propagating)"),
    "c4-stream": (8000, 64, 1.0, 0.5, 1, "root",
                  "C4 W-stream: n=8000, d=64, density 1.0, tightness 0.5; root enforcement (32.8 GB of masks)"),
    "w128-stream": (2000, 128, 1.0, 0.5, 1, "root",
                    "NEXT-4 wide domains: n=2000, d=128 (2 words per variable), density 1.0, tightness 0.5; root "
                    "enforcement (1 pass over 8.19 GB of 16-byte masks)"),
    "w128-prop": (2000, 128, 1.0, 0.93, 1, "root",
                  "NEXT-4 wide domains: n=2000, d=128, density 1.0, tightness 0.93; root enforcement "
                  "(propagating: wipeout after 3 passes)"),
    "w256-stream": (1000, 256, 1.0, 0.5, 1, "root",
                    "NEXT-4 wide domains: n=1000, d=256 (4 words per variable), density 1.0, tightness 0.5; root "
                    "enforcement (1 pass over 8.19 GB of 32-byte masks)"),
    "w128-batch": (200, 128, 0.8, 0.95, 1, "wrand",
                   "NEXT-4 wide batched: 1024 W-rand states (keep 0.8) on n=200, d=128, density 0.8, tightness "
                   "0.95; one batched enforcement per step (tensor-core passes: tcgen05 fp8 over every column, "
                   "per-state loop control)"),
    "c5-batch": (200, 16, 0.8, 0.3, 1, "dive",
                 "C5: 1024 W-dive states (search-tree nodes) on n=200, d=16, density 0.8, tightness 0.3; "
                 "one batched seeded enforcement per step (each state seeded with its assigned variable)"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def pass_bytes(live0, remd, iters, nbr_count, chg, d):
    """Per-enforcement byte counts from the removal epochs (see the comment at
    the call site).  live0: [n, d] bool live rows of D_in; remd: [n, d] epoch
    of each removal (0 = kept); chg: [n] bool variables tested in pass 1;
    nbr_count(chg) -> [n] count of declared c_xy with y in chg.  Returns
    (live rows per pass, must-read bytes, full-check bytes)."""
    live_per_pass, alg, full = [], 0.0, 0.0
    for t in range(1, iters + 1):
        alive = live0 & ((remd == 0) | (remd >= t))
        gone = (live0 & (remd == t)).sum(axis=1)
        lv = alive.sum(axis=1)
        nb = nbr_count(chg)
        live_per_pass.append(int(lv.sum()))
        full += float((lv * nb).sum()) * d / 8.0
        alg += (float(((lv - gone) * nb).sum()) + float((gone * (nb > 0)).sum())) * d / 8.0
        chg = (remd == t).any(axis=1)
    return live_per_pass, alg, full


def algorithmic_bytes(n, d, density_present_deg, live_per_pass):
    """Σ_t Σ_x |D_{t-1}(x)| · Σ_{y∈C_x} d_y / 8; uniform d."""
    return sum(live * deg * d for live, deg in zip(live_per_pass, density_present_deg)) / 8.0


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        self.t0 = time.time()

    def stop(self):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
        self.f.flush()
        rows = []
        try:
            with open(self.f.name) as fh:
                for line in fh:
                    parts = [s.strip() for s in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        finally:
            os.unlink(self.f.name)
        return rows

    @staticmethod
    def summarize(rows):
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ----------------------------------------------------------------------------- GPU arm
def run_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2407_11388_b200 import rac

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n, d, dens, tight, seed, kind, desc = WORKLOADS[args.workload]
    dq, tq = synth.quant_density(dens), synth.quant_tightness(tight)
    uid = None
    peer = world > 1 and args.exchange == "peer"
    if world > 1 and not peer:
        obj = [rac.rac_get_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    t0 = time.time()
    max_ctas = 0
    if os.environ.get("RAC_BENCH_SHARED_GPU") == "1" and world > 1:
        max_ctas = max(1, torch.cuda.get_device_properties(local_rank).multi_processor_count // world)
    def make_ctx():
        return rac.RacContext.create_random(n, d, dq, tq, seed, device=local_rank, rank=rank, world=world,
                                            nccl_unique_id=uid, peer=peer, max_ctas=max_ctas)

    ctx = make_ctx()
    if peer:
        # the regions' CUDA IPC handles travel over the process group; the
        # per-pass exchange then runs inside the one persistent kernel
        from paper_2407_11388_b200 import dist as rdist
        rdist.connect_peers(ctx)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    full = synth.full_domains(np.full(n, d)) if d <= 64 else synth.full_domains_wide(np.full(n, d))
    stream = torch.cuda.current_stream()

    # --- D_in
    seed_vars = None
    if kind == "seed":
        st, root, _ = ctx.enforce(full)
        d_in, sx, _ = synth.w_seed(root, seed)
        seed_vars = np.array([sx], dtype=np.int32)
    else:
        d_in = full
    batched = kind in ("dive", "wrand")
    S = args.states if batched else 1
    if kind == "dive":
        st, root, _ = ctx.enforce(full)
        states, svars = synth.dive_states(root, lambda D: ctx.enforce(D)[:2], S, seed=seed, return_seeds=True)
        din_h = np.stack(states)
        seed_vars = np.asarray(svars, dtype=np.int32)
    elif kind == "wrand":
        din_h = wrand_states(n, d, S)
    else:
        din_h = d_in[None, :]

    # --- instrumentation run (outside the timed region): iterations, status, live rows per pass
    if batched:
        res = [ctx.enforce(din_h[s], removed_at=True) for s in range(S)]
        iters_list = [r[2] for r in res]
        instr = {"iterations_mean": float(np.mean(iters_list)), "iterations_max": int(np.max(iters_list)),
                 "wipeout_frac": float(np.mean([r[0] == 1 for r in res]))}
        alg_bytes = None
        # Algorithmic support tests of Alg. 1 per state (seeded call):
        # pass t tests every live (x,a) against the declared c_xy whose y changed in
        # pass t-1 (the state's assigned variable in pass 1).  The removal epochs come
        # from the plain recurrence, whose trajectory the seeded call follows (DESIGN R12).
        xs_p, ys_p = synth.present_pairs(n, dq, seed)
        alg_tests = 0
        for s_i, r in enumerate(res):
            remd = r[3][:, :d]
            live0 = _live_bits(din_h[s_i], n, d)
            chg = np.zeros(n, dtype=bool)
            if seed_vars is not None:
                chg[seed_vars[s_i]] = True
            else:
                chg[:] = True
            for t in range(1, r[2] + 1):
                lv = (live0 & ((remd == 0) | (remd >= t))).sum(axis=1)
                nb = np.zeros(n, dtype=np.int64)
                np.add.at(nb, xs_p, chg[ys_p].astype(np.int64))
                np.add.at(nb, ys_p, chg[xs_p].astype(np.int64))
                alg_tests += int((lv * nb).sum())
                chg = (remd == t).any(axis=1)
        instr["support_tests"] = alg_tests
    else:
        # removal epochs on every rank (with world > 1 they are gathered with the exchange)
        stt, dout, it, rem = ctx.enforce(din_h[0], removed_at=True)
        instr = {"iterations": it, "status": "OK" if stt == 0 else "WIPEOUT"}
        # Algorithmic bytes of Alg. 1: pass t tests every live (x,a)
        # against the constraints c_xy with y changed in pass t-1 (all y in
        # pass 1 of a root call; the seed variables in pass 1 of a seeded call):
        #   full_t = Σ_x |D_{t-1}(x)| · |{y ∈ C_x : y ∈ changed_{t-1}}| · d / 8
        # (SURVEY §8(d)'s full-check figure).  The roofline charges the bytes a
        # correct pass MUST read: a row kept by pass t reads every tested mask
        # (any unread one could be the empty support set), a row removed at t
        # needs only its witness (Lemma 1: one mask, d/8 bytes).  Both
        # kernels stop reading a row at its first failed test, so the full figure
        # over-counts removal passes (w128-prop: 18.3 GB full, 12.7 GB DRAM read).
        # One-pass workloads remove nothing: both figures are the same.
        if rem is not None:
            remd = rem[:, :d]
            live0 = _live_bits(din_h[0], n, d)
            if dens >= 1.0:
                def nbr_count(chg):
                    return chg.sum() - chg.astype(np.int64)
            else:
                xs, ys = synth.present_pairs(n, dq, seed)

                def nbr_count(chg):
                    c = np.zeros(n, dtype=np.int64)
                    np.add.at(c, xs, chg[ys].astype(np.int64))
                    np.add.at(c, ys, chg[xs].astype(np.int64))
                    return c
            chg = np.zeros(n, dtype=bool)
            if kind == "seed":
                chg[seed_vars] = True
            else:
                chg[:] = True
            live_per_pass, alg_bytes, full_bytes = pass_bytes(live0, remd, it, nbr_count, chg, d)
            instr["full_test_bytes"] = full_bytes
        else:
            live_per_pass = [int(_live_bits(din_h[0], n, d).sum())] + [0] * (it - 1)
            alg_bytes = live_per_pass[0] * (n - 1) * d / 8.0 if it == 1 else None
        instr["live_rows_per_pass"] = live_per_pass

    # --- device buffers
    din = torch.from_numpy(din_h.view(np.int64).copy()).to(dev)
    dout = torch.zeros_like(din)
    its = torch.zeros(S, dtype=torch.int32, device=dev)
    sts = torch.zeros(S, dtype=torch.int32, device=dev)
    sv = torch.from_numpy(seed_vars).to(dev) if seed_vars is not None else None

    def step(st=None):
        st = st if st is not None else stream
        if kind == "dive":
            ctx.enforce_batch_seeded(S, din, dout, its, sts, sv, stream=st)
        elif kind == "wrand":
            ctx.enforce_batch(S, din, dout, its, sts, stream=st)
        elif kind == "seed":
            ctx.enforce_seeded_async(din, dout, its, sts, sv, 1, stream=st)
        else:
            ctx.enforce_async(din, dout, its, sts, stream=st)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = ctx.last_launch_count
    ref = (dout.clone(), its.clone(), sts.clone())

    # Single-GPU paths with no host loop are captured into a CUDA graph of G
    # steps (G divides K), so small enforcements are timed without the host's
    # per-call launch overhead (the launch-bound inner loop in a graph); the
    # graph's results are checked against the eager ones.  Multi-GPU paths (and
    # any path whose capture fails) run eagerly.
    graph, G, launch_mode = None, 1, "eager"
    if world == 1 and ctx.path not in ("sharded", "peer") and kind != "wrand" and \
            os.environ.get("RAC_BENCH_GRAPH", "1") == "1":  # the wide tensor-core batch reads a flag per pass
        G = max(g for g in range(1, min(args.steps, 50) + 1) if args.steps % g == 0)
        try:
            cs = torch.cuda.Stream()
            cs.wait_stream(stream)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=cs):
                for _ in range(G):
                    step(cs)
            for _ in range(max(1, args.warmup // G)):
                gr.replay()
            torch.cuda.synchronize()
            if not (torch.equal(dout, ref[0]) and torch.equal(its, ref[1]) and torch.equal(sts, ref[2])):
                raise RuntimeError("graph replay differs from the eager result")
            graph, launch_mode = gr, "CUDA graph of %d steps (captured async calls; results checked)" % G
        except Exception as e:  # report, and run eagerly
            launch_mode = "eager (graph capture failed: %s)" % (repr(e)[:120],)
            graph, G = None, 1
            torch.cuda.synchronize()
            if isinstance(e, rac.RacError):  # a CUDA error inside librac leaves the context unusable
                ctx.close()
                ctx = make_ctx()
                for _ in range(args.warmup):
                    step()
                torch.cuda.synchronize()

    clocks = ClockSampler(local_rank)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    R = args.steps // G
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(R + 1)]
    evs[0].record(stream)
    for k in range(R):
        if graph is not None:
            graph.replay()
        else:
            step()
        evs[k + 1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    per_step = [evs[k].elapsed_time(evs[k + 1]) / G for k in range(R)]
    total_ms = evs[0].elapsed_time(evs[-1])
    # clocks: keep the sampler running for at least ~1.5 s of the same step loop
    soak = 0
    while time.time() - clocks.t0 < 1.5:
        if graph is not None:
            graph.replay()
        else:
            step()
        soak += G
        if soak % 64 < G:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    crow = clocks.stop()
    clk = ClockSampler.summarize(crow)
    clk["window"] = "timed region" + (" + %d extra steps of the same loop (>=1.5 s sampling window)" % soak if soak
                                      else "")

    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())

    # --- e2e: the public host-buffer call, H2D + D2H inside the timed region
    e2e = None
    if not batched:
        host_call = (lambda: ctx.enforce_seeded(din_h[0], seed_vars)) if kind == "seed" else \
            (lambda: ctx.enforce(din_h[0]))
        for _ in range(3):
            host_call()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        reps = max(10, min(args.steps, 2000))
        torch.cuda.synchronize()
        t_wall = time.perf_counter()
        e0.record(stream)
        for _ in range(reps):
            host_call()
        e1.record(stream)
        torch.cuda.synchronize()
        wall_ms = (time.perf_counter() - t_wall) * 1e3
        if world > 1:
            t = torch.tensor([wall_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            wall_ms = float(t.item())
        e2e = {"value": reps / (wall_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": n * ctx.wq * 8 + (4 if kind == "seed" else 0),
               "d2h_bytes_per_step": n * ctx.wq * 8 + 8,
               "how": ("rac_enforce_seeded" if kind == "seed" else "rac_enforce") + " (host buffers; pinned staging, H2D + enforcement + D2H + sync per call), "
                      "host wall clock over %d calls, max over ranks" % reps}
    else:
        # batched: host states -> device -> batch enforcement -> results back, per step
        h_in = torch.from_numpy(din_h.view(np.int64).copy()).pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()
        h_st = torch.empty(S, dtype=torch.int32).pin_memory()
        reps = max(5, min(args.steps, 200))
        torch.cuda.synchronize()
        t_wall = time.perf_counter()
        for _ in range(reps):
            din.copy_(h_in, non_blocking=True)
            step()
            h_out.copy_(dout, non_blocking=True)
            h_st.copy_(sts, non_blocking=True)
            torch.cuda.synchronize()
        wall_ms = (time.perf_counter() - t_wall) * 1e3
        e2e = {"value": reps * S / (wall_ms / 1e3), "unit": "states/s", "h2d_bytes_per_step": int(din_h.nbytes),
               "d2h_bytes_per_step": int(din_h.nbytes) + S * 4,
               "how": "pinned host states -> device, rac_enforce_batch, D_out + status -> pinned host, sync"}

    ms_per_step = total_ms / args.steps
    if batched:
        value = S * args.steps / (total_ms / 1e3)
        unit = "states/s"
        metric = "AC enforcements/sec (batched search-tree states)" if kind == "dive" else \
            "AC enforcements/sec (batched states)"
    else:
        value = args.steps / (total_ms / 1e3)
        unit = UNIT
        metric = METRIC

    peak, peak_src = measured_peaks()
    roofline = None
    l2_roof = None
    if kind == "wrand":
        # Wide tensor-core batch: every pass is a dense tcgen05 contraction of
        # ALL states against every column (K = 128 per column, fp8 e4m3 0/1
        # operands by default, fp32 counts): 2 x rows x n x 128 x S_pad FLOPs per
        # pass, for as many passes as the slowest state runs.  Peak: the measured
        # dense bf16 cuBLAS figure x 2 for fp8 (x 1 for f16), MEASURED_PEAKS.json.
        kern_ms = statistics.median(per_step)
        s_pad = (S + 255) // 256 * 256
        passes = int(instr["iterations_max"])
        flops = 2.0 * n * d * n * 128 * s_pad * passes
        ach_tf = flops / (kern_ms / 1e3) / 1e12
        f16 = os.environ.get("RAC_WIDE_TC") == "f16"  # fp8 e4m3 operands by default (librac)
        try:
            pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
            peak_tf, src = float(pk["bf16_tflops"]), "measured dense bf16 cuBLAS (MEASURED_PEAKS.json bf16_tflops, burst)"
        except Exception:
            peak_tf, src = 1590.0, "fallback (B200_PROFILING.md)"
        if not f16:  # fp8: the measured bf16 figure x the nominal fp8 / bf16 ratio (4.5 / 2.25)
            peak_tf, src = 2.0 * peak_tf, src + " x 2 (nominal dense fp8 / bf16 ratio, B200_PROFILING.md)"
        roofline = {"bound": "tensor", "achieved": round(ach_tf, 1), "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": round(ach_tf / peak_tf, 4), "traffic": None, "kernel": "wide_tc_pass (+ wide_tc_update)",
                    "flops_per_launch": flops, "passes": passes, "launch_ms_median": round(kern_ms, 5),
                    "algorithmic_tests_per_launch": instr["support_tests"],
                    "tests_per_s": round(instr["support_tests"] / (kern_ms / 1e3), 1), "peak_source": src}
    if kind == "dive":
        # Bit-sliced batched pass (rac_batch_cl; rac_batch_bs in r01): a support test of (x,a) against
        # c_xy for 32 states is ceil(d/4) nibble-table lookups in shared memory;
        # the LDS issue rate (32 lanes x 4 B per clock per SM) bounds it:
        #   peak = 148 SM x 32 lookups/clk x f_max / ceil(d/4) x 32 states
        kern_ms = statistics.median(per_step)
        sm_mhz = 1965.0
        try:
            sm_mhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
        except Exception:
            pass
        peak_t = 148 * 32 * sm_mhz * 1e6 / ((d + 3) // 4) * 32 / 1e12
        ach_t = instr["support_tests"] / (kern_ms / 1e3) / 1e12
        roofline = {"bound": "alu", "achieved": round(ach_t, 4), "peak": round(peak_t, 2),
                    "unit": "T support-tests/s (x,a,y,state)", "frac": round(ach_t / peak_t, 4),
                    "traffic": None, "kernel": "rac_batch_cl",
                    "algorithmic_tests_per_launch": instr["support_tests"], "launch_ms_median": round(kern_ms, 5),
                    "peak_source": "derived: LDS lookups (148 SM x 32/clk x %.0f MHz) / ceil(d/4) lookups per "
                                   "32-state test; DESIGN.md section 7" % sm_mhz}
    if alg_bytes is not None and ctx.relation_bytes <= L2_BYTES // 2 and world == 1:
        # The relation is L2-resident (C1/C2): the bound is L2, not HBM.  Peak =
        # read bandwidth of an L2-resident buffer measured here (torch sum of a
        # buffer the size of the relation, back to back, CUDA events).
        l2_gbs = measure_l2_read_gbs(max(ctx.relation_bytes, 4 << 20), dev)
        kern_ms = statistics.median(per_step)
        ach = alg_bytes / (kern_ms / 1e3) / 1e9
        l2_roof = {"bound": "l2", "achieved": round(ach, 1), "peak": round(l2_gbs, 1), "unit": "GB/s",
                   "frac": round(ach / l2_gbs, 4),
                   "peak_source": "measured in this run: torch.sum over an L2-resident %d-byte buffer "
                                  "(read bandwidth, best of 20)" % max(ctx.relation_bytes, 4 << 20)}
    if alg_bytes is not None:
        kern_ms = statistics.median(per_step)
        achieved = alg_bytes / (kern_ms / 1e3) / 1e9
        traffic, traffic_src = None, None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            try:
                tj = json.load(open(tp))
                ent = tj.get(args.workload, {})
                traffic = ent.get("dram_bytes_per_launch")
                if traffic is not None:
                    traffic_src = "ncu --set full dram__bytes_read.sum + dram__bytes_write.sum, one launch, " \
                                  "captured in session %s (profiles/ncu_traffic.json), not in this run" % \
                                  ent.get("round", "?")
            except Exception:
                traffic = None
        full_b = instr.get("full_test_bytes")
        roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                    "kernel": ("wide_fused" if d > 64 else ("rac_state" if ctx.path == "one_block" else "rac_fused"))
                              if (world == 1 or peer) else "rac_pass (+ allgather)",
                    "algorithmic_bytes_per_launch": alg_bytes,
                    "byte_rule": "must-read",
                    "algorithmic_bytes_rule": "must-read: kept rows every tested mask, removed rows one witness "
                                              "mask (Lemma 1); SURVEY 8(d) full-check figure in frac_full_check",
                    "frac_full_check": round(full_b / (kern_ms / 1e3) / 1e9 / peak, 4) if full_b else
                                       round(achieved / peak, 4),
                    "launch_ms_median": round(kern_ms, 5),
                    "peak_source": peak_src + ("" if world == 1 else "; per-GPU bytes = total / N")}
        if ctx.relation_bytes > L2_BYTES:
            # context only (the peak stays MEASURED_PEAKS.json): this box's copy bandwidth,
            # measured here the way the driver measures hbm_gbs -- pool boxes differ
            try:
                roofline["box_copy_gbs"] = round(measure_copy_gbs(dev), 1)
                roofline["box_copy_note"] = ("this box, measured in this run (torch copy of 1 GiB of bf16, "
                                             "read+write bytes, best of 10); context for box-to-box variance, "
                                             "not the roofline denominator")
            except Exception:
                pass
        if world > 1:
            roofline["achieved"] = round(achieved / world, 1)
            roofline["frac"] = round(achieved / world / peak, 4)
    cfg = workload_config(args)
    setup = {"layout": ctx.layout, "relation_bytes": ctx.relation_bytes, "kernel_path": ctx.path,
             "launch": launch_mode,
             "parallelism": (("row-sharded x%d (peer-memory removal exchange + cross-rank barrier inside the "
                              "persistent kernel, NVLink P2P)" if peer else
                              "row-sharded x%d (NCCL all-gather of D per pass)") % world) if world > 1 else "1 GPU",
             "instance_generation_s": round(gen_s, 3)}
    if ctx.wq == 1 and ctx.layout == "dense":
        lay, ms_c, ms_r = ctx.full_pass_layout
        setup["full_pass_sweep"] = {"sweep": lay, "calibration_ms_columns": ms_c, "calibration_ms_rows": ms_r,
                                    "how": "rac_create times one root enforcement with full passes on each dense "
                                           "sweep and keeps the faster (0 = not measured)"}
    out = {"metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
           "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
           "dtype": {1: "u8", 2: "u16", 4: "u32", 8: "u64", 16: "2 x u64", 32: "4 x u64"}[ctx.mask_bytes] + " bitmasks",
           "data": "synthetic (seeded counter-based random CSP, synth/csp_synth.h)", "config": cfg,
           "gpu_launches": int(launches_per_step * args.steps), "clocks": clk, "e2e": e2e,
           "enforcement": instr, "roofline": roofline, "setup": setup, "paper_context": PAPER_CONTEXT}
    if l2_roof is not None:
        out["roofline_l2"] = l2_roof
    if roofline:
        out["relation_gbs_per_iter"] = roofline["achieved"] * (world if world > 1 else 1)
    return out, (n, d, dq, tq, seed, kind, din_h)


L2_BYTES = 126 * (1 << 20)

# BASELINE.md / PAPER.md context: the paper publishes no throughput; its only
# numbers are Table 1's per-assignment counts on its own (unpublished) instances.
PAPER_CONTEXT = {
    "source": "PAPER.md Table 1 (lines 253-288); setup lines 225-236",
    "hardware": "RTAC: Python + PyTorch (fp32 tensors) on an RTX 3090; AC3: Python + JIT on an i9-10900K "
                "(PAPER.md line 229)",
    "table1_recurrence_per_assignment": [3.441, 4.831],
    "table1_revision_per_assignment": [307.6, 107680.5],
    "time_per_assignment": "Fig. 3 (ms per assignment, mean of 50K) -- image missing from the paper text, "
                           "no number recoverable (PAPER.md lines 238-243)",
    "comparable": "no: instances, domain size and tightness unpublished; counts are context only "
                  "(this build's Table-1 trend: DESIGN.md section 7)",
}

# L2-resident workloads (relation well under the 126 MB L2): stated, not flushed
L2_RESIDENT = {"c1-seed", "c2-root", "c5-batch"}


def workload_config(args):
    """The workload-defining keys only (identical in the GPU arm and the reference arm)."""
    n, d, dens, tight, seed, kind, desc = WORKLOADS[args.workload]
    return {"workload": args.workload + ": " + desc, "n": n, "d": d, "density": dens, "tightness": tight,
            "t_q16": synth.quant_tightness(tight), "seed": seed,
            "states": args.states if kind in ("dive", "wrand") else 1,
            "l2": "relation L2-resident (warm; stated, not flushed)" if args.workload in L2_RESIDENT else
                  "inputs larger than L2 (no flush)"}


def wrand_states(n, d, S):
    """S W-rand states (value kept with probability 0.8, seed 1000 + s)."""
    dom = np.full(n, d)
    if d > 64:
        return np.stack([synth.w_rand_wide(dom, 0.8, seed=1000 + s) for s in range(S)])
    return np.stack([synth.w_rand(dom, 0.8, seed=1000 + s) for s in range(S)])


def measure_copy_gbs(dev):
    import torch
    a = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2.0 * (1 << 30) * 2 / (best / 1e3) / 1e9


def measure_l2_read_gbs(nbytes, dev):
    import torch
    buf = torch.ones(nbytes // 4, dtype=torch.float32, device=dev)
    for _ in range(5):
        buf.sum()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            buf.sum()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 10)
    return nbytes / (best / 1e3) / 1e9


def _live_bits(D, n, d):
    """[n, d] bool: value a of x live in the domain state D ([n] or [n * wq] words)."""
    D = np.asarray(D, dtype=np.uint64)
    wq = D.size // n
    W = D.reshape(n, wq)
    out = np.zeros((n, d), dtype=bool)
    for a in range(d):
        out[:, a] = ((W[:, a >> 6] >> np.uint64(a & 63)) & np.uint64(1)).astype(bool)
    return out


# ----------------------------------------------------------------------------- CPU oracle
def oracle_baseline(n, d, dq, tq, seed, kind, din_h, budget_s=20.0, passes=None):
    """The oracle as it stands (single-threaded C, oracle/oracle.c) on a bounded
    sample of the same workload, on this host."""
    import oracle
    if d > 64 and kind == "wrand":
        # wide batched states: O1w per state, one core, bounded
        t0 = time.time()
        orc = oracle.WideOracle.from_synth(n, d, dq, tq, seed)
        build_s = time.time() - t0
        done, t1 = 0, time.perf_counter()
        while True:
            orc.rac(din_h[done % din_h.shape[0]], with_epochs=False)
            done += 1
            el = time.perf_counter() - t1
            if el > budget_s or done >= din_h.shape[0]:
                break
        return {"value": done / el, "unit": "states/s", "cores": 1, "kind": "oracle",
                "sample": "%d state(s) of the batch by orc_rac_wide (O1w, 1 thread) in %.1f s; oracle instance "
                          "build %.1f s excluded" % (done, el, build_s)}
    if d > 64:
        # Wide domains (NEXT-4): the oracle's build is O(n^2 d^2) generator calls,
        # so time one Eq. 1 step over the rows of a block of B variables (O1w's
        # step, orc_wpass_block) and scale by n/B and the pass count.
        B = max(1, min(n, int(4e6 / (n * d))))
        t0 = time.time()
        orc = oracle.WideOracle.from_synth_block(n, d, dq, tq, seed, 0, B)
        build_s = time.time() - t0
        reps, t1 = 0, time.perf_counter()
        while True:
            orc.pass_block(din_h[0], 0, B)
            reps += 1
            el = time.perf_counter() - t1
            if el > budget_s / 3 or reps >= 20:
                break
        t_block = el / reps
        npass = passes or 1
        t_enf = t_block * (n / B) * npass
        return {"value": 1.0 / t_enf, "unit": UNIT, "cores": 1, "kind": "oracle",
                "sample": "pass over the rows of variables [0,%d) of %d (orc_wpass_block, the O1w step, 1 thread), "
                          "%d reps, %.4f s each; scaled x n/B = %.1f and x %d pass(es); block build %.1f s excluded"
                          % (B, n, reps, t_block, n / B, npass, build_s)}
    if kind != "dive" and float(n) * n * d * d / 8 > 2e9:
        # C4-size: the oracle's own instance would not fit / take minutes to build.
        # Sample: arcs of a block of B variables, one Eq. 1 step over its rows,
        # scaled by n/B and by the enforcement's pass count.
        B = max(1, min(n, int(2e8 / (n * d * 8))))
        t0 = time.time()
        orc = oracle.Oracle.from_synth_block(n, d, dq, tq, seed, 0, B)
        build_s = time.time() - t0
        reps, t1 = 0, time.perf_counter()
        while True:
            orc.pass_block(din_h[0], 0, B)
            reps += 1
            el = time.perf_counter() - t1
            if el > budget_s / 3 or reps >= 20:
                break
        t_block = el / reps
        npass = passes or 1
        t_enf = t_block * (n / B) * npass
        return {"value": 1.0 / t_enf, "unit": UNIT, "cores": 1, "kind": "oracle",
                "sample": "pass over the rows of variables [0,%d) of %d (orc_pass_block, the O1 step, 1 thread), "
                          "%d reps, %.4f s each; scaled x n/B = %.1f and x %d pass(es); block build %.1f s excluded"
                          % (B, n, reps, t_block, n / B, npass, build_s)}
    t0 = time.time()
    if kind == "dive":
        inst = synth.random_csp(n, d, 0.8, 0.3, seed)
        orc = oracle.Oracle.from_instance(inst)
    else:
        orc = oracle.Oracle.from_synth(n, d, dq, tq, seed)
    build_s = time.time() - t0
    unit = "states/s" if kind == "dive" else UNIT
    S = din_h.shape[0]
    cores = oracle.max_threads()

    def timed(fn, budget, per_call_units=1):
        """calls of fn() until `budget` seconds (at least one); returns units/s, calls, seconds"""
        done, t1 = 0, time.perf_counter()
        while True:
            fn(done)
            done += 1
            el = time.perf_counter() - t1
            if el > budget or done >= 64 * max(1, S):
                break
        return done * per_call_units / el, done, el

    # (1) O1 on one core
    v_one, calls1, el1 = timed(lambda k: orc.rac(din_h[k % S], with_epochs=False), budget_s * 0.3)
    one = {"value": v_one, "unit": unit, "cores": 1, "kind": "oracle",
           "sample": "%d enforcement(s) by orc_rac (O1, gcc -O2, 1 thread) in %.1f s" % (calls1, el1)}
    # (2) O1 on every host core
    if kind == "dive":
        v_all, calls, el = timed(lambda k: orc.rac_many(din_h, threads=0), budget_s * 0.4, per_call_units=S)
        s_all = "%d batch(es) of %d W-dive states, states spread over %d OpenMP threads (orc_rac_many, O1)" % (
            calls, S, cores)
    else:
        v_all, calls, el = timed(lambda k: orc.rac_par(din_h[0], threads=0), budget_s * 0.4)
        s_all = "%d enforcement(s) of the same D_in, each pass's variables over %d OpenMP threads (orc_rac_par, O1)" % (
            calls, cores)
    allc = {"value": v_all, "unit": unit, "cores": cores, "kind": "oracle",
            "sample": s_all + " in %.1f s; oracle instance build %.1f s excluded" % (el, build_s)}
    # (3) AC-3 on one core: the paper's baseline class (inherently sequential)
    v_ac3, calls3, el3 = timed(lambda k: orc.ac3(din_h[k % S]), budget_s * 0.3)
    ac3 = {"value": v_ac3, "unit": unit, "cores": 1, "kind": "oracle (AC-3, O2)",
           "sample": "%d enforcement(s) by orc_ac3 (FIFO AC-3, the paper's baseline class, PAPER.md line 227) "
                     "in %.1f s" % (calls3, el3)}
    # Headline: every core where a pass has enough work to split (batches of states;
    # an enforcement of >= 2 ms on one core); a small enforcement is synchronisation-
    # bound across threads, and its honest host figure is the single-thread one.
    head = allc if (kind == "dive" or v_one < 500.0) else one
    out = dict(head)
    out["one_core"] = one
    out["all_cores"] = allc
    out["ac3_one_core"] = ac3
    return out


def run_reference(args):
    """--impl reference: the CPU oracle on the same workload (the base contract's
    reference arm for this tier)."""
    n, d, dens, tight, seed, kind, desc = WORKLOADS[args.workload]
    dq, tq = synth.quant_density(dens), synth.quant_tightness(tight)
    import oracle
    if d > 64 and kind == "wrand":
        din_h = wrand_states(n, d, args.states)
        cb = oracle_baseline(n, d, dq, tq, seed, kind, din_h, budget_s=min(120.0, 10.0 * max(1, args.steps)))
        val = cb["value"]
        return {"metric": "AC enforcements/sec (batched states)", "value": val, "unit": "states/s", "n_gpus": 0,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": args.states / val * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64 bitsets",
                "data": "synthetic (seeded counter-based random CSP, synth/csp_synth.h)",
                "config": workload_config(args), "impl": "reference", "cpu_baseline": cb,
                "e2e": {"value": val, "unit": "states/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if d > 64:
        # Wide domains: the oracle instance is O(n^2 d^2) to build; each step is the
        # block-sampled O1w estimate of one enforcement (see oracle_baseline).
        full = synth.full_domains_wide(np.full(n, d))
        cb = oracle_baseline(n, d, dq, tq, seed, kind, full[None, :], budget_s=min(60.0, 6.0 * max(1, args.steps)))
        val = cb["value"]
        return {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": 0, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 / val, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u64 bitsets", "data": "synthetic (seeded counter-based random CSP, "
                "synth/csp_synth.h)", "config": workload_config(args),
                "impl": "reference", "cpu_baseline": cb,
                "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if kind == "dive":
        inst = synth.random_csp(n, d, dens, tight, seed)
        orc = oracle.Oracle.from_instance(inst)
        _, root, _, _ = orc.rac(inst.full_domains(), with_epochs=False)
        din_h = np.stack(synth.dive_states(root, lambda D: orc.rac(D, with_epochs=False)[:2], args.states, seed))
    else:
        orc = oracle.Oracle.from_synth(n, d, dq, tq, seed)
        full = synth.full_domains(np.full(n, d))
        if kind == "seed":
            _, root, _, _ = orc.rac(full, with_epochs=False)
            d_in, _, _ = synth.w_seed(root, seed)
        else:
            d_in = full
        din_h = d_in[None, :]
    # bounded sample, on every host core: each step = one enforcement (orc_rac_par:
    # each pass's variables over OpenMP threads) or, batched, one batch of states
    # (orc_rac_many: states over threads); cap the total time
    cores = oracle.max_threads()
    S = din_h.shape[0]
    t0 = time.perf_counter()
    orc.rac(din_h[0], with_epochs=False)
    one = time.perf_counter() - t0
    if kind == "dive":
        def one_step(k):
            orc.rac_many(din_h, threads=0)
    elif one >= 2e-3:
        def one_step(k):
            orc.rac_par(din_h[0], threads=0)
    else:  # small enforcement: threads only add synchronisation (see oracle_baseline)
        cores = 1

        def one_step(k):
            orc.rac(din_h[0], with_epochs=False)
    t0 = time.perf_counter()
    one_step(0)
    one = time.perf_counter() - t0
    budget = 150.0
    steps = args.steps
    if one * (args.steps + args.warmup) > budget:
        steps = max(3, int(budget / max(one, 1e-9)) - args.warmup)
    for k in range(min(args.warmup, 3)):
        one_step(k)
    t0 = time.perf_counter()
    for k in range(steps):
        one_step(k)
    el = time.perf_counter() - t0
    unit = "states/s" if kind == "dive" else UNIT
    val = steps * (S if kind == "dive" else 1) / el
    sample = ("%d of %d requested steps, each %s by the oracle's O1 on %d thread(s)" %
              (steps, args.steps, ("one batch of %d states (orc_rac_many)" % S) if kind == "dive" else
               "one full enforcement (%s)" % ("orc_rac_par" if cores > 1 else "orc_rac"), cores))
    return {"metric": METRIC if kind != "dive" else "AC enforcements/sec (batched search-tree states)",
            "value": val, "unit": unit, "n_gpus": 0, "steps": steps, "warmup": args.warmup,
            "ms_per_step": el / steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u64 bitsets", "data": "synthetic (seeded counter-based random CSP, synth/csp_synth.h)",
            "config": workload_config(args),
            "impl": "reference",
            "cpu_baseline": {"value": val, "unit": unit, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--workload", default="c3-stream", choices=sorted(WORKLOADS))
    ap.add_argument("--states", type=int, default=1024)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="N > 1: per-pass exchange through peer memory inside the fused kernel (default) "
                         "or an NCCL all-gather between per-pass launches")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # Testing knob: RAC_BENCH_SHARED_GPU=1 runs every rank on cuda:0 (gloo process
    # group, peer exchange, grids capped so they fit together) to exercise the N > 1
    # code path on a one-GPU box.  Numbers from it are not throughput claims.
    shared = os.environ.get("RAC_BENCH_SHARED_GPU") == "1" and world > 1
    if shared:
        local_rank = 0

    if args.impl == "reference":
        if rank != 0:
            return 0
        out = run_reference(args)
        print(json.dumps(out), flush=True)
        return 0

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out, wl = run_gpu(args, rank, world, local_rank)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            try:
                out["cpu_baseline"] = oracle_baseline(*wl, budget_s=args.cpu_budget,
                                                      passes=out.get("enforcement", {}).get("iterations"))
            except Exception as e:  # report, never hide
                out["cpu_baseline"] = {"value": None, "error": repr(e)}
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
