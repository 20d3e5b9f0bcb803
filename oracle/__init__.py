"""CPU oracle for Recurrent Arc Consistency (RAC), arXiv 2407.11388.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2407_11388_b200``) never imports it and
shares no code with it.

Contents
  * ``Oracle`` -- ctypes wrapper over ``oracle/oracle.c`` (plain C, built with
    gcc): O1 naive RAC (Eq. 1, loop of Alg. 1 lines
    198-210), O2 AC-3 (line 29), the AC definition audit (lines 49-61) and the
    O4 certificate (Lemma 1, lines 79-82).
  * ``brute_force_dac`` -- O3: D_ac as the union of all arc-consistent subsets
    of D, by enumerating every subset (tiny inputs).
  * ``Oracle.rac_seeded`` -- O5: Alg. 1 tensorAC(Vars, @changed) as written
    (lines 198-221), the paper's incremental per-assignment call (line 392).
  * ``Oracle.search`` -- O6: Alg. 2 backtracking search (lines 369-417) over
    O5 / O1 / O2 enforcement.
  * ``rac_python`` -- a pure-Python transcription of Eq. 1 (tiny inputs), used
    to cross-check the C transcription.

Parity status: every function here is pinned by tests/test_oracle.py
(brute force, closed forms, hand traces from SPEC.md, AC-3 agreement,
certificate acceptance/rejection, invariants).  No function is unpinned.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK = 0
WIPEOUT = 1

_lib = None


_CFLAGS = ["-O2", "-std=c11", "-shared", "-fPIC", "-Wall", "-fopenmp"]


def _source_hash() -> str:
    """sha256 of the sources and flags; a library with another stamp is rebuilt
    (file times are not trusted: the tree is copied between machines)."""
    import hashlib
    h = hashlib.sha256()
    for p in (_SRC, os.path.join(_HERE, "..", "synth", "csp_synth.h")):
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(_CFLAGS).encode())
    return h.hexdigest()


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (plain C, -O2, no SIMD
    intrinsics; OpenMP only for the independent per-variable loops of the
    certificate and of the all-core timing leg)."""
    stamp = _LIB + ".srchash"
    want = _source_hash()
    have = open(stamp).read().strip() if os.path.exists(stamp) else ""
    if force or not os.path.exists(_LIB) or have != want:
        tmp = _LIB + ".tmp.%d" % os.getpid()
        subprocess.check_call(["gcc", *_CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
        with open(stamp, "w") as f:
            f.write(want + "\n")
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        u64p = ctypes.POINTER(ctypes.c_uint64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        lib.orc_build.restype = P
        lib.orc_build.argtypes = [ctypes.c_int, i32p, ctypes.c_int, i32p, i32p, u64p, ctypes.c_int]
        lib.orc_build_synth.restype = P
        lib.orc_build_synth.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64]
        lib.orc_free.argtypes = [P]
        lib.orc_free.restype = None
        lib.orc_rac.argtypes = [P, u64p, u64p, i32p, i32p, ctypes.c_int]
        lib.orc_rac.restype = ctypes.c_int
        lib.orc_rac_par.argtypes = [P, u64p, u64p, i32p, ctypes.c_int, ctypes.c_int]
        lib.orc_rac_par.restype = ctypes.c_int
        lib.orc_rac_many.argtypes = [P, ctypes.c_int, u64p, u64p, i32p, i32p, ctypes.c_int, ctypes.c_int]
        lib.orc_rac_many.restype = ctypes.c_int
        lib.orc_max_threads.argtypes = []
        lib.orc_max_threads.restype = ctypes.c_int
        lib.orc_rac_seeded.argtypes = [P, u64p, i32p, ctypes.c_int, u64p, i32p, i32p, ctypes.c_int]
        lib.orc_rac_seeded.restype = ctypes.c_int
        lib.orc_search.argtypes = [P, u64p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, i32p,
                                   ctypes.POINTER(ctypes.c_int64)]
        lib.orc_search.restype = ctypes.c_int
        lib.orc_ac3.argtypes = [P, u64p, u64p, ctypes.POINTER(ctypes.c_int64)]
        lib.orc_ac3.restype = ctypes.c_int
        lib.orc_is_ac.argtypes = [P, u64p]
        lib.orc_is_ac.restype = ctypes.c_int
        lib.orc_certify.argtypes = [P, u64p, u64p, i32p, ctypes.c_int]
        lib.orc_certify.restype = ctypes.c_int
        lib.orc_support.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, i32p]
        lib.orc_support.restype = ctypes.c_uint64
        lib.orc_degree.argtypes = [P, ctypes.c_int]
        lib.orc_degree.restype = ctypes.c_int
        lib.orc_row_supported_synth.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32,
                                                ctypes.c_uint64, ctypes.c_int, ctypes.c_int, u64p]
        lib.orc_row_supported_synth.restype = ctypes.c_int
        lib.orc_build_synth_block.restype = P
        lib.orc_build_synth_block.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32,
                                              ctypes.c_uint64, ctypes.c_int, ctypes.c_int]
        lib.orc_pass_block.restype = ctypes.c_int64
        lib.orc_pass_block.argtypes = [P, u64p, ctypes.c_int, ctypes.c_int, u64p]
        lib.orc_certify_trajectory.argtypes = [P, u64p, u64p, i32p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        lib.orc_certify_trajectory.restype = ctypes.c_int
        lib.orc_wcertify_trajectory.argtypes = [P, u64p, u64p, i32p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        lib.orc_wcertify_trajectory.restype = ctypes.c_int
        lib.orc_certify_trajectory_synth.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32,
                                                     ctypes.c_uint64, u64p, u64p, i32p, ctypes.c_int, ctypes.c_int,
                                                     ctypes.c_int, ctypes.c_int]
        lib.orc_certify_trajectory_synth.restype = ctypes.c_int
        lib.orc_wbuild.restype = P
        lib.orc_wbuild.argtypes = [ctypes.c_int, i32p, ctypes.c_int, i32p, i32p, u64p, ctypes.c_int]
        lib.orc_wbuild_synth.restype = P
        lib.orc_wbuild_synth.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32,
                                         ctypes.c_uint64]
        lib.orc_wbuild_synth_block.restype = P
        lib.orc_wbuild_synth_block.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32,
                                               ctypes.c_uint64, ctypes.c_int, ctypes.c_int]
        lib.orc_wpass_block.restype = ctypes.c_int64
        lib.orc_wpass_block.argtypes = [P, u64p, ctypes.c_int, ctypes.c_int, u64p]
        lib.orc_wfree.argtypes = [P]
        lib.orc_wfree.restype = None
        lib.orc_wq.argtypes = [P]
        lib.orc_wq.restype = ctypes.c_int
        lib.orc_rac_wide.argtypes = [P, u64p, u64p, i32p, i32p, ctypes.c_int]
        lib.orc_rac_wide.restype = ctypes.c_int
        lib.orc_wis_ac.argtypes = [P, u64p]
        lib.orc_wis_ac.restype = ctypes.c_int
        lib.orc_wsearch.argtypes = [P, u64p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, i32p,
                                    ctypes.POINTER(ctypes.c_int64)]
        lib.orc_wsearch.restype = ctypes.c_int
        lib.orc_wac3.argtypes = [P, u64p, u64p]
        lib.orc_wac3.restype = ctypes.c_int
        _lib = lib
    return _lib


def _u64p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def _i32p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


class Oracle:
    """One CSP instance in the oracle's own per-arc layout."""

    def __init__(self, handle, n: int, dom: np.ndarray):
        self._h = handle
        self.n = n
        self.dom = dom

    @classmethod
    def from_instance(cls, inst) -> "Oracle":
        lib = _load()
        dom = np.ascontiguousarray(inst.dom, dtype=np.int32)
        xs = np.ascontiguousarray(inst.xs, dtype=np.int32)
        ys = np.ascontiguousarray(inst.ys, dtype=np.int32)
        rows = np.ascontiguousarray(inst.rows, dtype=np.uint64)
        stride = rows.shape[1] if rows.ndim == 2 and rows.shape[0] else int(dom.max())
        if rows.size == 0:
            rows = np.zeros((1, max(stride, 1)), dtype=np.uint64)
        h = lib.orc_build(inst.n, _i32p(dom), xs.shape[0], _i32p(xs), _i32p(ys), _u64p(rows), stride)
        if not h:
            raise ValueError("invalid instance")
        return cls(h, inst.n, dom)

    @classmethod
    def from_synth(cls, n: int, d: int, dens_q32: int, t_q16: int, seed: int) -> "Oracle":
        lib = _load()
        h = lib.orc_build_synth(n, d, dens_q32, t_q16, seed)
        if not h:
            raise ValueError("invalid synth parameters")
        return cls(h, n, np.full(n, d, dtype=np.int32))

    @classmethod
    def from_synth_block(cls, n: int, d: int, dens_q32: int, t_q16: int, seed: int, x_lo: int, x_hi: int):
        """Arcs of variables [x_lo, x_hi) only (sampled timing at C4 size); use pass_block only."""
        lib = _load()
        h = lib.orc_build_synth_block(n, d, dens_q32, t_q16, seed, x_lo, x_hi)
        if not h:
            raise ValueError("invalid synth parameters")
        o = cls(h, n, np.full(n, d, dtype=np.int32))
        o.block = (x_lo, x_hi)
        return o

    def pass_block(self, D, x_lo: int, x_hi: int):
        """One Eq. 1 step for rows of [x_lo, x_hi): (new words, number removed)."""
        D = np.ascontiguousarray(D, dtype=np.uint64)
        out = np.zeros(max(x_hi - x_lo, 1), dtype=np.uint64)
        r = _load().orc_pass_block(self._h, _u64p(D), x_lo, x_hi, _u64p(out))
        return out[: x_hi - x_lo], int(r)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_free(self._h)
            self._h = None

    def rac(self, d_in, full: bool = False, with_epochs: bool = True):
        """O1. Returns (status, d_out, iterations, removed_at[n,64] or None)."""
        lib = _load()
        d_in = np.ascontiguousarray(d_in, dtype=np.uint64)
        d_out = np.zeros(self.n, dtype=np.uint64)
        it = np.zeros(1, dtype=np.int32)
        rem = np.zeros(self.n * 64, dtype=np.int32) if with_epochs else None
        st = lib.orc_rac(self._h, _u64p(d_in), _u64p(d_out), _i32p(it),
                         _i32p(rem) if rem is not None else None, 1 if full else 0)
        return st, d_out, int(it[0]), (rem.reshape(self.n, 64) if rem is not None else None)

    def rac_par(self, d_in, full: bool = False, threads: int = 0):
        """O1 with each step's variables split over `threads` OpenMP threads (0 =
        all host cores; the all-core CPU baseline).  Returns (status, d_out, iterations)."""
        lib = _load()
        d_in = np.ascontiguousarray(d_in, dtype=np.uint64)
        d_out = np.zeros(self.n, dtype=np.uint64)
        it = np.zeros(1, dtype=np.int32)
        st = lib.orc_rac_par(self._h, _u64p(d_in), _u64p(d_out), _i32p(it), 1 if full else 0, int(threads))
        return st, d_out, int(it[0])

    def rac_many(self, states, full: bool = False, threads: int = 0):
        """O1 on every row of states [S, n], states spread over OpenMP threads.
        Returns (status[S], d_out[S, n], iterations[S])."""
        states = np.ascontiguousarray(states, dtype=np.uint64)
        S = states.shape[0]
        out = np.zeros_like(states)
        it = np.zeros(S, dtype=np.int32)
        st = np.zeros(S, dtype=np.int32)
        _load().orc_rac_many(self._h, S, _u64p(states), _u64p(out), _i32p(it), _i32p(st), 1 if full else 0,
                             int(threads))
        return st, out, it

    def rac_seeded(self, d_in, seeds, full: bool = False, with_epochs: bool = True):
        """O5: Alg. 1 tensorAC(Vars, @changed = seeds) as written.  Returns like rac()."""
        lib = _load()
        d_in = np.ascontiguousarray(d_in, dtype=np.uint64)
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.int32).reshape(-1))
        d_out = np.zeros(self.n, dtype=np.uint64)
        it = np.zeros(1, dtype=np.int32)
        rem = np.zeros(self.n * 64, dtype=np.int32) if with_epochs else None
        st = lib.orc_rac_seeded(self._h, _u64p(d_in), _i32p(seeds) if seeds.size else None, int(seeds.size),
                                _u64p(d_out), _i32p(it), _i32p(rem) if rem is not None else None, 1 if full else 0)
        return st, d_out, int(it[0]), (rem.reshape(self.n, 64) if rem is not None else None)

    def search(self, d_in, max_assignments: int = 0, engine: str = "seeded", all_solutions: bool = False,
               full: bool = False):
        """O6: Alg. 2 backtracking search.  Returns (result, solution, stats) with result 0 = solution,
        1 = unsat, 2 = budget; stats keys as in rac_search_stats."""
        lib = _load()
        d_in = np.ascontiguousarray(d_in, dtype=np.uint64)
        sol = np.full(self.n, -1, dtype=np.int32)
        st = (ctypes.c_int64 * 6)()
        eng = {"seeded": 0, "full": 1, "ac3": 2}[engine]
        r = lib.orc_search(self._h, _u64p(d_in), int(max_assignments), eng, 1 if all_solutions else 0,
                           1 if full else 0, _i32p(sol), st)
        keys = ["assignments", "recurrences", "wipeouts", "solutions", "max_depth", "root_iterations"]
        return r, sol, dict(zip(keys, [int(v) for v in st]))

    def ac3(self, d_in):
        """O2. Returns (status, d_out, revisions)."""
        lib = _load()
        d_in = np.ascontiguousarray(d_in, dtype=np.uint64)
        d_out = np.zeros(self.n, dtype=np.uint64)
        rev = ctypes.c_int64(0)
        st = lib.orc_ac3(self._h, _u64p(d_in), _u64p(d_out), ctypes.byref(rev))
        return st, d_out, int(rev.value)

    def is_ac(self, D) -> bool:
        D = np.ascontiguousarray(D, dtype=np.uint64)
        return bool(_load().orc_is_ac(self._h, _u64p(D)))

    def certify(self, d_in, d_out, removed_at, check_ac: bool = True) -> int:
        """O4. 0 = accepted; nonzero = reason code (see oracle.c)."""
        d_in = np.ascontiguousarray(d_in, dtype=np.uint64)
        d_out = np.ascontiguousarray(d_out, dtype=np.uint64)
        rem = np.ascontiguousarray(np.asarray(removed_at, dtype=np.int32).reshape(-1))
        return int(_load().orc_certify(self._h, _u64p(d_in), _u64p(d_out), _i32p(rem), 1 if check_ac else 0))

    def certify_trajectory(self, d_in, d_out, removed_at, iterations: int, status: int, full: bool = False) -> int:
        """O7: 0 iff (status, d_out, iterations, removed_at) is exactly the RAC
        recurrence's output on d_in (see oracle.c); else a reason code."""
        d_in = np.ascontiguousarray(d_in, dtype=np.uint64)
        d_out = np.ascontiguousarray(d_out, dtype=np.uint64)
        rem = np.ascontiguousarray(np.asarray(removed_at, dtype=np.int32).reshape(-1))
        assert rem.size == self.n * 64
        return int(_load().orc_certify_trajectory(self._h, _u64p(d_in), _u64p(d_out), _i32p(rem), int(iterations),
                                                  int(status), 1 if full else 0))

    def support(self, x: int, y: int, a: int) -> Tuple[bool, int]:
        p = ctypes.c_int32(0)
        s = _load().orc_support(self._h, x, y, a, ctypes.byref(p))
        return bool(p.value), int(s)

    def degree(self, x: int) -> int:
        return int(_load().orc_degree(self._h, x))


class WideOracle:
    """Wide-domain instance (NEXT-4, domains up to 256 values): domain states are
    [n * wq] uint64 words, wq = ceil(max dom / 64); removal epochs [n, 64 * wq]."""

    def __init__(self, handle, n: int, dom: np.ndarray):
        self._h = handle
        self.n = n
        self.dom = dom
        self.wq = int(_load().orc_wq(handle))

    @classmethod
    def from_instance(cls, inst) -> "WideOracle":
        """inst.rows: uint64 [n_rel, max_dom, wq] (synth.wide_from_constraints / random_csp_wide)."""
        lib = _load()
        dom = np.ascontiguousarray(inst.dom, dtype=np.int32)
        xs = np.ascontiguousarray(inst.xs, dtype=np.int32)
        ys = np.ascontiguousarray(inst.ys, dtype=np.int32)
        wq = max(1, (int(dom.max()) + 63) // 64)
        rows = np.ascontiguousarray(inst.rows, dtype=np.uint64)
        stride = rows.shape[1] if rows.ndim == 3 and rows.shape[0] else int(dom.max())
        if rows.size == 0:
            rows = np.zeros((1, stride, wq), dtype=np.uint64)
        assert rows.shape[2] == wq, "rows must be [n_rel, max_dom, ceil(max_dom/64)]"
        h = lib.orc_wbuild(inst.n, _i32p(dom), xs.shape[0], _i32p(xs), _i32p(ys), _u64p(rows), stride)
        if not h:
            raise ValueError("invalid instance")
        return cls(h, inst.n, dom)

    @classmethod
    def from_synth(cls, n: int, d: int, dens_q32: int, t_q16: int, seed: int) -> "WideOracle":
        h = _load().orc_wbuild_synth(n, d, dens_q32, t_q16, seed)
        if not h:
            raise ValueError("invalid generator parameters")
        return cls(h, n, np.full(n, d, dtype=np.int32))

    @classmethod
    def from_synth_block(cls, n: int, d: int, dens_q32: int, t_q16: int, seed: int, x_lo: int, x_hi: int):
        """Arcs of the variables [x_lo, x_hi) only (sampled CPU timing; pass_block only)."""
        h = _load().orc_wbuild_synth_block(n, d, dens_q32, t_q16, seed, x_lo, x_hi)
        if not h:
            raise ValueError("invalid generator parameters")
        return cls(h, n, np.full(n, d, dtype=np.int32))

    def pass_block(self, D, x_lo: int, x_hi: int):
        """One Eq. 1 step over the rows of [x_lo, x_hi).  Returns (out [n*wq], removed)."""
        D = np.ascontiguousarray(D, dtype=np.uint64).reshape(-1)
        out = D.copy()
        r = _load().orc_wpass_block(self._h, _u64p(D), x_lo, x_hi, _u64p(out))
        return out, int(r)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_wfree(self._h)
            self._h = None

    def rac(self, d_in, full: bool = False, with_epochs: bool = True):
        """O1w. Returns (status, d_out [n*wq], iterations, removed_at [n, 64*wq] or None)."""
        lib = _load()
        d_in = np.ascontiguousarray(d_in, dtype=np.uint64).reshape(-1)
        assert d_in.size == self.n * self.wq
        d_out = np.zeros(self.n * self.wq, dtype=np.uint64)
        it = np.zeros(1, dtype=np.int32)
        rem = np.zeros(self.n * 64 * self.wq, dtype=np.int32) if with_epochs else None
        st = lib.orc_rac_wide(self._h, _u64p(d_in), _u64p(d_out), _i32p(it),
                              _i32p(rem) if rem is not None else None, 1 if full else 0)
        return st, d_out, int(it[0]), (rem.reshape(self.n, 64 * self.wq) if rem is not None else None)

    def is_ac(self, D) -> bool:
        D = np.ascontiguousarray(D, dtype=np.uint64).reshape(-1)
        return bool(_load().orc_wis_ac(self._h, _u64p(D)))

    def certify_trajectory(self, d_in, d_out, removed_at, iterations: int, status: int, full: bool = False) -> int:
        """O7 on wide domains: 0 iff the claim is exactly the recurrence's output."""
        d_in = np.ascontiguousarray(d_in, dtype=np.uint64).reshape(-1)
        d_out = np.ascontiguousarray(d_out, dtype=np.uint64).reshape(-1)
        rem = np.ascontiguousarray(np.asarray(removed_at, dtype=np.int32).reshape(-1))
        assert rem.size == self.n * 64 * self.wq and d_in.size == self.n * self.wq
        return int(_load().orc_wcertify_trajectory(self._h, _u64p(d_in), _u64p(d_out), _i32p(rem), int(iterations),
                                                   int(status), 1 if full else 0))

    def search(self, d_in, max_assignments: int = 0, all_solutions: bool = False, full: bool = False):
        """O6w: Alg. 2 backtracking search over O1w.  Returns (result, solution, stats) like Oracle.search."""
        d_in = np.ascontiguousarray(d_in, dtype=np.uint64).reshape(-1)
        sol = np.full(self.n, -1, dtype=np.int32)
        st = (ctypes.c_int64 * 6)()
        r = _load().orc_wsearch(self._h, _u64p(d_in), int(max_assignments), 1 if all_solutions else 0,
                                1 if full else 0, _i32p(sol), st)
        keys = ["assignments", "recurrences", "wipeouts", "solutions", "max_depth", "root_iterations"]
        return r, sol, dict(zip(keys, [int(v) for v in st]))

    def ac3(self, d_in):
        """AC-3 to the fixpoint on wide domains.  Returns (status, d_out)."""
        d_in = np.ascontiguousarray(d_in, dtype=np.uint64).reshape(-1)
        d_out = np.zeros(self.n * self.wq, dtype=np.uint64)
        st = _load().orc_wac3(self._h, _u64p(d_in), _u64p(d_out))
        return st, d_out


def certify_trajectory_synth(n: int, d: int, dens_q32: int, t_q16: int, seed: int, d_in, d_out, removed_at,
                             iterations: int, status: int, full: bool = False, threads: int = 0) -> int:
    """O7 on the seeded random instance (d <= 256), regenerating the support sets
    of one variable at a time from synth/csp_synth.h (C4 / wide bench sizes).
    Domain states [n * ceil(d/64)] words, epochs [n, 64 * ceil(d/64)]."""
    wq = (d + 63) // 64
    d_in = np.ascontiguousarray(d_in, dtype=np.uint64).reshape(-1)
    d_out = np.ascontiguousarray(d_out, dtype=np.uint64).reshape(-1)
    rem = np.ascontiguousarray(np.asarray(removed_at, dtype=np.int32).reshape(-1))
    assert d_in.size == n * wq and d_out.size == n * wq and rem.size == n * 64 * wq
    return int(_load().orc_certify_trajectory_synth(n, d, dens_q32, t_q16, seed, _u64p(d_in), _u64p(d_out),
                                                    _i32p(rem), int(iterations), int(status), 1 if full else 0,
                                                    int(threads)))


def max_threads() -> int:
    """OpenMP threads the oracle's parallel legs use by default (the host's cores)."""
    return int(_load().orc_max_threads())


def row_supported_synth(n: int, d: int, dens_q32: int, t_q16: int, seed: int, x: int, a: int, D) -> bool:
    """Would (x,a) survive one step of Eq. 1 from D?  Straight from the generator."""
    D = np.ascontiguousarray(D, dtype=np.uint64)
    return bool(_load().orc_row_supported_synth(n, d, dens_q32, t_q16, seed, x, a, _u64p(D)))


# ----------------------------------------------------------------------------- pure Python
def _support_sets(inst):
    """{(x,y): {a: set(b)}} for both orientations of every declared constraint."""
    sup = {}
    for k in range(inst.n_rel):
        x, y = int(inst.xs[k]), int(inst.ys[k])
        fw = {a: set() for a in range(int(inst.dom[x]))}
        bw = {b: set() for b in range(int(inst.dom[y]))}
        for a in range(int(inst.dom[x])):
            r = int(inst.rows[k, a])
            for b in range(int(inst.dom[y])):
                if (r >> b) & 1:
                    fw[a].add(b)
                    bw[b].add(a)
        sup[(x, y)] = fw
        sup[(y, x)] = bw
    return sup


def _to_set(D) -> set:
    return {(x, a) for x in range(len(D)) for a in range(64) if (int(D[x]) >> a) & 1}


def _from_set(S, n) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    for (x, a) in S:
        out[x] |= np.uint64(1) << np.uint64(a)
    return out


def _is_ac_set(sup, S: set) -> bool:
    """PAPER.md lines 49-61, literally: ∀(x,a)∈S ∀c_xy∈C_x: c_xy|(x,a) ∩ S ≠ ∅."""
    for (x, a) in S:
        for (xx, y), rows in sup.items():
            if xx != x:
                continue
            if not any((y, b) in S for b in rows[a]):
                return False
    return True


def brute_force_dac(inst, d_in) -> np.ndarray:
    """O3: D_ac = ⋃{D' ⊆ D : D' arc consistent}, by
    enumerating all 2^|D| subsets.  Only for |D| <= ~16."""
    sup = _support_sets(inst)
    elems = sorted(_to_set(d_in))
    if len(elems) > 18:
        raise ValueError("brute force limited to |D| <= 18")
    union = set()
    for mask in range(1 << len(elems)):
        S = {elems[i] for i in range(len(elems)) if (mask >> i) & 1}
        if _is_ac_set(sup, S):
            union |= S
    return _from_set(union, inst.n)


def rac_python(inst, d_in, full: bool = False):
    """Eq. 1 in set notation, pure Python, tiny inputs.

    D~(0) = ∅; D~(k) = D~(k-1) ∪ {(x,a) | ∃y: c_xy|(x,a) ∩ (D \\ D~(k-1)) = ∅}
    with Alg. 1's loop control (lines 198-210).  Returns (status, d_out, iterations,
    list of per-step removal sets V^(k))."""
    sup = _support_sets(inst)
    D = _to_set(d_in)
    removed = set()
    trace: List[set] = []
    k = 0
    while True:
        k += 1
        live = D - removed
        new = set()
        for (x, a) in live:
            for (xx, y), rows in sup.items():
                if xx == x and not any((y, b) in live for b in rows[a]):
                    new.add((x, a))
                    break
        removed |= new
        trace.append(new)
        cur = D - removed
        wipe = any(not any((x, a) in cur for a in range(int(inst.dom[x]))) for x in range(inst.n))
        if wipe and not full:
            return WIPEOUT, _from_set(cur, inst.n), k, trace
        if not new:
            return (WIPEOUT if wipe else OK), _from_set(cur, inst.n), k, trace
