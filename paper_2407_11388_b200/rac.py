"""Thin ctypes binding of librac.so (include/rac.h).  Argument marshalling
only: every step of the enforcement runs in the library's CUDA kernels.

The functions keep the C names (``rac_create``, ``rac_enforce``, ...).
``RacContext`` is a small owning wrapper that also accepts torch tensors
(device memory / streams come from torch: plumbing, not the product).

There is no CPU fallback: if librac.so is missing or cannot be loaded this
module raises at import time.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RAC_LIB_PATH") or os.path.join(_HERE, "librac.so")  # override: A/B tooling

RAC_OK = 0
RAC_WIPEOUT = 1
RAC_BUDGET = 2
RAC_SEARCH_ALL = 1 << 8
RAC_EINVAL = -1
RAC_ENOMEM = -2
RAC_ECUDA = -3
RAC_ENCCL = -4
RAC_ESTATE = -5
RAC_EUNSUPPORTED = -6
RAC_EPEER = -7
RAC_FULL_FIXPOINT = 1
RAC_OPT_NCCL_SELF = 1
RAC_OPT_PEER = 2
RAC_OPT_SPARSE = 4
RAC_OPT_DENSE = 8
RAC_LAYOUT_DENSE = 0
RAC_LAYOUT_SPARSE = 1
RAC_MAX_DOM = 64
RAC_MAX_DOM_WIDE = 256
RAC_NCCL_ID_BYTES = 128
RAC_MAX_RANKS = 8
RAC_IPC_HANDLE_BYTES = 64

_ERRNAMES = {RAC_EINVAL: "RAC_EINVAL", RAC_ENOMEM: "RAC_ENOMEM", RAC_ECUDA: "RAC_ECUDA", RAC_ENCCL: "RAC_ENCCL",
             RAC_ESTATE: "RAC_ESTATE", RAC_EUNSUPPORTED: "RAC_EUNSUPPORTED", RAC_EPEER: "RAC_EPEER"}


class RacError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__("%s (%d): %s" % (_ERRNAMES.get(code, "RAC_E?"), code, msg))
        self.code = code


class rac_relation(ctypes.Structure):
    _fields_ = [("x", ctypes.c_int32), ("y", ctypes.c_int32), ("rows", ctypes.POINTER(ctypes.c_uint64))]


class rac_search_stats(ctypes.Structure):
    _fields_ = [("assignments", ctypes.c_int64), ("recurrences", ctypes.c_int64), ("wipeouts", ctypes.c_int64),
                ("solutions", ctypes.c_int64), ("max_depth", ctypes.c_int64), ("root_iterations", ctypes.c_int32),
                ("root_status", ctypes.c_int32), ("enforce_seconds", ctypes.c_double)]


class rac_options(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("flags", ctypes.c_uint32), ("rank", ctypes.c_int32),
                ("world", ctypes.c_int32), ("nccl_unique_id", ctypes.c_void_p), ("virtual_shards", ctypes.c_int32),
                ("max_ctas", ctypes.c_int32)]


# Every symbol include/rac.h declares (checked by tests/test_abi.py).
EXPORTS = ["rac_default_options", "rac_create", "rac_create_random", "rac_enforce", "rac_enforce_ex",
           "rac_enforce_async", "rac_enforce_batch", "rac_enforce_seeded", "rac_enforce_seeded_async",
           "rac_enforce_batch_seeded", "rac_search", "rac_batch_pass_eval", "rac_n_vars", "rac_max_dom", "rac_mask_bytes", "rac_words_per_var",
           "rac_layout", "rac_relation_bytes", "rac_shard_range", "rac_local_range", "rac_read_row", "rac_get_nccl_unique_id",
           "rac_peer_handle", "rac_connect_peers", "rac_peer_region", "rac_connect_peers_local",
           "rac_last_launch_count", "rac_full_pass_layout", "rac_path", "rac_last_error", "rac_destroy"]

PATHS = {0: "fused", 1: "one_block", 2: "sparse", 3: "sharded", 4: "peer", 5: "wide"}


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError("librac.so not built (%s); run `python -c 'import __graft_entry__ as g; g.build()'`"
                          % LIB_PATH)
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    P = ctypes.c_void_p
    i32, u32, i64, u64 = ctypes.c_int32, ctypes.c_uint32, ctypes.c_int64, ctypes.c_uint64
    i32p = ctypes.POINTER(ctypes.c_int32)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    sig = {
        "rac_default_options": (None, [ctypes.POINTER(rac_options)]),
        "rac_create": (ctypes.c_int, [i32, i32p, i32, ctypes.POINTER(rac_relation), ctypes.POINTER(rac_options),
                                      ctypes.POINTER(P)]),
        "rac_create_random": (ctypes.c_int, [i32, i32, u64, u32, u64, ctypes.POINTER(rac_options),
                                             ctypes.POINTER(P)]),
        # the blocking host-buffer calls take addresses (ints): see _addr()
        "rac_enforce": (ctypes.c_int, [P, P, P, P]),
        "rac_enforce_ex": (ctypes.c_int, [P, P, P, P, P, u32]),
        "rac_enforce_async": (ctypes.c_int, [P, P, P, P, P, P, u32, P]),
        "rac_enforce_batch": (ctypes.c_int, [P, i32, P, P, P, P, u32, P]),
        "rac_enforce_seeded": (ctypes.c_int, [P, P, P, P, P, i32, u32]),
        "rac_enforce_seeded_async": (ctypes.c_int, [P, P, P, P, P, P, i32, u32, P]),
        "rac_enforce_batch_seeded": (ctypes.c_int, [P, i32, P, P, P, P, P, u32, P]),
        "rac_search": (ctypes.c_int, [P, u64p, ctypes.c_int64, u32, i32p, ctypes.POINTER(rac_search_stats)]),
        "rac_batch_pass_eval": (ctypes.c_int, [P, i32, i32, P, P, P]),
        "rac_n_vars": (i32, [P]),
        "rac_max_dom": (i32, [P]),
        "rac_mask_bytes": (i32, [P]),
        "rac_words_per_var": (i32, [P]),
        "rac_layout": (i32, [P]),
        "rac_relation_bytes": (i64, [P]),
        "rac_shard_range": (ctypes.c_int, [i32, i32, i32, i32p, i32p]),
        "rac_local_range": (ctypes.c_int, [P, i32p, i32p]),
        "rac_read_row": (ctypes.c_int, [P, i32, i32, u64p, ctypes.POINTER(ctypes.c_uint8)]),
        "rac_get_nccl_unique_id": (ctypes.c_int, [P]),
        "rac_peer_handle": (ctypes.c_int, [P, P]),
        "rac_connect_peers": (ctypes.c_int, [P, P]),
        "rac_peer_region": (ctypes.c_int, [P, ctypes.POINTER(P)]),
        "rac_connect_peers_local": (ctypes.c_int, [P, ctypes.POINTER(P), i32p]),
        "rac_last_launch_count": (i64, [P]),
        "rac_full_pass_layout": (i32, [P, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]),
        "rac_path": (i32, [P]),
        "rac_last_error": (ctypes.c_char_p, [P]),
        "rac_destroy": (None, [P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def _u64p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def _i32p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def _addr(a: np.ndarray) -> int:
    """Address of a C-contiguous array's data (marshalling only).  `a.ctypes.data`
    costs ~1.4 us per call; a ctypes view of the buffer ~0.4 us (writable arrays)."""
    try:
        return ctypes.addressof(ctypes.c_char.from_buffer(a))
    except (TypeError, ValueError):
        return a.ctypes.data


_U64 = np.dtype(np.uint64)
_I32 = np.dtype(np.int32)


def _as_u64(a, nw: int) -> np.ndarray:
    """d_in as a contiguous uint64 vector of nw words (no copy when it already is one)."""
    if type(a) is np.ndarray and a.dtype is _U64 and a.flags.c_contiguous and a.size == nw:
        return a.reshape(-1) if a.ndim != 1 else a
    a = np.ascontiguousarray(a, dtype=np.uint64).reshape(-1)
    if a.size != nw:
        raise ValueError("d_in must have shape (n_vars * words_per_var,)")
    return a


def last_error(ctx=None) -> str:
    s = lib.rac_last_error(ctx)
    return s.decode() if s else ""


def _check(rc: int, ctx=None) -> int:
    if rc < 0:
        raise RacError(rc, last_error(ctx))
    return rc


def rac_shard_range(n_vars: int, world: int, rank: int) -> Tuple[int, int]:
    lo, hi = ctypes.c_int32(0), ctypes.c_int32(0)
    _check(lib.rac_shard_range(n_vars, world, rank, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def rac_get_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(RAC_NCCL_ID_BYTES)
    _check(lib.rac_get_nccl_unique_id(buf))
    return buf.raw


def make_options(device: int = 0, rank: int = 0, world: int = 1, nccl_unique_id: Optional[bytes] = None,
                 virtual_shards: int = 0, nccl_self: bool = False, peer: bool = False, max_ctas: int = 0,
                 layout: str = "auto"):
    o = rac_options()
    lib.rac_default_options(ctypes.byref(o))
    o.device, o.rank, o.world, o.virtual_shards, o.max_ctas = device, rank, world, virtual_shards, max_ctas
    o.flags = (RAC_OPT_NCCL_SELF if nccl_self else 0) | (RAC_OPT_PEER if peer else 0) | \
        {"auto": 0, "sparse": RAC_OPT_SPARSE, "dense": RAC_OPT_DENSE}[layout]
    keep = None
    if nccl_unique_id is not None:
        keep = ctypes.create_string_buffer(bytes(nccl_unique_id), RAC_NCCL_ID_BYTES)
        o.nccl_unique_id = ctypes.cast(keep, ctypes.c_void_p)
    return o, keep


def _stream_ptr(stream) -> int:
    if stream is None:
        try:
            import torch
            return int(torch.cuda.current_stream().cuda_stream)
        except Exception:  # pragma: no cover - no torch / no cuda
            return 0
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


def _ptr(t) -> int:
    if t is None:
        return 0
    if isinstance(t, int):
        return t
    return int(t.data_ptr())


class RacContext:
    """Owning wrapper of a rac_ctx*."""

    def __init__(self, handle, n: int, dmax: int):
        self._h = handle
        self.n = n
        self.dmax = dmax
        self.wq = int(lib.rac_words_per_var(handle))  # words per variable of every domain state
        self._it = ctypes.c_int32(0)  # the blocking calls' iteration count (read right after each call)
        self._it_addr = ctypes.addressof(self._it)

    # ---- creation
    @classmethod
    def create(cls, n_vars: int, dom_sizes, xs, ys, rows, device: int = 0, rank: int = 0, world: int = 1,
               nccl_unique_id: Optional[bytes] = None, virtual_shards: int = 0,
               nccl_self: bool = False, peer: bool = False, max_ctas: int = 0,
               layout: str = "auto") -> "RacContext":
        """rac_create from relation arrays: constraint k on (xs[k], ys[k]) with
        rows[k, a] = c_xy|(x,a) bitsets (uint64); wide domains (max dom > 64):
        rows[k, a, w] = word w of the bitset, w < ceil(max dom / 64)."""
        dom = np.ascontiguousarray(dom_sizes, dtype=np.int32)
        xs = np.ascontiguousarray(xs, dtype=np.int32)
        ys = np.ascontiguousarray(ys, dtype=np.int32)
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        m = xs.shape[0]
        rel = (rac_relation * max(m, 1))()
        if m:
            stride = rows.strides[0]
            base = rows.ctypes.data
            arr = np.frombuffer(rel, dtype=np.dtype([("x", np.int32), ("y", np.int32), ("rows", np.uint64)]),
                                count=m)
            arr["x"] = xs
            arr["y"] = ys
            arr["rows"] = base + stride * np.arange(m, dtype=np.uint64)
        opt, keep = make_options(device, rank, world, nccl_unique_id, virtual_shards, nccl_self, peer, max_ctas,
                                 layout)
        h = ctypes.c_void_p()
        rc = lib.rac_create(n_vars, _i32p(dom), m, rel if m else None, ctypes.byref(opt), ctypes.byref(h))
        _check(rc)
        del keep
        return cls(h, n_vars, int(dom.max()))

    @classmethod
    def from_instance(cls, inst, **kw) -> "RacContext":
        return cls.create(inst.n, inst.dom, inst.xs, inst.ys, inst.rows, **kw)

    @classmethod
    def create_random(cls, n_vars: int, d: int, dens_q32: int, t_q16: int, seed: int, device: int = 0,
                      rank: int = 0, world: int = 1, nccl_unique_id: Optional[bytes] = None,
                      virtual_shards: int = 0, nccl_self: bool = False, peer: bool = False,
                      max_ctas: int = 0, layout: str = "auto") -> "RacContext":
        opt, keep = make_options(device, rank, world, nccl_unique_id, virtual_shards, nccl_self, peer, max_ctas,
                                 layout)
        h = ctypes.c_void_p()
        _check(lib.rac_create_random(n_vars, d, dens_q32, t_q16, seed, ctypes.byref(opt), ctypes.byref(h)))
        del keep
        return cls(h, n_vars, d)

    @property
    def full_pass_layout(self):
        """(layout, ms_columns, ms_rows): the sweep of full passes ("rows" / "columns") and the
        create-time calibration times (0 when not measured)."""
        a, b = ctypes.c_float(0), ctypes.c_float(0)
        r = int(lib.rac_full_pass_layout(self._h, ctypes.byref(a), ctypes.byref(b)))
        return ("columns" if r == 1 else "rows"), round(a.value, 5), round(b.value, 5)

    def close(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.rac_destroy(self._h)
        self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- enforcement
    def enforce(self, d_in, full: bool = False, removed_at: bool = False):
        """rac_enforce / rac_enforce_ex with host buffers.
        Returns (status, d_out, iterations[, removed_at[n, 64*wq]]); domain states
        are [n_vars * wq] words (wq = 1 unless the domains are wider than 64)."""
        nw = self.n * self.wq
        d_in = _as_u64(d_in, nw)
        d_out = np.empty(nw, dtype=np.uint64)
        it = self._it
        if full or removed_at:
            rem = np.zeros(self.n * 64 * self.wq, dtype=np.int32) if removed_at else None
            rc = lib.rac_enforce_ex(self._h, _addr(d_in), _addr(d_out), self._it_addr,
                                    _addr(rem) if rem is not None else None, RAC_FULL_FIXPOINT if full else 0)
            _check(rc, self._h)
            if removed_at:
                return rc, d_out, it.value, rem.reshape(self.n, 64 * self.wq)
            return rc, d_out, it.value
        rc = lib.rac_enforce(self._h, _addr(d_in), _addr(d_out), self._it_addr)
        if rc < 0:
            _check(rc, self._h)
        return rc, d_out, it.value

    def enforce_seeded(self, d_in, seeds, full: bool = False):
        """rac_enforce_seeded (Alg. 1 tensorAC(Vars, @changed = seeds)), host buffers.
        Returns (status, d_out, iterations)."""
        nw = self.n * self.wq
        d_in = _as_u64(d_in, nw)
        if not (type(seeds) is np.ndarray and seeds.dtype is _I32 and seeds.flags.c_contiguous):
            seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.int32).reshape(-1))
        d_out = np.empty(nw, dtype=np.uint64)
        ns = seeds.size
        rc = lib.rac_enforce_seeded(self._h, _addr(d_in), _addr(d_out), self._it_addr,
                                    _addr(seeds) if ns else None, ns, RAC_FULL_FIXPOINT if full else 0)
        if rc < 0:
            _check(rc, self._h)
        return rc, d_out, self._it.value

    def enforce_seeded_async(self, d_in_dev, d_out_dev, iters_dev, status_dev, seeds_dev, n_seeds: int,
                             full: bool = False, stream=None) -> None:
        _check(lib.rac_enforce_seeded_async(self._h, _ptr(d_in_dev), _ptr(d_out_dev), _ptr(iters_dev),
                                            _ptr(status_dev), _ptr(seeds_dev), n_seeds,
                                            RAC_FULL_FIXPOINT if full else 0, _stream_ptr(stream)), self._h)

    def enforce_batch_seeded(self, n_states: int, d_in_dev, d_out_dev, iters_dev, status_dev, seed_var_dev,
                             full: bool = False, stream=None) -> None:
        """rac_enforce_batch_seeded: state s seeded with variable seed_var_dev[s] (-1 = all)."""
        _check(lib.rac_enforce_batch_seeded(self._h, n_states, _ptr(d_in_dev), _ptr(d_out_dev), _ptr(iters_dev),
                                            _ptr(status_dev), _ptr(seed_var_dev), RAC_FULL_FIXPOINT if full else 0,
                                            _stream_ptr(stream)), self._h)

    def search(self, d_in, max_assignments: int = 0, all_solutions: bool = False, full: bool = False):
        """rac_search: Alg. 2 backtracking search with seeded enforcement per assignment.
        Returns (result, solution or None, stats dict).  Domain states of wide
        contexts are [n_vars * words_per_var] words."""
        d_in = np.ascontiguousarray(d_in, dtype=np.uint64).reshape(-1)
        sol = np.full(self.n, -1, dtype=np.int32)
        st = rac_search_stats()
        flags = (RAC_SEARCH_ALL if all_solutions else 0) | (RAC_FULL_FIXPOINT if full else 0)
        rc = lib.rac_search(self._h, _u64p(d_in), int(max_assignments), flags, _i32p(sol), ctypes.byref(st))
        _check(rc, self._h)
        stats = {k: getattr(st, k) for k, _ in rac_search_stats._fields_}
        return rc, (sol if rc == RAC_OK else None), stats

    def batch_pass_eval(self, impl: int, n_states: int, d_in_dev, d_out_dev, stream=None) -> None:
        """rac_batch_pass_eval: one Eq. 1 pass for n_states states (0 = bit-sliced, 1 = tcgen05)."""
        _check(lib.rac_batch_pass_eval(self._h, impl, n_states, _ptr(d_in_dev), _ptr(d_out_dev),
                                       _stream_ptr(stream)), self._h)

    def enforce_async(self, d_in_dev, d_out_dev, iters_dev, status_dev, removed_at_dev=None, full: bool = False,
                      stream=None) -> None:
        """rac_enforce_async on device buffers (torch tensors or raw pointers)."""
        _check(lib.rac_enforce_async(self._h, _ptr(d_in_dev), _ptr(d_out_dev), _ptr(iters_dev), _ptr(status_dev),
                                     _ptr(removed_at_dev), RAC_FULL_FIXPOINT if full else 0, _stream_ptr(stream)),
               self._h)

    def enforce_batch(self, n_states: int, d_in_dev, d_out_dev, iters_dev, status_dev, full: bool = False,
                      stream=None) -> None:
        """rac_enforce_batch on device buffers: [n_states, n] uint64 states."""
        _check(lib.rac_enforce_batch(self._h, n_states, _ptr(d_in_dev), _ptr(d_out_dev), _ptr(iters_dev),
                                     _ptr(status_dev), RAC_FULL_FIXPOINT if full else 0, _stream_ptr(stream)),
               self._h)

    # ---- peer-memory exchange (RAC_OPT_PEER)
    def peer_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(RAC_IPC_HANDLE_BYTES)
        _check(lib.rac_peer_handle(self._h, buf), self._h)
        return buf.raw

    def connect_peers(self, handles: Sequence[bytes]) -> None:
        """handles[q] = rank q's peer_handle() (world entries, rank order)."""
        blob = b"".join(bytes(h) for h in handles)
        buf = ctypes.create_string_buffer(blob, len(blob))
        _check(lib.rac_connect_peers(self._h, buf), self._h)

    def peer_region(self) -> int:
        p = ctypes.c_void_p()
        _check(lib.rac_peer_region(self._h, ctypes.byref(p)), self._h)
        return int(p.value or 0)

    def connect_peers_local(self, regions: Sequence[int], devices: Sequence[int]) -> None:
        """Ranks driven by this one process: regions[q] = rank q's peer_region()."""
        arr = (ctypes.c_void_p * len(regions))(*regions)
        dev = np.ascontiguousarray(devices, dtype=np.int32)
        _check(lib.rac_connect_peers_local(self._h, arr, _i32p(dev)), self._h)

    # ---- introspection
    @property
    def mask_bytes(self) -> int:
        return int(lib.rac_mask_bytes(self._h))

    @property
    def layout(self) -> str:
        """"dense" or "sparse" (arc blocks, rac.h RAC_OPT_SPARSE)."""
        return "sparse" if int(lib.rac_layout(self._h)) == RAC_LAYOUT_SPARSE else "dense"

    @property
    def relation_bytes(self) -> int:
        return int(lib.rac_relation_bytes(self._h))

    @property
    def last_launch_count(self) -> int:
        return int(lib.rac_last_launch_count(self._h))

    @property
    def path(self) -> str:
        """rac_path: which kernel runs a single-state enforcement ("fused", "one_block", ...)."""
        return PATHS[int(lib.rac_path(self._h))]

    def local_range(self) -> Tuple[int, int]:
        lo, hi = ctypes.c_int32(0), ctypes.c_int32(0)
        _check(lib.rac_local_range(self._h, ctypes.byref(lo), ctypes.byref(hi)), self._h)
        return lo.value, hi.value

    def read_row(self, x: int, a: int) -> Tuple[np.ndarray, np.ndarray]:
        masks = np.zeros(self.n, dtype=np.uint64)
        pres = np.zeros(self.n, dtype=np.uint8)
        _check(lib.rac_read_row(self._h, x, a, _u64p(masks), pres.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))),
               self._h)
        return masks, pres
