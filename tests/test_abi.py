"""CPU-side checks of the C ABI: librac.so loads, exports every function that
include/rac.h declares, and its host-only logic (argument validation, shard
ranges) behaves as documented.  No compute calls (no GPU here)."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2407_11388_b200 import rac

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "rac.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rac_[a-z_0-9]+)\s*\(", text)))


def test_header_symbols_exported():
    names = header_functions()
    assert len(names) >= 15
    lib = ctypes.CDLL(rac.LIB_PATH)
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(rac.EXPORTS) == names


def test_library_is_sm100a():
    """The shared library carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", rac.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("n,world", [(1, 1), (10, 3), (2000, 8), (8000, 8), (7, 8), (513, 2)])
def test_shard_ranges_partition(n, world):
    """Row blocks are contiguous, disjoint and cover [0, n)."""
    covered = []
    for r in range(world):
        lo, hi = rac.rac_shard_range(n, world, r)
        assert 0 <= lo <= hi <= n
        covered.extend(range(lo, hi))
    assert covered == list(range(n))


def test_create_validation_errors():
    """RAC_EINVAL before any device work: duplicate pair, x == y, out of range,
    bits beyond dom(y), bad domain sizes (include/rac.h rac_create)."""
    bad = [
        (3, [2, 2, 2], [0, 1], [1, 0], [[1, 2], [1, 2]]),   # duplicate pair (either orientation)
        (3, [2, 2, 2], [0], [0], [[1, 2]]),                 # x == y
        (3, [2, 2, 2], [0], [3], [[1, 2]]),                 # y out of range
        (3, [2, 2, 2], [0], [1], [[4, 2]]),                 # bit 2 beyond dom(y) = 2
        (3, [2, 0, 2], [], [], []),                         # dom size 0
        (3, [2, 257, 2], [], [], []),                       # dom size > 256 (RAC_MAX_DOM_WIDE)
    ]
    for n, dom, xs, ys, rows in bad:
        rows = np.asarray(rows, dtype=np.uint64).reshape(len(xs), -1) if xs else np.zeros((0, 1), np.uint64)
        with pytest.raises(rac.RacError) as ei:
            rac.RacContext.create(n, dom, xs, ys, rows)
        assert ei.value.code == rac.RAC_EINVAL
        assert rac.last_error(None)
    h = ctypes.c_void_p()
    assert rac.lib.rac_create(0, None, 0, None, None, ctypes.byref(h)) == rac.RAC_EINVAL


def test_create_random_validation():
    h = ctypes.c_void_p()
    assert rac.lib.rac_create_random(10, 257, 1 << 31, 100, 1, None, ctypes.byref(h)) == rac.RAC_EINVAL
    assert rac.lib.rac_create_random(10, 8, (1 << 32) + 1, 100, 1, None, ctypes.byref(h)) == rac.RAC_EINVAL
    assert rac.lib.rac_create_random(10, 8, 1 << 31, 65537, 1, None, ctypes.byref(h)) == rac.RAC_EINVAL
    assert rac.lib.rac_create_random(0, 8, 1 << 31, 100, 1, None, ctypes.byref(h)) == rac.RAC_EINVAL


def test_null_context_calls():
    assert rac.lib.rac_enforce(None, None, None, None) == rac.RAC_EINVAL
    assert rac.lib.rac_n_vars(None) == rac.RAC_EINVAL
    rac.lib.rac_destroy(None)  # no-op
    assert isinstance(rac.last_error(None), str)


def test_world_options_validation():
    o, keep = rac.make_options(world=2, rank=0, nccl_unique_id=None)
    h = ctypes.c_void_p()
    dom = np.full(4, 2, dtype=np.int32)
    rc = rac.lib.rac_create(4, rac._i32p(dom), 0, None, ctypes.byref(o), ctypes.byref(h))
    assert rc == rac.RAC_EINVAL  # world > 1 without a unique id
    o2, _ = rac.make_options(world=2, rank=0, nccl_unique_id=b"x" * 128, nccl_self=True)
    assert rac.lib.rac_create(4, rac._i32p(dom), 0, None, ctypes.byref(o2), ctypes.byref(h)) == rac.RAC_EINVAL
