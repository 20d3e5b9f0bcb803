"""Build librac.so (sm_100a) in-tree with nvcc.  No torch types are involved:
the library is a plain C ABI (include/rac.h) over CUDA kernels."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librac.so")
SOURCES = ["rac_api.cu", "rac_kernels.cu", "rac_pack.cu", "rac_batch.cu", "rac_batch_tc.cu", "rac_wide.cu", "rac_state.cu", "rac_batch_cl.cu", "rac_wide_tc.cu"]
DEPS = SOURCES + ["rac_internal.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _source_hash(defines=()) -> str:
    """sha256 over every source the library is built from, the nvcc flags and the
    nvcc version.  Stored next to librac.so: a library whose stamp differs (or
    is missing) is rebuilt, so a .so copied from another machine, or one older
    than the sources whatever the file times say, is never used."""
    import hashlib
    h = hashlib.sha256()
    deps = [os.path.join(CSRC, f) for f in DEPS] + [os.path.join(ROOT, "include", "rac.h"),
                                                      os.path.join(ROOT, "synth", "csp_synth.h")]
    for d in deps:
        with open(d, "rb") as f:
            h.update(os.path.basename(d).encode() + b"\0" + f.read())
    h.update(" ".join(ARCH + ["-O3", "-lineinfo"] + list(defines)).encode())
    try:
        h.update(subprocess.run([nvcc_path(), "--version"], capture_output=True, text=True).stdout.encode())
    except Exception:
        pass
    return h.hexdigest()


def _stale() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(LIB + ".srchash"):
        return True
    with open(LIB + ".srchash") as f:
        return f.read().strip() != _source_hash()


def build(force: bool = False, verbose: bool = False, out: str = None, defines=(), src_dir: str = None) -> str:
    """src_dir (A/B tooling, with `out`): build from another copy of csrc/ (e.g. an older revision)."""
    lib = out or LIB
    csrc = src_dir or CSRC
    if not force and out is None and not _stale():
        return LIB
    tmp = lib + ".tmp.%d" % os.getpid()
    objdir = tmp + ".obj"
    os.makedirs(objdir, exist_ok=True)
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
             "-Xptxas", "-v" if verbose else "-O3"] + ["-D" + d for d in defines]
    objs = [os.path.join(objdir, s.replace(".cu", ".o")) for s in SOURCES]

    def compile_one(i):
        return subprocess.run([nvcc_path(), *flags, "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(ROOT, "synth"),
                               "-c", os.path.join(csrc, SOURCES[i]), "-o", objs[i]],
                              capture_output=True, text=True)

    # one nvcc per translation unit, in parallel (rac_kernels.cu dominates)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(len(SOURCES)) as ex:
        results = list(ex.map(compile_one, range(len(SOURCES))))
    results.append(subprocess.run([nvcc_path(), *ARCH, "-shared", "-o", tmp] + objs + ["-ldl"],
                                  capture_output=True, text=True))
    shutil.rmtree(objdir, ignore_errors=True)
    for res in results:
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed building librac.so")
        if verbose:
            sys.stderr.write(res.stderr)
    os.replace(tmp, lib)
    if out is None and not defines and src_dir is None:
        with open(LIB + ".srchash", "w") as f:
            f.write(_source_hash() + "\n")
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force=True, verbose="-v" in sys.argv, out=outs[0] if outs else None, defines=defs))
