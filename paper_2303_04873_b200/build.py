"""Build libmorea.so (the C-ABI + sm_100a kernels) in-tree with nvcc."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libmorea.so")
# the same sources with device-side index and invariant checks (MOREA_CHECK -> assert);
# used by tests/test_gpu_debug_checks.py only
LIB_DEBUG = os.path.join(PKG, "libmorea_debug.so")
SOURCES = ["morea_kernels.cu", "morea_api.cu"]
HEADERS = [os.path.join(CSRC, h) for h in ("morea_internal.h", "morea_sobol_setup.cuh", "morea_sobol.cuh", "morea_repair.cuh", "morea_export.cuh", "morea_mix.cuh")] + \
    [os.path.join(INCLUDE, "morea.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=default",
    "-Xptxas", "-v",
]


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + HEADERS + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    lib = out or LIB
    if not force and out is None and not _stale():
        return LIB
    tag = "" if out is None else ".alt"
    objs, procs = [], []
    for s in SOURCES:  # the translation units compile in parallel
        src = os.path.join(CSRC, s)
        obj = os.path.join(CSRC, s.replace(".cu", tag + ".o"))
        cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", INCLUDE, "-I", CSRC, "-c", src, "-o", obj]
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        objs.append(obj)
    for s, p in procs:
        so, se = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(so + se)
            raise RuntimeError(f"nvcc failed on {s}")
        if verbose:
            sys.stderr.write(se)
        if out is None:  # the resource report of this build (compile times dropped: reproducible)
            with open(os.path.join(CSRC, s + ".ptxas.txt"), "w") as f:
                f.write("".join(l for l in se.splitlines(True) if "Compile time" not in l))
    tmp = lib + ".tmp"
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
           "-Xcompiler", "-fPIC"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, lib)
    return lib


def build_debug(force: bool = False) -> str:
    """libmorea_debug.so: the product sources with -DMOREA_DEBUG_CHECKS."""
    if not force and os.path.exists(LIB_DEBUG) and os.path.getmtime(LIB_DEBUG) >= max(
            os.path.getmtime(d) for d in [os.path.join(CSRC, x) for x in SOURCES] + HEADERS):
        return LIB_DEBUG
    return build(force=True, out=LIB_DEBUG, defines=("MOREA_DEBUG_CHECKS",))


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
