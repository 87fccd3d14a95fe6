"""Build libsmgpu.so in-tree with nvcc for sm_100a (no JIT cache, no torch build)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libsmgpu.so")
LIB_DEBUG = os.path.join(HERE, "libsmgpu_debug.so")
LIB_COUNTERS = os.path.join(HERE, "libsmgpu_counters.so")

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "--expt-relaxed-constexpr",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(INCLUDE, "*.h")) + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, debug: bool = False, counters: bool = False) -> str:
    """debug=True: libsmgpu_debug.so with device-side bounds assertions (-DSMGPU_DEBUG_CHECKS);
    counters=True: libsmgpu_counters.so with compare-step counters (-DSMGPU_COUNTERS)."""
    lib = LIB_DEBUG if debug else (LIB_COUNTERS if counters else LIB)
    if not force and not _stale(lib):
        return lib
    objdir = os.path.join(HERE, "build_debug" if debug else ("build_counters" if counters else "build"))
    defs = (["-DSMGPU_DEBUG_CHECKS"] if debug else []) + (["-DSMGPU_COUNTERS"] if counters else [])
    os.makedirs(objdir, exist_ok=True)
    # outputs get the build's START time as mtime: a source edited while nvcc runs stays newer
    t_start = time.time()
    objs = []
    procs = []
    # an object is rebuilt when it is older than its source, any header, or this script
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(INCLUDE, "*.h")) + [__file__]
    newest_header = max(os.path.getmtime(h) for h in headers)
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if not force and os.path.exists(obj) and \
                os.path.getmtime(obj) >= max(os.path.getmtime(src), newest_header):
            continue
        cmd = ["nvcc", *NVCC_FLAGS, *defs, "-I", INCLUDE, "-I", CSRC,
               "-c", src, "-o", obj + ".tmp.o"]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = False
    for src, obj, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out.decode(errors="replace"))
        if p.returncode != 0:
            failed = True
        else:
            os.replace(obj + ".tmp.o", obj)
            os.utime(obj, (t_start, t_start))
    if failed:
        raise RuntimeError("nvcc failed")
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call(["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs])
    os.replace(tmp, lib)
    os.utime(lib, (t_start, t_start))
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv,
                counters="--counters" in sys.argv))
