"""Build libprngd_b200.so in-tree with nvcc for sm_100a (no GPU needed to build).

    python -m paper_1401_8230_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libprngd_b200.so")
SOURCES = [os.path.join(CSRC, f) for f in ("prngd_kernels.cu", "prngd_host.cpp", "prngd_jump.cpp",
                                           "prngd_mc.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("prngd_device.cuh", "prngd_internal.h")] + [
    os.path.join(ROOT, "include", "prngd.h"), os.path.abspath(__file__)]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-ffp-contract=off", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Build the library (to `out` with extra -D `defines` for A/B variants)."""
    lib = out or LIB
    if not (force or out or _stale()):
        return LIB
    objs = []
    objdir = tempfile.mkdtemp(prefix="prngd_build_")  # per build: variant builds may run in parallel
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        else:
            cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-Wno-deprecated-gpu-targets",
                   "-x", "c++", "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(obj)
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", tmp, *objs,
           "-Xlinker", "-rpath,/usr/local/cuda/lib64", "-Xcompiler", "-fvisibility=hidden"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, lib)
    shutil.rmtree(objdir, ignore_errors=True)
    return lib


TOOL_SRC = os.path.join(ROOT, "tools", "write_ceiling.cu")
TOOL_LIB = os.path.join(ROOT, "tools", "libwriteceil.so")


def build_tools(force: bool = False) -> str:
    """B13 write-roofline microbenchmark used by bench.py (measurement only)."""
    if force or not os.path.exists(TOOL_LIB) or os.path.getmtime(TOOL_LIB) < os.path.getmtime(TOOL_SRC):
        cmd = [NVCC, *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-cudart",
               "shared", "-o", TOOL_LIB, TOOL_SRC]
        subprocess.check_call(cmd)
    return TOOL_LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--out", default=None, help="variant output path (A/B experiments)")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose, out=a.out, defines=tuple(a.defines)))
    print(build_tools(force=a.force))
