"""Build libtqr.so in-tree: C++ schedule compiler + sm_100a CUDA engine.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo; cudart linked
statically so the library loads without a GPU (schedule-only use on CPU).
Object files are cached in build/ keyed on source mtimes.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
# TQR_BUILD_DIR / TQR_LIB_OUT: separate object dir and output for instrumented
# builds (TQR_EXTRA_NVCC_FLAGS), so they never mix with the product library
BUILD = os.environ.get("TQR_BUILD_DIR") or os.path.join(ROOT, "build")
OUT = os.environ.get("TQR_LIB_OUT") or os.path.join(HERE, "libtqr.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CXXFLAGS = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-lineinfo", "-I", os.path.join(ROOT, "include")]
# experiment hook (ablation macros); changing it requires a clean build/
CXXFLAGS += os.environ.get("TQR_EXTRA_NVCC_FLAGS", "").split()
HEADERS = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh"))] + \
    [os.path.join(ROOT, "include", "tqr.h")]


def _stale(obj, src):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in [src] + HEADERS)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))
    return r


def build(verbose=False):
    os.makedirs(BUILD, exist_ok=True)
    objs, jobs = [], []
    for src in sorted(os.listdir(CSRC)):
        if not src.endswith((".cpp", ".cu")):
            continue
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if _stale(obj, path):
            cmd = [NVCC] + ARCH + CXXFLAGS + ["-c", path, "-o", obj]
            if src.endswith(".cu"):
                cmd += ["-Xptxas", "-v"] if verbose else []
            else:
                cmd += ["-x", "c++"]
            if verbose:
                print(" ".join(cmd))
            jobs.append(cmd)
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for r in ex.map(_run, jobs):
            if verbose:
                sys.stdout.write(r.stdout + r.stderr)
    if not os.path.exists(OUT) or any(os.path.getmtime(o) > os.path.getmtime(OUT) for o in objs):
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", OUT] + objs + ["-lpthread", "-ldl", "-lrt"])
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
