"""Build libfbspca.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = (["csrc/plan.cpp", "csrc/kernels_polar.cu"] + [f"csrc/polar_part{i}.cu" for i in range(1, 7)] +
       ["csrc/kernels_linalg.cu", "csrc/kernels_tma.cu", "csrc/kernels_synth.cu", "csrc/kernels_params.cu", "csrc/capi.cu"])
HDR = ["csrc/internal.h", "csrc/fft_device.cuh", "csrc/kernels_polar.cu", os.path.join("..", "include", "fbspca.h")]
LIB = os.path.join(PKG, "lib", "libfbspca.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    hdrs = [os.path.join(PKG, h) for h in HDR]
    procs, objs = [], []
    for s in SRC:
        src = os.path.join(PKG, s)
        obj = os.path.join(objdir, os.path.basename(s) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            cmd = [NVCC] + FLAGS + ["-c", src, "-o", obj]
            log = open(obj + ".log", "w")
            procs.append((s, subprocess.Popen(cmd, stdout=log, stderr=subprocess.STDOUT), obj + ".log"))
    for s, p, logf in procs:
        if p.wait() != 0:
            sys.stderr.write(open(logf).read())
            raise RuntimeError(f"nvcc failed on {s}; see {logf}")
        if verbose:
            sys.stdout.write(open(logf).read())
    if force or procs or _stale(LIB, objs):
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB] + objs + ["-ldl"]
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
