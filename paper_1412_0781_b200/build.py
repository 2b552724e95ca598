"""Build libfbspca.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

Staleness is decided by content, not mtimes: every object has a sidecar with the SHA-256 of its source, the
shared headers and the flags; the library has a sidecar with the hash of all sources (also compiled into
fbspca_version(), so a loaded library names the sources it was built from).  A pushed prebuilt .so whose
sidecar does not match the tree is rebuilt."""
from __future__ import annotations

import hashlib
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


def _digest(paths, extra=()) -> str:
    h = hashlib.sha256()
    for p in paths:
        h.update(os.path.basename(p).encode())
        h.update(open(p, "rb").read())
    for e in extra:
        h.update(e.encode())
    return h.hexdigest()[:16]


def source_hash() -> str:
    """Hash of every source and header the library is built from (and the flags)."""
    return _digest([os.path.join(PKG, s) for s in SRC] + [os.path.join(PKG, h) for h in HDR], FLAGS)


def _sidecar(path: str) -> str | None:
    try:
        return open(path + ".hash").read().strip()
    except OSError:
        return None


def build(force: bool = False, verbose: bool = False, lib: str | None = None, defines: tuple = ()) -> str:
    """Build (if stale) the library.  `lib` / `defines` build a variant elsewhere (A/B experiments: e.g.
    lib=".../lib_alt/libfbspca.so", defines=("FBSPCA_TW_RECURRENCE=1",)), loaded with FBSPCA_LIB=<path>."""
    LIB_ = lib or LIB
    extra = [f"-D{d}" for d in defines]
    objdir = os.path.join(PKG, "build" if not defines else "build_" + hashlib.sha256(" ".join(extra).encode()).hexdigest()[:8])
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(os.path.dirname(LIB_), exist_ok=True)
    hdrs = [os.path.join(PKG, h) for h in HDR]
    shash = _digest([os.path.join(PKG, s) for s in SRC] + hdrs, FLAGS + extra)
    if not force and os.path.exists(LIB_) and _sidecar(LIB_) == shash:
        return LIB_                      # built from exactly these sources (objects need not be present)
    procs, objs = [], []
    for s in SRC:
        src = os.path.join(PKG, s)
        obj = os.path.join(objdir, os.path.basename(s) + ".o")
        objs.append(obj)
        flags = FLAGS + extra + ([f'-DFBSPCA_SRC_HASH="{shash}"'] if s.endswith("capi.cu") else [])
        want = _digest([src] + hdrs, flags)
        if force or not os.path.exists(obj) or _sidecar(obj) != want:
            cmd = [NVCC] + flags + ["-c", src, "-o", obj]
            log = open(obj + ".log", "w")
            procs.append((s, subprocess.Popen(cmd, stdout=log, stderr=subprocess.STDOUT), obj, want))
    for s, p, obj, want in procs:
        if p.wait() != 0:
            sys.stderr.write(open(obj + ".log").read())
            raise RuntimeError(f"nvcc failed on {s}; see {obj}.log")
        open(obj + ".hash", "w").write(want + "\n")
        if verbose:
            sys.stdout.write(open(obj + ".log").read())
    if force or procs or not os.path.exists(LIB_) or _sidecar(LIB_) != shash:
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB_] + objs + ["-ldl"]
        subprocess.check_call(cmd)
        open(LIB_ + ".hash", "w").write(shash + "\n")
    return LIB_


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--lib", default=None, help="output path of a variant library")
    ap.add_argument("-D", action="append", default=[], help="extra preprocessor define for a variant")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.v, lib=a.lib, defines=tuple(a.D)))
