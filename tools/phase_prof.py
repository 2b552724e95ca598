"""Per-stage cycle breakdown of the polar kernel (debug build with -DFBSPCA_PHASE_PROF).

    python tools/phase_prof.py [--n 4096] [--config C3]
Builds paper_1412_0781_b200/lib_prof/libfbspca.so if needed, runs one expand, prints cycles/image/stage."""
import argparse
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PROF_LIB = os.path.join(ROOT, "paper_1412_0781_b200", "lib_prof", "libfbspca.so")


def build():
    from paper_1412_0781_b200 import build as B
    os.makedirs(os.path.dirname(PROF_LIB), exist_ok=True)
    objs = []
    for src in B.SRC:
        obj = os.path.join("/tmp", "prof_" + os.path.basename(src) + ".o")
        subprocess.check_call([B.NVCC] + [f for f in B.FLAGS if f != "-v" and f != "-Xptxas"] +
                              ["-DFBSPCA_PHASE_PROF", "-DFBSPCA_POLAR_SINGLE_TU", "-c", os.path.join(B.PKG, src), "-o", obj])
        objs.append(obj)
    subprocess.check_call([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", PROF_LIB] + objs + ["-ldl"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--build-only", action="store_true")
    a = ap.parse_args()
    if not os.path.exists(PROF_LIB):
        build()
    if a.build_only:
        return
    import paper_1412_0781_b200._lib as LB
    LB.LIB_PATH = PROF_LIB
    import torch
    import paper_1412_0781_b200 as F
    import synth
    cfg = synth.config(a.config)
    imgs = synth.blob_images(cfg, 0, a.n, device="cuda", sigma_n=1.0)
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], device=0, max_batch=a.n)
    F.fbspca_expand(plan, imgs)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (148 * 8))()
    LB.lib().fbspca_debug_phase_prof(buf, 148 * 8)
    names = ["rowpass", "fill", "colfft", "gather", "ang-wait", "write", "ang-U", "ang-V"]
    per = [sum(buf[b * 8 + i] for b in range(148)) / a.n for i in range(8)]
    tot = sum(per)
    for nm, v in zip(names, per):
        if v:
            print(f"{nm:10s} {v:12.0f} cycles/image  {100 * v / tot:5.1f}%")
    print(f"{'total':10s} {tot:12.0f} cycles/image per CTA")


if __name__ == "__main__":
    main()
