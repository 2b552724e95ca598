"""Small invocations of every library kernel family, for compute-sanitizer (memcheck / racecheck / synccheck).
usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1412_0781_b200 as F  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")


def run(name, L, c, R, n, dtype=F.F32, eps=0.0, max_batch=64):
    if name in synth.CONFIGS:
        cfg = synth.config(name)
        imgs = synth.blob_images(cfg, 0, n, device=dev) if dtype == F.F32 else None
    if name not in synth.CONFIGS or imgs is None:
        rng = np.random.default_rng(L)
        imgs = torch.from_numpy(rng.standard_normal((n, L, L))).to(dev)
        imgs = imgs.float() if dtype == F.F32 else imgs
    plan = F.fbspca_plan(L, c, R, eps=eps, dtype=dtype, device=0, max_batch=max_batch)
    coeffs = F.fbspca_expand(plan, imgs)
    blocks, mean = F.fbspca_covariance(plan, coeffs)
    evals, evecs = F.fbspca_eig(plan, blocks)
    out = F.fbspca_project(plan, coeffs, mean, evals, evecs, sigma2=1.0, mode=1)
    F.fbspca_radial_eigenfunctions(plan, evecs)
    ahat = F.fbspca_backproject(plan, out, mean, evecs)
    F.fbspca_synthesize(plan, ahat[:, :2].contiguous())
    if n <= 64:
        F.fbspca_svd(plan, coeffs)
    torch.cuda.synchronize()
    print(f"{name} L={L} M={plan.M} w={plan.w} dtype={'f32' if dtype == F.F32 else 'f64'}: ok", flush=True)


which = sys.argv[1:] or ["pow2", "runtime", "fp64", "tc"]
if "pow2" in which:
    run("C2", 64, 0.5, 32.0, 10)                      # compile-time M = 128 polar kernel, tcgen05 K4/K5
if "runtime" in which:
    run("C2", 64, 0.5, 32.0, 6, eps=1e-6)             # runtime-radix w = 7 polar kernel
    run("x", 40, 0.5, 20.0, 5)                        # runtime M = 80
if "fp64" in which:
    run("x", 32, 0.5, 16.0, 6, dtype=F.F64)           # <double, 13, 64>
    run("x", 33, 0.5, 16.0, 4, dtype=F.F64)           # <double, 13, 0>
if "tc" in which:
    run("C3", 128, 0.5, 64.0, 150, max_batch=160)     # M = 256 kernel, K4 with > 1 row tile, K5 b = 64
print("sanitize run done")
