"""Time the steps outside the benchmark metric on C3 (1 GPU): K6 eig, Alg. 2 line 5, K7 projection, NEXT-1
back-projection + synthesis, NEXT-2 parameter estimation.  CUDA events on the current stream; one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_0781_b200 as F  # noqa: E402
import synth  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    cfg = synth.config("C3")
    n = cfg["n"]
    dev = torch.device("cuda:0")
    imgs = synth.blob_images(cfg, 0, n, device=dev)
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], device=0, max_batch=25000)
    coeffs = F.fbspca_expand(plan, imgs)
    blocks, mean = F.fbspca_covariance(plan, coeffs)
    evals, evecs = F.fbspca_eig(plan, blocks)
    sigma2 = float(synth.blobs.noise_sigma(cfg, device=dev)) ** 2
    out = {"config": "C3", "n": n}
    out["eig_K6_ms"] = timed(lambda: F.fbspca_eig(plan, blocks))
    out["radial_eigenfunctions_ms"] = timed(lambda: F.fbspca_radial_eigenfunctions(plan, evecs))
    chat = torch.empty_like(coeffs)
    out["project_K7_ms_100k"] = timed(lambda: F.fbspca_project(plan, coeffs, mean, evals, evecs, sigma2, 1, out=chat))
    ahat = torch.empty_like(coeffs)
    out["backproject_ms_100k"] = timed(lambda: F.fbspca_backproject(plan, chat, mean, evecs, out=ahat))
    sub = ahat[:, :4096].contiguous()
    imgs_out = torch.empty((4096, cfg["L"], cfg["L"]), dtype=torch.float32, device=dev)
    out["synthesize_ms_4096"] = timed(lambda: F.fbspca_synthesize(plan, sub, out=imgs_out))
    out["estimate_params_ms_100k"] = timed(lambda: F.fbspca_estimate_params(imgs, 0.999), reps=1)
    s2, R, c = F.fbspca_estimate_params(imgs, 0.999)
    out["estimates"] = {"sigma2": s2, "R": R, "c": c, "sigma2_model": sigma2}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
