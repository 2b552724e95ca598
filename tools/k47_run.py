"""C3 expand + covariance + eig + project on `n` images (default 16384): the K4 / K5 / K7 launches to profile.
usage: python tools/k47_run.py [n]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1412_0781_b200 as F  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
cfg = synth.config("C3")
imgs = synth.blob_images(cfg, 0, n, device=torch.device("cuda:0"))
plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], device=0, max_batch=n)
for _ in range(2):
    coeffs = F.fbspca_expand(plan, imgs)
    blocks, mean = F.fbspca_covariance(plan, coeffs)
    evals, evecs = F.fbspca_eig(plan, blocks)
    out = F.fbspca_project(plan, coeffs, mean, evals, evecs, sigma2=1.0, mode=1)
torch.cuda.synchronize()
print("k47 run ok", n)
