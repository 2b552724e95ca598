"""W = 5 window (eps = 1e-4) probe at C3: per-image coefficient rel l2 against the fp64 oracle on n images, for
eps in {1e-5, 1e-4}.  Prints max / mean / p99 of the per-image error."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import paper_1412_0781_b200 as F
import synth
from oracle import fb as O

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = synth.config("C3")
imgs = synth.blob_images(cfg, 0, n, device=torch.device("cuda", 0))
basis = O.build_basis(cfg["c"], cfg["R"])
ref = O.to_flat(O.expand(imgs.double().cpu().numpy(), basis))
for eps in (1e-5, 1e-4):
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], eps=eps, device=0, max_batch=n)
    got = F.fbspca_expand(plan, imgs).cpu().numpy().astype(np.complex128)
    d = got - ref
    wt = np.ones(ref.shape[0]); wt[basis.p[0]:] = 2.0          # reading Q12: the +-k norm
    rel = np.sqrt((wt[:, None] * np.abs(d) ** 2).sum(0) / (wt[:, None] * np.abs(ref) ** 2).sum(0))
    print(f"eps {eps:g} w {plan.w}: rel l2 max {rel.max():.3e} mean {rel.mean():.3e} p99 {np.quantile(rel, 0.99):.3e}", flush=True)
