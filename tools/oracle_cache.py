"""Write cached fp64 ORACLE results for a whole BASELINE.json config (test fixtures under tests/golden/).

    python tools/oracle_cache.py C2        # n = 10,000, L = 64   (seconds)
    python tools/oracle_cache.py C3        # n = 100,000, L = 128 (about half an hour on 8 cores)

Calls only `synth` (the seeded input generator, on the CPU) and `oracle/` (Alg. 1 with the exact Fourier sum,
Alg. 2 lines 1-4): O.expand -> O.covariance_partials (summed over image chunks) -> O.finalize_covariance ->
O.block_eig.  Nothing here touches the CUDA library.  The file records the SHA-256 of the fp32 image stack it
consumed so a test can tell which inputs the numbers belong to.

Stored (npz): p (p_k), n, mean (p_0), lam (concatenated per k, descending), U (concatenated row-major p_k x p_k
blocks, columns = eigenvectors, sign reading Q10), C (concatenated row-major p_k x p_k blocks), sha256, config.
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import synth  # noqa: E402

CHUNK = 2048


def main(name: str, n: int | None = None, out: str | None = None) -> str:
    cfg = synth.config(name)
    n = n or cfg["n"]
    basis = O.build_basis(cfg["c"], cfg["R"])
    sig = synth.blobs.noise_sigma(cfg)
    h = hashlib.sha256()
    S = s0 = None
    t0 = time.time()
    for a in range(0, n, CHUNK):
        b = min(n, a + CHUNK)
        imgs = synth.blob_images(cfg, a, b - a, sigma_n=sig).numpy()          # fp32, CPU
        h.update(np.ascontiguousarray(imgs).tobytes())
        A = O.expand(imgs.astype(np.float64), basis)
        Sc, s0c, _ = O.covariance_partials(A)
        S = Sc if S is None else [x + y for x, y in zip(S, Sc)]
        s0 = s0c if s0 is None else s0 + s0c
        print(f"{name}: {b}/{n} images, {time.time() - t0:.0f} s", flush=True)
    mean, C = O.finalize_covariance(S, s0, n)
    lam, U = O.block_eig(C)
    out = out or os.path.join(ROOT, "tests", "golden", f"oracle_{name}.npz")
    np.savez_compressed(out, p=np.asarray(basis.p), n=n, mean=mean, lam=np.concatenate(lam),
                        U=np.concatenate([u.ravel() for u in U]), C=np.concatenate([c.ravel() for c in C]),
                        sha256=h.hexdigest(), config=name, sigma_n=sig)
    print(f"wrote {out} ({time.time() - t0:.0f} s), sha256 {h.hexdigest()}")
    return out


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
