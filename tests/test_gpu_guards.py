"""Memory-safety and race checks of our own (compute-sanitizer is closed on this GPU pool):

* guard bands: every output of every call lives inside a larger NaN-filled allocation; after the call the guard
  bands must still be NaN bit for bit (no write outside [0, size)) and the output must be finite.  Inputs sit
  between NaN guard images, so a read past either end of the stack would put NaN into some output.
* determinism: each call run twice on the same inputs gives bit-identical outputs (a shared-memory race or a
  missing barrier shows up as run-to-run differences), and a batch split differently gives the same
  coefficients image by image.
Covers the compile-time polar kernels (M = 128, 256), the runtime-radix w = 7 kernel, both fp64 kernels, K4/K5 on
tcgen05, the fp64 k = 0 path and the SIMT fallbacks, K6 (eig, SVD), K7, back-projection, synthesis.
"""
import numpy as np
import pytest
import torch

import paper_1412_0781_b200 as F
import synth

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0") if torch.cuda.is_available() else None
G = 4096        # guard elements on each side


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g
    g.build()


def guarded(shape, dtype):
    """NaN-filled buffer with G guard elements on each side (complex: both parts NaN) and the output view."""
    n = int(np.prod(shape))
    if dtype.is_complex:
        rdt = torch.float32 if dtype == torch.complex64 else torch.float64
        buf = torch.view_as_complex(torch.full((n + 2 * G, 2), float("nan"), dtype=rdt, device=DEV))
    else:
        buf = torch.full((n + 2 * G,), float("nan"), dtype=dtype, device=DEV)
    return buf, buf[G:G + n].view(*shape)


def check(buf, what):
    head, tail = buf[:G], buf[-G:]
    assert torch.isnan(head).all() and torch.isnan(tail).all(), f"{what}: write outside the output"
    body = buf[G:-G]
    assert torch.isfinite(body).all(), f"{what}: non-finite output (read outside the input?)"


CASES = [("C2", 64, 0.5, 32.0, F.F32, 0.0, 40), ("C2e6", 64, 0.5, 32.0, F.F32, 1e-6, 24),
         ("fp64-64", 32, 0.5, 16.0, F.F64, 0.0, 20), ("fp64-72", 33, 0.5, 16.0, F.F64, 0.0, 12),
         ("C3", 128, 0.5, 64.0, F.F32, 0.0, 300), ("C3w5", 128, 0.5, 64.0, F.F32, 1e-4, 300),
         ("C2w5", 64, 0.5, 32.0, F.F32, 1e-4, 40), ("f32-64", 32, 0.5, 16.0, F.F32, 0.0, 20),
         ("f32-64w5", 32, 0.5, 16.0, F.F32, 1e-4, 20)]


@pytest.mark.parametrize("name,L,c,R,dt,eps,n", CASES)
def test_guard_bands_and_determinism(name, L, c, R, dt, eps, n):
    rdt = torch.float32 if dt == F.F32 else torch.float64
    cdt = torch.complex64 if dt == F.F32 else torch.complex128
    if name.startswith("C") and dt == F.F32:
        src = synth.blob_images(synth.config(name[:2]), 0, n, device=DEV)
    else:
        src = torch.from_numpy(np.random.default_rng(L).standard_normal((n, L, L))).to(DEV, rdt)
    ibuf, imgs = guarded((n, L, L), rdt)
    imgs.copy_(src)
    plan = F.fbspca_plan(L, c, R, eps=eps, dtype=dt, device=0, max_batch=max(8, n // 3))
    cbuf, coeffs = guarded((plan.n_coef, n), cdt)
    F.fbspca_expand(plan, imgs, coeffs)
    bbuf, blocks = guarded((plan.n_blk,), torch.float64)
    mbuf, mean = guarded((int(plan.p[0]),), torch.float64)
    F.fbspca_covariance(plan, coeffs, n, n, None, blocks, mean)
    evals, evecs = F.fbspca_eig(plan, blocks)
    obuf, out = guarded((plan.n_coef, n), cdt)
    F.fbspca_project(plan, coeffs, mean, evals, evecs, sigma2=1.0, mode=1, out=out)
    abuf, ahat = guarded((plan.n_coef, n), cdt)
    F.fbspca_backproject(plan, out, mean, evecs, out=ahat)
    sbuf, simg = guarded((min(n, 4), L, L), rdt)
    F.fbspca_synthesize(plan, ahat[:, :min(n, 4)].contiguous(), out=simg)
    torch.cuda.synchronize()
    for b, w in ((cbuf, "expand"), (bbuf, "covariance blocks"), (mbuf, "mean"), (obuf, "project"),
                 (abuf, "backproject"), (sbuf, "synthesize")):
        check(torch.view_as_real(b) if b.is_complex() else b, w)
    assert torch.isfinite(evals).all() and torch.isfinite(evecs).all()
    # determinism: the same calls again, bit for bit
    c2 = F.fbspca_expand(plan, imgs)
    b2, m2 = F.fbspca_covariance(plan, c2)
    e2, v2 = F.fbspca_eig(plan, b2)
    o2 = F.fbspca_project(plan, c2, m2, e2, v2, sigma2=1.0, mode=1)
    torch.cuda.synchronize()
    assert torch.equal(c2, coeffs) and torch.equal(b2, blocks) and torch.equal(m2, mean)
    assert torch.equal(e2, evals) and torch.equal(v2, evecs) and torch.equal(o2, out)
    # another batch split: the same per-image coefficients (each image's arithmetic is independent of its slot)
    plan2 = F.fbspca_plan(L, c, R, eps=eps, dtype=dt, device=0, max_batch=max(5, n // 2 + 1))
    c3 = F.fbspca_expand(plan2, imgs)
    torch.cuda.synchronize()
    scale = coeffs.abs().max()
    assert ((c3 - coeffs).abs().max() / scale).item() <= (1e-6 if dt == F.F32 else 1e-13)


def test_svd_guard_bands():
    cfg = synth.config("C2")
    n = 16
    imgs = synth.blob_images(cfg, 0, n, device=DEV)
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], device=0, max_batch=64)
    coeffs = F.fbspca_expand(plan, imgs)
    ebuf, ev = guarded((plan.n_coef,), torch.float64)
    vbuf, vv = guarded((int(plan.evec_off[-1]),), torch.float64)
    mbuf, mn = guarded((int(plan.p[0]),), torch.float64)
    from paper_1412_0781_b200._lib import check as chk, lib
    import ctypes
    chk(lib().fbspca_svd(ctypes.c_void_p(plan.handle), coeffs.data_ptr(), n, mn.data_ptr(), ev.data_ptr(),
                         vv.data_ptr(), torch.cuda.current_stream().cuda_stream), "svd")
    torch.cuda.synchronize()
    for b, w in ((ebuf, "svd evals"), (vbuf, "svd evecs"), (mbuf, "svd mean")):
        check(b, w)
