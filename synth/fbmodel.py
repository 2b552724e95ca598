"""C1 input model (BASELINE.json configs[0]): random FB coefficients rendered on the pixel grid.

Image = sum_q a_{0q} F^{-1}psi^{0q} + 2 Re sum_{k>=1,q} a_{kq} F^{-1}psi^{kq} at pixel centres
with r <= R (zero outside), plus white noise.  F^{-1}psi is the closed form of Eq. (IFT_FB)
 with reading Q2: i^{+k} in the numerator, removable singularity
c sqrt(pi) (-1)^{q+1} i^k J_{k+1}(R_{kq}) e^{ik phi}.  Derivation: DESIGN.md "Readings" Q2.

Coefficients: a_{k,q} ~ CN(0, v), v = exp(-R_{k,q}^2/200) (Re, Im each N(0, v/2)); a_{0,q} ~ N(0, v).
Census from scipy.special.jn_zeros (library), independent of oracle/ and of the product plan.
"""
from __future__ import annotations

import math

import numpy as np
import torch
from scipy.special import jn_zeros, jv

from .rng import normal01


def fb_census_scipy(c: float, R: float):
    """(p_k list, zeros list with q = 1..p_k) via scipy jn_zeros and R_{k,q+1} <= 2 pi c R."""
    X = 2 * math.pi * c * R
    p, zeros = [], []
    k = 0
    while True:
        z = jn_zeros(k, int(X / math.pi) + 4)
        pk = int(np.sum(z[1:] <= X))
        if pk == 0:
            break
        p.append(pk)
        zeros.append(z[:pk])
        k += 1
    return p, zeros


def ift_fb(k: int, Rkq: float, q: int, c: float, r: np.ndarray, phi: np.ndarray) -> np.ndarray:
    """F^{-1}(psi_c^{k,q})(r, phi), Eq. (IFT_FB) with i^{+k} in the numerator (reading Q2), k >= 0."""
    x = 2 * math.pi * c * r
    den = x * x - Rkq * Rkq
    near = np.abs(x - Rkq) < 1e-8
    safe = np.where(near, 1.0, den)
    val = 2 * c * math.sqrt(math.pi) * (-1) ** q * Rkq * jv(k, x) / safe
    lim = c * math.sqrt(math.pi) * (-1) ** (q + 1) * jv(k + 1, Rkq)
    val = np.where(near, lim, val)
    return val * (1j ** k) * np.exp(1j * k * phi)


def synth_fb_images(coeffs: list, zeros: list, c: float, R: float, L: int,
                    mask: bool = True) -> np.ndarray:
    """coeffs[k]: (p_k, n) complex (k=0 real).  Returns (n, L, L) float64 (zero at r > R if mask)."""
    idx = np.arange(L) - L // 2
    i1, i2 = np.meshgrid(idx, idx, indexing="ij")             # axis 0 = i1 (x), axis 1 = i2 (y)
    r = np.hypot(i1, i2).ravel()
    phi = np.arctan2(i2, i1).ravel()
    inside = (r <= R) if mask else np.ones_like(r, dtype=bool)
    n = coeffs[0].shape[1]
    img = np.zeros((n, L * L))
    for k, Ak in enumerate(coeffs):
        for q in range(Ak.shape[0]):
            basis = ift_fb(k, zeros[k][q], q + 1, c, r, phi) * inside
            if k == 0:
                img += np.outer(Ak[q].real, basis.real)
            else:
                img += 2.0 * np.real(np.outer(Ak[q], basis))
    return img.reshape(n, L, L)


def c1_coefficients(n: int, c: float = 0.5, R: float = 16.0, seed: int = 0, first: int = 0):
    """Seeded C1 coefficients for images first..first+n-1 (counter-keyed per image)."""
    p, zeros = fb_census_scipy(c, R)
    img = torch.arange(first, first + n, dtype=torch.int64)[:, None]
    coeffs, t = [], 0
    for k, pk in enumerate(p):
        v = np.exp(-zeros[k] ** 2 / 200.0)                    # (p_k,)
        cnt = torch.arange(t, t + pk, dtype=torch.int64)[None, :]
        z1 = normal01(seed, img, 1, 2 * cnt).numpy().T           # (p_k, n)
        z2 = normal01(seed, img, 1, 2 * cnt + 1).numpy().T
        if k == 0:
            a = np.sqrt(v)[:, None] * z1 + 0j
        else:
            a = np.sqrt(v / 2)[:, None] * (z1 + 1j * z2)
        coeffs.append(a)
        t += pk
    return coeffs, p, zeros


def c1_images(n: int = 256, L: int = 32, R: float = 16.0, c: float = 0.5, sigma: float = 0.5,
              seed: int = 0, first: int = 0, return_coeffs: bool = False, mask: bool = True):
    """BASELINE configs[0]: fp64 (n, L, L) images (+ the planted coefficients if asked)."""
    coeffs, p, zeros = c1_coefficients(n, c, R, seed, first)
    clean = synth_fb_images(coeffs, zeros, c, R, L, mask)
    img = torch.arange(first, first + n, dtype=torch.int64)[:, None]
    pix = torch.arange(L * L, dtype=torch.int64)[None, :]
    noise = normal01(seed, img, 2, pix).numpy().reshape(n, L, L)
    out = clean + sigma * noise
    return (out, coeffs) if return_coeffs else out
