"""C2-C5 input model (BASELINE.json configs[1..4]): Gaussian blobs, low-passed to c, plus noise.

Per image i (all draws counter-keyed by (seed, i), so shard-invariant):
  centres   r = 0.7 R sqrt(u), phi = 2 pi v  (uniform by area in the disk of radius 0.7R)
  widths    sigma_b ~ U[lo, hi] px;  amplitudes A_b ~ U[0.5, 1]
  rotation  (C3 only) phi += alpha, alpha ~ U[0, 2 pi)  -- an exact in-plane rotation
  clean     sum_b A_b exp(-|x - mu_b|^2 / (2 sigma_b^2)), x = (i1, i2), i = a - floor(L/2)
  lowpass   L x L DFT, zero |xi| > c, inverse, real part
  noise     sigma_n^2 = var(clean over images 0..min(n,1024)-1) / SNR   (reading Q15)
Images are produced in chunks aligned to absolute multiples of CHUNK so that the bits of
image i never depend on which range was requested (batched FFT plans can vary with batch).
"""
from __future__ import annotations

import math

import torch

from .rng import normal01, uniform01

CHUNK = 512

CONFIGS = {
    # name: n, L, R, c, dtype, blobs, sigma range (px), SNR, rotate
    "C1": dict(n=256, L=32, R=16.0, c=0.5, dtype="f64", model="fb", sigma=0.5),
    "C2": dict(n=10_000, L=64, R=32.0, c=0.5, dtype="f32", model="blobs", nblobs=20,
               sig=(1.0, 4.0), snr=1 / 10, rotate=False),
    "C3": dict(n=100_000, L=128, R=64.0, c=0.5, dtype="f32", model="blobs", nblobs=40,
               sig=(2.0, 8.0), snr=1 / 20, rotate=True),
    "C4": dict(n=500_000, L=256, R=128.0, c=0.5, dtype="f32", model="blobs", nblobs=60,
               sig=(3.0, 12.0), snr=1 / 30, rotate=False),
    "C5": dict(n=50_000, L=360, R=180.0, c=0.5, dtype="f32", model="blobs", nblobs=80,
               sig=(4.0, 16.0), snr=1 / 20, rotate=False),
    # the paper's own timing workload (Table III): 10^5 images of N(0,1) noise, 300 x 300, R = 150, c = 1/2
    "T3": dict(n=100_000, L=300, R=150.0, c=0.5, dtype="f32", model="noise"),
    # the paper's ribosome experiment shape: 10^5 images of 240 x 240, R = 98, c = 0.196,
    # SNR 1/30 -- n_theta = ceil(16 c R) = 308 = 4 7 11 (radix-7/11 angular FFTs); synthetic blobs stand in for
    # the EMDB-2762 projections (dataset absent)
    "RB": dict(n=100_000, L=240, R=98.0, c=0.196, dtype="f32", model="blobs", nblobs=50,
               sig=(3.0, 12.0), snr=1 / 30, rotate=False),
}


def config(name: str) -> dict:
    d = dict(CONFIGS[name])
    d["name"] = name
    return d


def _clean_chunk(cfg: dict, first: int, count: int, device, seed: int) -> torch.Tensor:
    if cfg["model"] == "noise":
        return torch.zeros((count, cfg["L"], cfg["L"]), dtype=torch.float64, device=device)
    L, R, c, nb = cfg["L"], cfg["R"], cfg["c"], cfg["nblobs"]
    lo, hi = cfg["sig"]
    img = torch.arange(first, first + count, dtype=torch.int64, device=device)[:, None]
    b = torch.arange(nb, dtype=torch.int64, device=device)[None, :]
    u = lambda s: uniform01(seed, img, s, b)                           # (count, nb) float64
    r = 0.7 * R * torch.sqrt(u(10))
    phi = 2 * math.pi * u(11)
    if cfg.get("rotate"):
        alpha = 2 * math.pi * uniform01(seed, img, 12, torch.zeros_like(img))
        phi = phi + alpha
    sig = lo + (hi - lo) * u(13)
    amp = 0.5 + 0.5 * u(14)
    mu1, mu2 = r * torch.cos(phi), r * torch.sin(phi)
    x = (torch.arange(L, device=device, dtype=torch.float64) - L // 2)[None, None, :]
    g1 = torch.exp(-(x - mu1[..., None]) ** 2 / (2 * sig[..., None] ** 2))   # (count, nb, L) over i1
    g2 = torch.exp(-(x - mu2[..., None]) ** 2 / (2 * sig[..., None] ** 2))   # over i2
    clean = torch.einsum("nba,nbc->nac", amp[..., None] * g1, g2)            # (count, L, L)
    f = torch.fft.fftfreq(L, device=device, dtype=torch.float64)
    mask = (f[:, None] ** 2 + f[None, :] ** 2) <= c * c
    clean = torch.fft.ifft2(torch.fft.fft2(clean) * mask).real
    return clean


def noise_sigma(cfg: dict, device="cpu", seed: int = 0) -> float:
    """sigma_n = sqrt(var(clean images 0..min(n,1024)-1) / SNR)  (reading Q15); 1 for pure-noise configs."""
    if cfg["model"] == "noise":
        return 1.0
    m = min(cfg["n"], 1024)
    parts = [_clean_chunk(cfg, s, min(CHUNK, m - s), device, seed) for s in range(0, m, CHUNK)]
    v = torch.cat(parts).var().item()
    return math.sqrt(v / cfg["snr"])


def blob_images(cfg: dict, first: int, count: int, device="cpu", seed: int = 0,
                sigma_n: float | None = None, out: torch.Tensor | None = None,
                dtype=torch.float32) -> torch.Tensor:
    """Images first..first+count-1 of config cfg as a (count, L, L) tensor on device."""
    L = cfg["L"]
    if sigma_n is None:
        sigma_n = noise_sigma(cfg, device, seed)
    if out is None:
        out = torch.empty((count, L, L), dtype=dtype, device=device)
    end = first + count
    s = (first // CHUNK) * CHUNK
    while s < end:
        clean = _clean_chunk(cfg, s, CHUNK, device, seed)
        img = torch.arange(s, s + CHUNK, dtype=torch.int64, device=device)[:, None]
        pix = torch.arange(L * L, dtype=torch.int64, device=device)[None, :]
        noisy = clean + sigma_n * normal01(seed, img, 3, pix).view(CHUNK, L, L)
        a, b = max(s, first), min(s + CHUNK, end)
        out[a - first:b - first] = noisy[a - s:b - s].to(dtype)
        s += CHUNK
    return out
