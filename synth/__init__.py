"""Seeded synthetic inputs for the five BASELINE.json configs (C1-C5).

This module is the ONLY code shared by the oracle side (tests) and the product
side (bench.py / GPU tests): it produces images and nothing else.  It holds none
of the hot path's arithmetic (no NUFFT, angular FFT, radial quadrature,
covariance, eig or projection).

* ``rng``      counter-based hash RNG keyed by (seed, image index, stream, counter):
               every image is independent of how the stack is sharded.
* ``fbmodel``  C1: random FB coefficients synthesised on the pixel grid through the
               closed form of Eq. (IFT_FB) with reading Q2 (i^{+k} in the
               numerator).  Its Bessel zeros come from ``scipy.special.jn_zeros``
               (a library routine) -- not from the oracle or from the product plan.
* ``blobs``    C2-C5: isotropic Gaussian blobs, low-passed to c, plus white noise.
"""
from .rng import uniform01, normal01  # noqa: F401
from .fbmodel import c1_images, fb_census_scipy, synth_fb_images  # noqa: F401
from .blobs import blob_images, CONFIGS, config  # noqa: F401
