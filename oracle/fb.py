"""fp64 oracle: Algorithm 1 (Fast FB expansion) and Algorithm 2 (steerable PCA).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  P:n = PAPER.md line n.

Data conventions (shared *by definition* with the product, not by code):
  images : (n, L, L) float, axis 0 = i1, axis 1 = i2, i = a - floor(L/2)   (Q3)
  A      : list over k = 0..k_max of complex arrays (p_k, n); rows q, columns images
           (the paper's A^(k))
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from numpy.polynomial.legendre import leggauss
from scipy.optimize import brentq
from scipy.special import jv

__all__ = [
    "Basis", "bessel_zeros_upto", "build_basis", "gauss_legendre", "polar_grid",
    "radial_table", "polar_ft_direct", "angular_transform", "radial_quadrature",
    "expand", "expand_polar", "synthesize_polar", "mean_and_center",
    "block_covariance", "covariance_partials", "finalize_covariance",
    "block_eig", "svd_route", "sign_normalize", "radial_eigenfunctions", "spca_coeffs", "mp_edge", "mp_select",
    "shrink_weights", "project", "backproject", "synthesize_pixels", "rotate_coeffs", "reflect_coeffs",
    "flat_index", "to_flat", "from_flat",
    "radial_profile", "estimate_noise_variance", "estimate_support", "estimate_bandlimit",
]


# --------------------------------------------------------------------------
# O1 census: Bessel roots and the Klug-Crowther truncation
# --------------------------------------------------------------------------
def bessel_zeros_upto(k: int, xmax: float, step: float = 0.25) -> np.ndarray:
    """All positive zeros R_{k,q} of J_k with R_{k,q} <= xmax, plus the first one above.

    P:87 "R_{k,q} is the q-th root of the Bessel function J_k".  Bracketing by a
    sign scan of step 0.25 (< pi, the lower bound on the spacing of consecutive
    zeros, so each bracket holds one root; J_k has no zeros below x = k), then
    brentq, then Newton polish with J_k' = (J_{k-1} - J_{k+1})/2.
    """
    x0 = max(float(k), 0.05)
    hi = xmax + 2 * math.pi
    roots = []
    while not roots or roots[-1] <= xmax:
        xs = np.arange(x0, hi + step, step)
        v = jv(k, xs)
        for i in np.nonzero(np.sign(v[:-1]) * np.sign(v[1:]) < 0)[0]:
            r = brentq(lambda x: jv(k, x), xs[i], xs[i + 1], xtol=1e-14, rtol=1e-15, maxiter=200)
            for _ in range(3):  # Newton polish
                d = 0.5 * (jv(k - 1, r) - jv(k + 1, r))
                r = r - jv(k, r) / d
            roots.append(r)
            if r > xmax:
                break
        x0, hi = xs[-1], hi + 4 * math.pi       # no root above xmax yet: scan further
    return np.asarray(roots)


@dataclass
class Basis:
    """Truncated FB basis for band limit c and support radius R."""
    c: float
    R: float
    k_max: int
    p: list                      # p_k, k = 0..k_max
    zeros: list                  # zeros[k] = array of R_{k,q}, q = 1..p_k+1
    norm: list                   # norm[k][q-1] = N_{k,q}
    n_xi: int = 0
    n_theta: int = 0

    @property
    def coef_off(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(self.p)]).astype(np.int64)

    @property
    def n_coef(self) -> int:
        return int(sum(self.p))


def _ceil_int(x: float) -> int:
    # DESIGN.md reading Q4: ceil with a 1e-9 guard against representation noise.
    return int(math.ceil(x - 1e-9))


def build_basis(c: float, R: float) -> Basis:
    """Census under Eq. (criterion1) R_{k,q+1} <= 2 pi c R.

    p_k = #{q >= 1 : R_{k,q+1} <= 2 pi c R}; k runs 0,1,... until the first p_k = 0
    ("k_max is the maximal possible value of k satisfying Eq. (criterion1)").
    Also fixes n_xi = ceil(4cR), n_theta = ceil(16cR) (Alg. 1 step 1).
    """
    X = 2.0 * math.pi * c * R
    p, zeros, norm = [], [], []
    k = 0
    while True:
        z = bessel_zeros_upto(k, X)
        pk = int(np.sum(z[1:] <= X)) if len(z) > 1 else 0
        if pk == 0:
            break
        p.append(pk)
        zeros.append(z[: pk + 1].copy())
        # N_{k,q} = (c sqrt(pi) |J_{k+1}(R_{k,q})|)^{-1}
        norm.append(1.0 / (c * math.sqrt(math.pi) * np.abs(jv(k + 1, z[:pk]))))
        k += 1
    return Basis(c=c, R=R, k_max=len(p) - 1, p=p, zeros=zeros, norm=norm,
                 n_xi=_ceil_int(4 * c * R), n_theta=_ceil_int(16 * c * R))


# --------------------------------------------------------------------------
# O2-O4 quadrature grid and radial table
# --------------------------------------------------------------------------
def gauss_legendre(m: int, a: float, b: float):
    """m-point Gauss-Legendre rule on [a, b], from numpy.leggauss."""
    x, w = leggauss(m)
    return a + (b - a) * (x + 1) / 2, w * (b - a) / 2


def polar_grid(basis: Basis):
    """xi_j (GL on [0,c], n_xi points), w_j, theta_l = 2 pi l / n_theta."""
    xi, w = gauss_legendre(basis.n_xi, 0.0, basis.c)
    theta = 2 * np.pi * np.arange(basis.n_theta) / basis.n_theta
    return xi, w, theta


def radial_table(basis: Basis, xi=None, w=None):
    """B_k[q][j] = N_{k,q} J_k(R_{k,q} xi_j / c) xi_j w(xi_j)  (Eq. (a))."""
    if xi is None:
        xi, w, _ = polar_grid(basis)
    out = []
    for k in range(basis.k_max + 1):
        Rk = basis.zeros[k][: basis.p[k]]
        Nk = basis.norm[k]
        out.append(Nk[:, None] * jv(k, np.outer(Rk, xi) / basis.c) * (xi * w)[None, :])
    return out


# --------------------------------------------------------------------------
# O5 direct Fourier sum at the polar nodes (Eq. (nufft); Q1 unit prefactor)
# --------------------------------------------------------------------------
def polar_ft_direct(images: np.ndarray, basis: Basis, chunk: int | None = None,
                    node_chunk: int = 1024, dense: bool | None = None) -> np.ndarray:
    """F(I)(xi_1, xi_2) = sum_{i1,i2} I(i1,i2) exp(-2 pi i (xi_1 i1 + xi_2 i2))   (Eq. (nufft), Q1 unit prefactor).

    Evaluated exactly (up to rounding) at every node (xi_j cos theta_l, xi_j sin theta_l), with
    E1[node, i1] = e^{-2 pi i xi_1 i1} and E2[node, i2] = e^{-2 pi i xi_2 i2}, in one of two orders of the same
    double sum (fp64 BLAS through torch, per block of node_chunk nodes):
      dense     (default for n >= 32): F = I_flat K^T with the dense kernel K[node, i1 L + i2] = E1 E2;
      separable (small n):            T[i1, node] = sum_{i2} I[i1, i2] E2[node, i2], F = sum_{i1} E1[node, i1] T.
    Nodes l < n_theta/2 are summed directly; for even n_theta the node l + n_theta/2 is the negated node l,
    where the sum for a real image is the complex conjugate (exact identity of the definition for real I,
    P:197).  `chunk` is accepted for compatibility and ignored.  Returns (n, n_xi, n_theta) complex128.
    """
    import torch
    images = np.asarray(images, dtype=np.float64)
    n, L, L2 = images.shape
    assert L == L2
    if dense is None:
        dense = n >= 32
    xi, _, theta = polar_grid(basis)
    nt = basis.n_theta
    half = nt // 2 if nt % 2 == 0 else nt
    idx = torch.arange(L, dtype=torch.float64) - L // 2                       # i = a - floor(L/2)
    k1 = torch.from_numpy(np.outer(xi, np.cos(theta[:half])).ravel())         # xi_1 at nodes
    k2 = torch.from_numpy(np.outer(xi, np.sin(theta[:half])).ravel())         # xi_2 at nodes
    I3 = torch.from_numpy(images)
    Fh = torch.empty((n, k1.numel()), dtype=torch.complex128)
    for s in range(0, k1.numel(), node_chunk):
        E1 = torch.exp(-2j * math.pi * torch.outer(k1[s:s + node_chunk], idx))   # (nodes, L): e^{-2pi i xi1 i1}
        E2 = torch.exp(-2j * math.pi * torch.outer(k2[s:s + node_chunk], idx))   # (nodes, L): e^{-2pi i xi2 i2}
        if dense:
            # K[node, i1 L + i2] = E1[node, i1] E2[node, i2], real and imaginary parts written out:
            #   Re K = Re E1 Re E2 - Im E1 Im E2,   Im K = Re E1 Im E2 + Im E1 Re E2   (batched outer products)
            e1r, e1i, e2r, e2i = E1.real, E1.imag, E2.real, E2.imag
            Kr = torch.bmm(torch.stack([e1r, -e1i], -1), torch.stack([e2r, e2i], 1)).reshape(-1, L * L)
            Ki = torch.bmm(torch.stack([e1r, e1i], -1), torch.stack([e2i, e2r], 1)).reshape(-1, L * L)
            If = I3.reshape(n, L * L)
            Fh[:, s:s + node_chunk] = torch.complex(If @ Kr.T, If @ Ki.T)
        else:
            for b in range(n):
                T = torch.complex(I3[b] @ E2.real.T.contiguous(), I3[b] @ E2.imag.T.contiguous())  # (i1, node)
                Fh[b, s:s + node_chunk] = (E1.T * T).sum(0)
    Fh = Fh.numpy().reshape(n, basis.n_xi, half)
    out = np.empty((n, basis.n_xi, nt), dtype=np.complex128)
    out[:, :, :half] = Fh
    if half != nt:
        out[:, :, half:] = np.conj(Fh)
    return out


# --------------------------------------------------------------------------
# O6-O7 angular FFT and radial quadrature (Eqs. (1DFFT) P:189 and (a) P:195)
# --------------------------------------------------------------------------
def angular_transform(F: np.ndarray, k_max: int) -> np.ndarray:
    """g^(xi_j, k) = (2 pi / n_theta) sum_l F(xi_j, theta_l) e^{-2 pi i k l / n_theta}, k=0..k_max."""
    nt = F.shape[-1]
    return (2 * np.pi / nt) * np.fft.fft(F, axis=-1)[..., : k_max + 1]


def radial_quadrature(ghat: np.ndarray, basis: Basis, table=None) -> list:
    """a_{k,q} = sum_j N_{k,q} J_k(R_{k,q} xi_j/c) g^(xi_j,k) xi_j w_j  (Eq. (a)).

    ghat: (n, n_xi, k_max+1).  Returns list A[k] of (p_k, n) complex.  Im a_{0,q} := 0 (Q8).
    """
    if table is None:
        table = radial_table(basis)
    A = []
    for k in range(basis.k_max + 1):
        Ak = table[k] @ ghat[:, :, k].T                           # (p_k, n)
        if k == 0:
            Ak = Ak.real.astype(np.complex128)
        A.append(Ak)
    return A


def expand_polar(F: np.ndarray, basis: Basis, table=None) -> list:
    """Steps (1DFFT) + (a) of Alg. 1 line 4 on given polar samples F (n, n_xi, n_theta)."""
    return radial_quadrature(angular_transform(F, basis.k_max), basis, table)


def expand(images: np.ndarray, basis: Basis, chunk: int | None = None) -> list:
    """Algorithm 1 with the exact Fourier sum in place of the NUFFT.

    Images go through polar_ft_direct in chunks of `chunk` (default: as many as keep the polar samples of a
    chunk near 4 GB; the dense kernel is rebuilt once per chunk, so larger chunks are faster)."""
    table = radial_table(basis)
    if chunk is None:
        chunk = max(1, int(4e9 // (16 * basis.n_xi * basis.n_theta)))
    parts = []
    for s in range(0, len(images), chunk):
        F = polar_ft_direct(images[s:s + chunk], basis)
        parts.append(expand_polar(F, basis, table))
    return [np.concatenate([p[k] for p in parts], axis=1) for k in range(basis.k_max + 1)]


def synthesize_polar(A: list, basis: Basis) -> np.ndarray:
    """P_{c,R} F(f) on the polar grid (Eq. (contapprox)), negative k by a_{-k}=conj(a_k).

    F(xi_j, theta_l) = sum_k sum_q a_{k,q} N_{k,q} J_k(R_{k,q} xi_j/c) e^{i k theta_l}.
    A[k] is (p_k, n) for k = 0..k_max; returns (n, n_xi, n_theta).
    Used only by oracle pins (exact-recovery test).
    """
    xi, _, theta = polar_grid(basis)
    n = A[0].shape[1]
    F = np.zeros((n, basis.n_xi, basis.n_theta), dtype=np.complex128)
    for k in range(basis.k_max + 1):
        Rk = basis.zeros[k][: basis.p[k]]
        rad = basis.norm[k][:, None] * jv(k, np.outer(Rk, xi) / basis.c)   # (p_k, n_xi)
        s = A[k].T @ rad                                                    # (n, n_xi)
        F += s[:, :, None] * np.exp(1j * k * theta)[None, None, :]
        if k > 0:
            s_neg = np.conj(A[k]).T @ (rad * (-1) ** k)     # psi^{-k,q} = (-1)^k J_k e^{-ik theta}
            F += s_neg[:, :, None] * np.exp(-1j * k * theta)[None, None, :]
    return F


# --------------------------------------------------------------------------
# O8 mean / covariance (Alg. 2 lines 1-4)
# --------------------------------------------------------------------------
def mean_and_center(A: list):
    """a^mean_{0,q} = (1/n) sum_j a^j_{0,q}; a^i_{0,q} <- a^i_{0,q} - mean (Alg. 2 line 1)."""
    mean = A[0].real.mean(axis=1)
    Ac = [A[0] - mean[:, None]] + list(A[1:])
    return mean, Ac


def block_covariance(A: list):
    """C^(k) = (1/n) Re{A^(k) A^(k)*} (Eq. (ck)); C^(0) = (1/n) A0 A0^* after centring."""
    n = A[0].shape[1]
    mean, Ac = mean_and_center(A)
    C = [np.real(Ak @ np.conj(Ak).T) / n for Ak in Ac]
    return mean, C


def covariance_partials(A: list):
    """Shard-local sums for the data-parallel form of (ck)/(ck_0):
    S_k = sum_i Re(a_i a_i^*), s0 = sum_i a_{0,i}, n.  ("each worker is allocated a subset")."""
    S = [np.real(Ak @ np.conj(Ak).T) for Ak in A]
    return S, A[0].real.sum(axis=1), A[0].shape[1]


def finalize_covariance(S: list, s0: np.ndarray, n: int):
    """C^(0) = S_0/n - s0 s0^T/n^2 (= (1/n) sum (a0-m)(a0-m)^T); C^(k) = S_k/n."""
    mean = s0 / n
    C = [S[0] / n - np.outer(mean, mean)] + [Sk / n for Sk in S[1:]]
    return mean, C


# --------------------------------------------------------------------------
# O9 eigendecomposition (Alg. 2 line 4)
# --------------------------------------------------------------------------
def sign_normalize(U: np.ndarray) -> np.ndarray:
    """Reading Q10: make the entry of largest |u(q)| positive (ties -> lowest q)."""
    U = U.copy()
    for l in range(U.shape[1]):
        q = int(np.argmax(np.abs(U[:, l])))      # argmax returns the lowest index on ties
        if U[q, l] < 0:
            U[:, l] = -U[:, l]
    return U


def block_eig(C: list):
    """lambda^(k)_1 >= ... >= lambda^(k)_{p_k}, u^(k)_l (numpy.linalg.eigh, sorted descending)."""
    lam, U = [], []
    for Ck in C:
        w, V = np.linalg.eigh(0.5 * (Ck + Ck.T))
        o = np.argsort(-w, kind="stable")
        lam.append(w[o])
        U.append(sign_normalize(V[:, o]))
    return lam, U


def svd_route(A: list):
    """Alg. 2 line 4, SVD form ("or perform SVD of A^(k) and take the left singular
    vectors", the route for n < p_k).  B_k = [Re A_k, Im A_k] / sqrt(n) (k = 0: A_0 minus the mean, real)
    has B_k B_k^T = C^(k) of Eqs. (ck)/(ck_0), so lambda = s^2 and U = left singular vectors
    (numpy.linalg.svd, full_matrices: a complete basis when rank < p_k; zero singular values appended).
    Returns (mean, lam, U) like covariance + block_eig."""
    n = A[0].shape[1]
    mean = A[0].real.mean(axis=1)
    lam, U = [], []
    for k, Ak in enumerate(A):
        if k == 0:
            B = (Ak.real - mean[:, None]) / math.sqrt(n)
        else:
            B = np.concatenate([Ak.real, Ak.imag], axis=1) / math.sqrt(n)
        Uk, sv, _ = np.linalg.svd(B, full_matrices=True)
        lk = np.zeros(B.shape[0])
        lk[: sv.size] = sv ** 2
        o = np.argsort(-lk, kind="stable")
        lam.append(lk[o])
        U.append(sign_normalize(Uk[:, o]))
    return mean, lam, U


def radial_eigenfunctions(basis: Basis, U: list, xi=None) -> list:
    """Alg. 2 line 5, Eq. (sPCArad) P:360-361:
    f^{k,l}(xi_j) = sum_q N_{k,q} J_k(R_{k,q} xi_j / c) u_l^(k)(q), at the GL nodes xi_j (default);
    returns (p_k, n_xi) per k, row l."""
    if xi is None:
        xi, _, _ = polar_grid(basis)
    out = []
    for k in range(basis.k_max + 1):
        Rk = basis.zeros[k][: basis.p[k]]
        Bk = basis.norm[k][:, None] * jv(k, np.outer(Rk, xi) / basis.c)      # [q][j]
        out.append(U[k].T @ Bk)
    return out


# --------------------------------------------------------------------------
# O10-O11 projection and MP filtering (Eq. (sPCAcoeff); Eq. (compselect))
# --------------------------------------------------------------------------
def spca_coeffs(Ac: list, U: list) -> list:
    """c^i_{k,l} = sum_q a^i_{k,q} u_l^(k)(q): returns (p_k, n) per k."""
    return [Uk.T @ Ak for Uk, Ak in zip(U, Ac)]


def mp_edge(sigma2: float, p_k: int, n: int, k: int) -> float:
    """lambda_+^(k) = sigma^2 (1 + sqrt(gamma_k))^2, gamma_0 = p_0/n, gamma_k = p_k/(2n)."""
    gamma = p_k / n if k == 0 else p_k / (2.0 * n)
    return sigma2 * (1.0 + math.sqrt(gamma)) ** 2


def mp_select(lam: list, basis: Basis, n: int, sigma2: float) -> list:
    """Eq. (compselect): keep lambda^(k)_l > sigma^2 (1 + sqrt(gamma_k))^2."""
    return [lk > mp_edge(sigma2, basis.p[k], n, k) for k, lk in enumerate(lam)]


def shrink_weights(lam: list, basis: Basis, n: int, sigma2: float, mode: int) -> list:
    """Filter weights per (k,l).

    mode 0: h = 1 (projection only).
    mode 1: MP-select (Eq. compselect) then h = l/(l+sigma^2), l = (lambda - sigma^2)_+  (Q13).
    mode 2: MP-select then spiked-model l = ((lambda - s(1+g)) + sqrt((lambda - s(1+g))^2 - 4 g s^2))/2,
            h = l/(l+s)   (SPEC S:442 optional mode; the paper defers to [Wu13]).
    """
    out = []
    for k, lk in enumerate(lam):
        if mode == 0:
            out.append(np.ones_like(lk))
            continue
        sel = lk > mp_edge(sigma2, basis.p[k], n, k)
        if mode == 1:
            ell = np.maximum(lk - sigma2, 0.0)
        else:
            g = basis.p[k] / n if k == 0 else basis.p[k] / (2.0 * n)
            t = lk - sigma2 * (1 + g)
            ell = 0.5 * (t + np.sqrt(np.maximum(t * t - 4 * g * sigma2 * sigma2, 0.0)))
        h = np.where(sel, ell / (ell + sigma2) if sigma2 > 0 else 1.0, 0.0)
        out.append(h)
    return out


def project(A: list, mean: np.ndarray, U: list, lam: list, basis: Basis,
            sigma2: float, mode: int, n_total: int) -> list:
    """Alg. 2 line 6 with optional filtering: out_k = diag(h_k) U_k^T a_k (k=0 centred)."""
    Ac = [A[0] - mean[:, None]] + list(A[1:])
    c = spca_coeffs(Ac, U)
    h = shrink_weights(lam, basis, n_total, sigma2, mode)
    return [hk[:, None] * ck for hk, ck in zip(h, c)]


def backproject(c: list, mean: np.ndarray, U: list) -> list:
    """Steerable-basis coefficients back to FB coefficients: a_k = U_k c_k (U_k orthogonal, so this inverts
    Eq. (sPCAcoeff)), plus the mean at k = 0 (Alg. 2 line 1 undone).  With c = filtered coefficients
    (project(mode 1/2)) this gives the FB coefficients of the denoised images."""
    out = [Uk @ ck for Uk, ck in zip(U, c)]
    out[0] = out[0] + mean[:, None]
    return out


def synthesize_pixels(A: list, basis: Basis, L: int, mask: bool = True) -> np.ndarray:
    """Images from FB coefficients on the L x L pixel grid (NEXT-1: eigenimages, denoised images):
    I(x) = sum_q a_{0,q} F^-1 psi^{0,q}(x) + 2 Re sum_{k>=1,q} a_{k,q} F^-1 psi^{k,q}(x)   (a_{-k} = conj a_k)
    with Eq. (IFT_FB) read with i^{+k} in the numerator (Q2):
      F^-1 psi^{k,q}(r, phi) = 2 c sqrt(pi) (-1)^q R_{k,q} i^k J_k(2 pi c r) e^{ik phi} / ((2 pi c r)^2 - R_{k,q}^2),
    (q = 1..p_k), removable singularity c sqrt(pi) (-1)^{q+1} i^k J_{k+1}(R_{k,q}) e^{ik phi}; pixels with r > R
    are zero when mask (the compact support of P:115).  Axis 0 = i1 = x (Q3).  Returns (n, L, L) float64."""
    idx = np.arange(L) - L // 2
    i1, i2 = np.meshgrid(idx, idx, indexing="ij")
    r = np.hypot(i1, i2).ravel()
    phi = np.arctan2(i2, i1).ravel()
    keep = (r <= basis.R) if mask else np.ones(r.shape, dtype=bool)
    x = 2 * np.pi * basis.c * r
    n = A[0].shape[1]
    img = np.zeros((n, L * L))
    for k in range(basis.k_max + 1):
        ang = (1j ** k) * np.exp(1j * k * phi)
        jk = jv(k, x)                                   # J_k(2 pi c r): the same for every q
        for q in range(basis.p[k]):
            Rq = basis.zeros[k][q]
            den = x * x - Rq * Rq
            near = np.abs(x - Rq) < 1e-8
            val = 2 * basis.c * np.sqrt(np.pi) * (-1) ** (q + 1) * Rq * jk / np.where(near, 1.0, den)
            val = np.where(near, basis.c * np.sqrt(np.pi) * (-1) ** (q + 2) * jv(k + 1, Rq), val)
            psi = val * ang * keep
            if k == 0:
                img += np.outer(A[0][q].real, psi.real)
            else:
                img += 2.0 * np.real(np.outer(A[k][q], psi))
    return img.reshape(n, L, L)


# --------------------------------------------------------------------------
# O(2) action on coefficients (Eqs. (rot), (refl) P:292)
# --------------------------------------------------------------------------
def rotate_coeffs(A: list, alpha: float) -> list:
    """a_{k,q} -> a_{k,q} e^{-i k alpha}."""
    return [Ak * np.exp(-1j * k * alpha) for k, Ak in enumerate(A)]


def reflect_coeffs(A: list, alpha: float = 0.0) -> list:
    """a_{k,q} -> a_{-k,q} e^{-i k alpha} = conj(a_{k,q}) e^{-i k alpha} for real images."""
    return [np.conj(Ak) * np.exp(-1j * k * alpha) for k, Ak in enumerate(A)]


# --------------------------------------------------------------------------
# layout helpers (k-major flat layout used by the C-ABI: block k at coef_off[k], rows q, cols images)
# --------------------------------------------------------------------------
def flat_index(basis: Basis):
    off = basis.coef_off
    return off


def to_flat(A: list) -> np.ndarray:
    """(sum_k p_k, n) complex array, block k = rows coef_off[k]..coef_off[k+1]."""
    return np.concatenate(A, axis=0)


def from_flat(flat: np.ndarray, basis: Basis) -> list:
    off = basis.coef_off
    return [flat[off[k]:off[k + 1]] for k in range(basis.k_max + 1)]


# --------------------------------------------------------------------------
# NEXT-2: parameter estimation (Fig. 5; SPEC estimate_noise_variance / _support / _bandlimit)
# --------------------------------------------------------------------------
def radial_profile(m: np.ndarray, offsets: np.ndarray, nbins: int, weights=None) -> np.ndarray:
    """Mean of a 2-D map over bins b = floor(r + 1/2), r = |(o1, o2)| of the given per-axis offsets (reading Q18)."""
    o1, o2 = np.meshgrid(offsets, offsets, indexing="ij")
    b = np.floor(np.hypot(o1, o2) + 0.5).astype(int)
    w = np.ones_like(m) if weights is None else weights
    out = np.zeros(nbins)
    for k in range(nbins):
        sel = b == k
        out[k] = (m[sel] * w[sel]).sum() / w[sel].sum() if sel.any() else 0.0
    return out


def _variance_profile(stack: np.ndarray) -> np.ndarray:
    L = stack.shape[1]
    var = ((stack - stack.mean(axis=0)) ** 2).mean(axis=0)           # divisor n (Q9's convention)
    return radial_profile(var, np.arange(L) - L // 2, L // 2)


def estimate_noise_variance(stack: np.ndarray) -> float:
    """sigma^2 = mean of the angularly averaged variance of the mean-subtracted images over the outer 10 % of
    radii below L/2: bins ceil(0.45 L) <= b < floor(L/2)  ("levels off at ... the noise variance"; Q19)."""
    L = stack.shape[1]
    prof = _variance_profile(stack)
    return float(prof[int(np.ceil(0.45 * L - 1e-12)):].mean())


def _fraction_point(w: np.ndarray, frac: float) -> int:
    tot = w.sum()
    if not tot > 0:
        raise ValueError("no signal above the noise level")
    return int(np.argmax(np.cumsum(w) >= frac * tot))


def estimate_support(stack: np.ndarray, sigma2: float, fraction: float = 0.999) -> float:
    """R = smallest radius bin at which the cumulative sum of max(var_b - sigma^2, 0) b (Jacobian r dr) reaches the
    fraction of its total over b < floor(L/2)  ("99.9% at r = 98")."""
    prof = _variance_profile(stack)
    b = np.arange(len(prof))
    return float(_fraction_point(np.maximum(prof - sigma2, 0.0) * b, fraction))


def estimate_bandlimit(stack: np.ndarray, sigma2: float, fraction: float = 0.999) -> float:
    """c = b / L for the smallest frequency bin 1 <= b <= floor(L/2) at which the cumulative sum of
    max(P_b - sigma^2, 0) b (Jacobian xi dxi) reaches the fraction of its total; P = mean |DFT2(I - mean)|^2 / L^2
    (white noise of variance s^2 -> level s^2, Q20), binned over integer frequencies ("c = 0.196")."""
    n, L, _ = stack.shape
    X = np.fft.fft2(stack - stack.mean(axis=0), axes=(1, 2))
    P = (np.abs(X) ** 2).mean(axis=0) / (L * L)
    f = np.round(np.fft.fftfreq(L) * L)
    prof = radial_profile(P, f, L // 2 + 1)
    b = np.arange(len(prof))
    w = np.maximum(prof - sigma2, 0.0) * b
    w[0] = 0.0
    return float(_fraction_point(w, fraction)) / L
