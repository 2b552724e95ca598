"""Pins for the fp64 oracle against what the paper and the mathematics fix (no GPU).

Each test names the passage it pins.  P:n = PAPER.md line n, S:n = SPEC.md line n.
A plausible slip in the oracle (dropped term, wrong sign/index, transposed operand,
wrong prefactor or orientation) fails at least one of these.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.special import jn_zeros, jv

import oracle as O
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


# ---------------------------------------------------------------- O1 census
def test_bessel_zero_values():
    g = GOLD["bessel"]
    z0 = O.bessel_zeros_upto(0, 3.0)
    assert abs(z0[0] - g["j_0_1"]) < 1e-12
    z1 = O.bessel_zeros_upto(1, 17.0)
    assert abs(z1[4] - g["R_1_5"]) < 1e-11


@pytest.mark.parametrize("k", [0, 1, 7, 50, 182])
def test_bessel_zeros_vs_library(k):
    X = 2 * math.pi * 0.5 * 64
    z = O.bessel_zeros_upto(k, X)
    ref = jn_zeros(k, len(z))
    assert np.max(np.abs(z - ref)) < 1e-10
    assert z[-1] > X and (len(z) < 2 or z[-2] <= X)
    # residual and interlacing R_{k,q} < R_{k+1,q} < R_{k,q+1}
    assert np.max(np.abs(jv(k, z))) < 1e-12
    zn = O.bessel_zeros_upto(k + 1, X)
    m = min(len(z) - 1, len(zn))
    assert np.all(z[:m] < zn[:m]) and np.all(zn[:m] < z[1:m + 1])


def test_census_0p5_30():
    g = GOLD["census_0.5_30"]
    b = O.build_basis(0.5, 30)
    assert b.p[0] == g["p0"] and b.n_xi == g["n_xi"] and b.n_theta == g["n_theta"]
    gg = GOLD["grid_0.196_98"]
    assert O.fb._ceil_int(4 * 0.196 * 98) == gg["n_xi"] and O.fb._ceil_int(16 * 0.196 * 98) == gg["n_theta"]


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_census_configs_and_paper_bounds(name):
    c, R, kmax, p0, ncoef = GOLD["census_configs"][name]
    if name in ("C4", "C5"):
        pytest.importorskip("scipy")
    b = O.build_basis(c, R)
    assert (b.k_max, b.p[0], b.n_coef) == (kmax, p0, ncoef)
    X = 2 * math.pi * c * R
    # Eq. (kmaxbs) P:154 and the total-count bounds P:157
    assert 4 * c * R - 3.517 < b.k_max < 2 * math.pi * c * R - 2.042
    ptot = b.p[0] + 2 * sum(b.p[1:])
    assert 8 * (c * R) ** 2 <= ptot <= 4 * math.pi * (c * R) ** 2
    for k, pk in enumerate(b.p):
        # Eq. (pkbs) P:149 (approximate: the paper uses 2 pi c R ~ R_{k,p_k+1}); one unit of slack
        assert 2 * c * R - k / 2 - 3.035 / 4 - 1 < pk < 2 * c * R - k / math.pi + 1.4 / 4 + 1
        # Eq. (criterion1) P:120 exactly: R_{k,p_k+1} <= X < R_{k,p_k+2}
        z = b.zeros[k]
        assert z[pk] <= X
        assert jn_zeros(k, pk + 2)[-1] > X
        if k:
            assert pk <= b.p[k - 1]          # p_k non-increasing
    assert jn_zeros(b.k_max + 1, 2)[1] > X   # p_{k_max+1} = 0


# ---------------------------------------------------------------- O2 GL
def test_gauss_legendre():
    g = GOLD["gl2"]
    x, w = O.gauss_legendre(2, 0.0, 1.0)
    assert np.allclose(x, g["nodes"], atol=1e-15) and np.allclose(w, g["weights"], atol=1e-15)
    x, w = O.gauss_legendre(8, 0.0, 0.5)
    for d in range(16):                                   # exact to degree 2m-1
        assert abs(np.sum(w * x ** d) - 0.5 ** (d + 1) / (d + 1)) < 1e-15 * max(1, 0.5 ** d) + 1e-16
    assert np.all(np.diff(x) > 0) and 0 < x[0] and x[-1] < 0.5


# ---------------------------------------------------------------- O3 table: quadrature orthonormality
@pytest.mark.parametrize("R,tol", [(16, 1e-5), (32, 1e-7), (64, 1e-12)])
def test_quadrature_orthonormality(R, tol):
    """2 pi sum_j N J_k(R_q xi_j/c) N J_k(R_q' xi_j/c) xi_j w_j = delta_{qq'}  (Lommel closed form
    int_0^c J_k(R_q xi/c)^2 xi dxi = (c^2/2) J_{k+1}(R_q)^2).  Tolerance scales with R (F4)."""
    b = O.build_basis(0.5, R)
    xi, w, _ = O.polar_grid(b)
    B = O.radial_table(b)
    worst = 0.0
    for k in range(b.k_max + 1):
        rad = b.norm[k][:, None] * jv(k, np.outer(b.zeros[k][: b.p[k]], xi) / b.c)
        G = 2 * np.pi * rad @ B[k].T
        worst = max(worst, np.max(np.abs(G - np.eye(b.p[k]))))
        # the table is N J_k(...) xi w (Eq. (a)): pin its xi_j w_j factor separately
        assert np.allclose(B[k], rad * (xi * w)[None, :], rtol=0, atol=1e-15 * np.abs(rad).max())
    assert worst < tol


def test_lommel_normalisation_closed_form():
    """N_{k,q} = (c sqrt(pi) |J_{k+1}(R_{k,q})|)^{-1} makes int |psi|^2 = 1, checked by a
    600-point GL rule that is exact to machine precision for these integrands."""
    b = O.build_basis(0.5, 12)
    x, w = O.gauss_legendre(600, 0.0, b.c)
    for k in (0, 3, 11):
        for q in range(b.p[k]):
            f = b.norm[k][q] * jv(k, b.zeros[k][q] * x / b.c)
            assert abs(2 * np.pi * np.sum(f * f * x * w) - 1.0) < 1e-12


# ---------------------------------------------------------------- worked example
def test_psi_1_5_worked_example():
    g = GOLD["psi_1_5"]
    b = O.build_basis(g["c"], g["R"])
    xi, _, th = O.polar_grid(b)
    k, q = g["k"], g["q"]
    F = (b.norm[k][q - 1] * jv(k, b.zeros[k][q - 1] * xi / b.c))[:, None] * np.exp(1j * k * th)[None, :]
    a = O.to_flat(O.expand_polar(F[None], b))[:, 0]
    ref = np.zeros_like(a)
    ref[b.coef_off[k] + q - 1] = 1.0
    e = np.abs(a - ref)
    rmse, mx = math.sqrt(np.mean(e ** 2)), e.max()
    assert rmse <= 10 * g["rmse_paper"] and mx <= 10 * g["max_abs_paper"]


def test_polar_synthesis_round_trip():
    """expand_polar(synthesize_polar(a)) = a with the closed-form table; error <= 10 E(R)."""
    b = O.build_basis(0.5, 64)
    rng = np.random.default_rng(1)
    A = [rng.standard_normal((pk, 3)) + 1j * rng.standard_normal((pk, 3)) for pk in b.p]
    A[0] = A[0].real + 0j
    back = O.expand_polar(O.synthesize_polar(A, b), b)
    err = np.linalg.norm(O.to_flat(back) - O.to_flat(A)) / np.linalg.norm(O.to_flat(A))
    assert err < 1e-12


# ---------------------------------------------------------------- O5 direct sum (Eq. nufft) pins
def test_direct_sum_delta_images():
    """Delta at the centre -> F == 1 (unit prefactor, reading Q1); delta at i=(1,0) -> e^{-2 pi i xi_1};
    delta at i=(0,1) -> e^{-2 pi i xi_2} (orientation: axis 0 multiplies xi_1 = xi cos theta, Q3)."""
    b = O.build_basis(0.5, 8)
    L = 17
    xi, _, th = O.polar_grid(b)
    X1, X2 = np.outer(xi, np.cos(th)), np.outer(xi, np.sin(th))
    I = np.zeros((3, L, L))
    c0 = L // 2
    I[0, c0, c0] = 1
    I[1, c0 + 1, c0] = 1
    I[2, c0, c0 + 1] = 1
    F = O.polar_ft_direct(I, b)
    assert np.max(np.abs(F[0] - 1)) < 1e-14
    assert np.max(np.abs(F[1] - np.exp(-2j * np.pi * X1))) < 1e-14
    assert np.max(np.abs(F[2] - np.exp(-2j * np.pi * X2))) < 1e-14


@pytest.mark.parametrize("dense", [True, False])
def test_direct_sum_matches_brute_force(dense):
    """Both summation orders of O5 (dense kernel matrix / separable) against the double sum written out."""
    b = O.build_basis(0.5, 4)
    L = 9
    rng = np.random.default_rng(2)
    I = rng.standard_normal((2, L, L))
    F = O.polar_ft_direct(I, b, dense=dense, node_chunk=7)
    xi, _, th = O.polar_grid(b)
    idx = np.arange(L) - L // 2
    for j in (0, b.n_xi - 1):
        for l in (0, 3, b.n_theta // 2 + 1, b.n_theta - 1):
            x1, x2 = xi[j] * math.cos(th[l]), xi[j] * math.sin(th[l])
            ref = sum(I[1, a, bb] * np.exp(-2j * np.pi * (x1 * idx[a] + x2 * idx[bb]))
                      for a in range(L) for bb in range(L))
            assert abs(F[1, j, l] - ref) < 1e-12


def test_direct_sum_orders_agree():
    """The dense (n >= 32) and separable (n < 32) orders of the same sum agree to rounding at L = 33, R = 16."""
    b = O.build_basis(0.5, 16)
    I = np.random.default_rng(5).standard_normal((3, 33, 33))
    Fd = O.polar_ft_direct(I, b, dense=True)
    Fs = O.polar_ft_direct(I, b, dense=False)
    assert np.max(np.abs(Fd - Fs)) < 1e-12 * np.abs(Fd).max()


# ---------------------------------------------------------------- O6 angular pins
def test_angular_single_harmonics():
    nt, kmax = 32, 10
    th = 2 * np.pi * np.arange(nt) / nt
    F = np.stack([np.full(nt, 0.7 + 0.2j), np.exp(1j * th), np.exp(3j * th)])[None]
    g = O.angular_transform(F, kmax)[0]
    e0 = np.zeros(kmax + 1, complex); e0[0] = 2 * np.pi * (0.7 + 0.2j)
    e1 = np.zeros(kmax + 1, complex); e1[1] = 2 * np.pi
    e3 = np.zeros(kmax + 1, complex); e3[3] = 2 * np.pi
    for got, ref in zip(g, (e0, e1, e3)):
        assert np.max(np.abs(got - ref)) < 1e-13


# ---------------------------------------------------------------- exact recovery from pixel synthesis
def test_pixel_grid_recovery_and_sign_reading():
    """Images synthesised from known coefficients with Eq. (IFT_FB) (reading Q2: i^{+k} numerator) are
    recovered by the oracle; the truncation error shrinks on zero-padded grids.  The printed form (i^k in the
    denominator) does not recover (F2).  Pins prefactor (Q1), sign and orientation (Q3)."""
    b = O.build_basis(0.5, 16)
    errs = []
    for L in (32, 64):
        imgs, co = synth.c1_images(4, L=L, sigma=0.0, return_coeffs=True, mask=False)
        a = O.expand(imgs, b)
        errs.append(np.linalg.norm(O.to_flat(a) - O.to_flat(co)) / np.linalg.norm(O.to_flat(co)))
    assert errs[0] < 1e-2 and errs[1] < 0.3 * errs[0]
    # printed (misprinted) variant: i^k in the denominator == i^{-k} numerator
    p, zeros = synth.fb_census_scipy(0.5, 16)
    co_conj = [np.conj(1j ** (-2 * k)) * Ak for k, Ak in enumerate(co)]   # i^{-k} = i^{k} * i^{-2k}
    imgs_bad = synth.synth_fb_images(co_conj, zeros, 0.5, 16, 32, mask=False)
    a_bad = O.expand(imgs_bad, b)
    bad = np.linalg.norm(O.to_flat(a_bad) - O.to_flat(co)) / np.linalg.norm(O.to_flat(co))
    assert bad > 0.3


# ---------------------------------------------------------------- O(2) identities (Eqs. rot, refl)
def test_rotation_reflection_identities_odd_L():
    b = O.build_basis(0.5, 16)
    assert b.n_theta % 4 == 0
    L = 33
    rng = np.random.default_rng(3)
    I = rng.standard_normal((1, L, L))
    a = O.expand(I, b)
    rot = O.expand(np.rot90(I, 1, axes=(1, 2)).copy(), b)          # CCW 90 deg in (i1, i2)
    fud = O.expand(I[:, ::-1, :].copy(), b)                          # x -> -x
    flr = O.expand(I[:, :, ::-1].copy(), b)                          # y -> -y
    scale = np.abs(O.to_flat(a)).max()
    for k in range(b.k_max + 1):
        assert np.max(np.abs(rot[k] - a[k] * np.exp(-1j * k * np.pi / 2))) < 1e-12 * scale
        assert np.max(np.abs(fud[k] - np.conj(a[k]))) < 1e-12 * scale
        assert np.max(np.abs(flr[k] - (-1) ** k * np.conj(a[k]))) < 1e-12 * scale
    # rotate_coeffs / reflect_coeffs agree with those identities (Eqs. (rot), (refl) P:292)
    r2 = O.rotate_coeffs(a, np.pi / 2)
    assert max(np.max(np.abs(x - y)) for x, y in zip(r2, rot)) < 1e-12 * scale
    # reflect_coeffs(a, alpha) = conj(a) e^{-ik alpha}: alpha = 0 is the flip of axis 0 (x -> -x), alpha = pi the flip
    # of axis 1, alpha = pi/2 the flip followed by the 90-degree rotation.  A reflect_coeffs without the conj (a
    # rotation) or with the wrong phase sign fails at least one of the three.
    rud = O.expand(np.rot90(I[:, ::-1, :], 1, axes=(1, 2)).copy(), b)
    for alpha, ref in ((0.0, fud), (np.pi, flr), (np.pi / 2, rud)):
        got = O.reflect_coeffs(a, alpha)
        assert max(np.max(np.abs(x - y)) for x, y in zip(got, ref)) < 1e-12 * scale, alpha


# ---------------------------------------------------------------- white noise (Fig. 3)
def _dense_operator(b, L):
    """T* as a dense complex matrix (sum_k p_k x L^2): the oracle applied to every unit impulse."""
    E = np.eye(L * L).reshape(L * L, L, L)
    cols = O.to_flat(O.expand(E, b, chunk=64))
    return cols                                                      # (sum p_k, L^2)


def test_white_noise_blocks_near_sigma2_identity():
    b = O.build_basis(0.5, 16)
    L = 32
    T = _dense_operator(b, L)
    off = b.coef_off
    for k in range(b.k_max + 1):
        Tk = T[off[k]:off[k + 1]]
        Ek = np.real(Tk @ np.conj(Tk).T)                            # E[C^(k)] / sigma^2 (F6)
        ev = np.linalg.eigvalsh(Ek)
        assert ev.min() > 0.93 and ev.max() < 1.0 + 1e-3              # T* nearly unitary
    # sampled white noise, sigma^2 = 1: C^(k) vs sigma^2 Re(T_k T_k^H) within sampling error
    n = 6000
    X = np.random.default_rng(4).standard_normal((L * L, n))
    A = O.from_flat(T @ X, b)
    A[0] = A[0].real + 0j
    _, C = O.block_covariance(A)
    diag = np.concatenate([np.diag(Ck) for Ck in C])
    assert abs(diag.mean() - 1.0) < 0.02
    for k in (0, 1, 10, b.k_max):
        Tk = T[off[k]:off[k + 1]]
        Ek = np.real(Tk @ np.conj(Tk).T) * ((n - 1) / n if k == 0 else 1.0)
        assert np.max(np.abs(C[k] - Ek)) < 6.0 / math.sqrt(n)


# ---------------------------------------------------------------- brute-force augmented PCA
def test_bruteforce_augmented_covariance():
    b = O.build_basis(0.5, 4)
    nt = b.n_theta
    assert nt > 2 * b.k_max
    n = 6
    rng = np.random.default_rng(5)
    A = [rng.standard_normal((pk, n)) + 1j * rng.standard_normal((pk, n)) for pk in b.p]
    A[0] = A[0].real + 2.0 + 0j                                      # nonzero mean at k = 0
    ks = list(range(-b.k_max, b.k_max + 1))
    def full(Ai):  # coefficient vector over all k in ks
        return np.concatenate([Ai[abs(k)] if k >= 0 else np.conj(Ai[-k]) for k in ks])
    rows = []
    for i in range(n):
        Ai = [Ak[:, i] for Ak in A]
        for refl in (False, True):
            Bi = [np.conj(x) for x in Ai] if refl else Ai             # a_k -> a_{-k} (Eq. refl)
            v = full(Bi)
            kk = np.concatenate([np.full(b.p[abs(k)], k) for k in ks])
            for m in range(nt):
                rows.append(v * np.exp(-1j * kk * 2 * np.pi * m / nt))
    V = np.array(rows)                                                # (2 n nt, dims)
    mean = V.mean(axis=0)
    kk = np.concatenate([np.full(b.p[abs(k)], k) for k in ks])
    assert np.max(np.abs(mean[kk != 0])) < 1e-13                      # only k=0 survives (Eq. mean2)
    D = (V - mean).T @ np.conj(V - mean) / V.shape[0]
    m0, C = O.block_covariance(A)
    assert np.allclose(mean[kk == 0].real, m0, atol=1e-13)
    for k in ks:
        sel = np.nonzero(kk == k)[0]
        assert np.max(np.abs(D[np.ix_(sel, sel)] - C[abs(k)])) < 1e-12
        other = np.nonzero(kk != k)[0]
        assert np.max(np.abs(D[np.ix_(sel, other)])) < 1e-12        # block diagonal
    # dense spectrum = union of block spectra, k > 0 doubled (Fig. 7 pairs)
    dense = np.sort(np.linalg.eigvalsh(D))
    lam, _ = O.block_eig(C)
    blocks = np.sort(np.concatenate([lam[0]] + [np.repeat(l, 2) for l in lam[1:]]))
    assert np.allclose(dense, blocks, atol=1e-12)


# ---------------------------------------------------------------- eig, projection, MP
def _random_A(b, n, seed):
    rng = np.random.default_rng(seed)
    scale = [np.exp(-np.asarray(z[:pk]) / 20.0) for z, pk in zip(b.zeros, b.p)]
    A = [s[:, None] * (rng.standard_normal((pk, n)) + 1j * rng.standard_normal((pk, n)))
         for s, pk in zip(scale, b.p)]
    A[0] = A[0].real + 1.0 + 0j
    return A


def test_eig_matches_svd_route_and_sign_convention():
    """Alg. 2 line 4 alternatives: eig of C^(k) vs SVD of the real-augmented block."""
    b = O.build_basis(0.5, 8)
    n = 50
    A = _random_A(b, n, 6)
    mean, C = O.block_covariance(A)
    lam, U = O.block_eig(C)
    _, Ac = O.mean_and_center(A)
    for k, (Ak, lk, Uk) in enumerate(zip(Ac, lam, U)):
        M = np.concatenate([Ak.real, Ak.imag], axis=1) / math.sqrt(n)
        s = np.linalg.svd(M, compute_uv=False)
        sv = np.zeros(len(lk)); sv[: len(s)] = s ** 2
        assert np.allclose(lk, sv, atol=1e-12 * max(1, sv.max()))
        assert np.all(np.diff(lk) <= 1e-15)
        assert np.allclose(Uk @ np.diag(lk) @ Uk.T, C[k], atol=1e-12)
        for l in range(Uk.shape[1]):
            q = np.argmax(np.abs(Uk[:, l]))
            assert Uk[q, l] > 0


@pytest.mark.parametrize("n", [1, 4, 9])
def test_svd_route_rank_deficient(n):
    """O.svd_route (n < p_k): the eigenpairs of C^(k) (Eqs. (ck)/(ck_0)) from the SVD of A_k, with a
    complete basis and exactly p_k - rank zero eigenvalues (rank 2n for k >= 1, n - 1 for the centred k = 0)."""
    b = O.build_basis(0.5, 16)
    A = _random_A(b, n, 11)
    mean_c, C = O.block_covariance(A)
    lam_e, _ = O.block_eig(C)
    mean, lam, U = O.svd_route(A)
    assert np.allclose(mean, mean_c, atol=1e-15)
    for k, (lk, le, Uk, Ck) in enumerate(zip(lam, lam_e, U, C)):
        pk = b.p[k]
        scale = max(1.0, le.max())
        assert np.allclose(lk, le, atol=1e-12 * scale)
        rank = min(pk, n - 1 if k == 0 else 2 * n)
        assert np.all(lk[:rank] > 1e-8 * scale) and np.all(np.abs(lk[rank:]) <= 1e-12 * scale)
        assert np.allclose(Uk.T @ Uk, np.eye(pk), atol=1e-12)
        assert np.allclose(Ck @ Uk, Uk * lk[None, :], atol=1e-11 * scale)
        for l in range(pk):
            q = np.argmax(np.abs(Uk[:, l]))
            assert Uk[q, l] > 0


def test_projection_properties():
    b = O.build_basis(0.5, 8)
    n = 30
    A = _random_A(b, n, 7)
    mean, C = O.block_covariance(A)
    lam, U = O.block_eig(C)
    c = O.project(A, mean, U, lam, b, 0.0, 0, n)
    _, Ac = O.mean_and_center(A)
    for ck, ak in zip(c, Ac):                                          # norm preserving per block
        assert np.allclose(np.linalg.norm(ck, axis=0), np.linalg.norm(ak, axis=0), rtol=1e-12)
    alpha = 0.37                                                       # steerability
    c_rot = O.project(O.rotate_coeffs(A, alpha), mean, U, lam, b, 0.0, 0, n)
    for k, (x, y) in enumerate(zip(c_rot, c)):
        assert np.allclose(x, y * np.exp(-1j * k * alpha), atol=1e-12)
    eye = [np.eye(pk) for pk in b.p]
    c_id = O.spca_coeffs(Ac, eye)
    assert all(np.array_equal(x, y) for x, y in zip(c_id, Ac))


def test_mp_selection_and_shrinkage():
    g = GOLD["mp_select"]
    edge = g["sigma2"] * (1 + math.sqrt(g["gamma"])) ** 2
    assert abs(edge - 2.25) < 1e-15
    # gamma_k = p_k/(2n) for k > 0: p_k = 50, n = 100 -> gamma = 0.25
    assert abs(O.mp_edge(1.0, 50, 100, 1) - 2.25) < 1e-15
    assert abs(O.mp_edge(1.0, 25, 100, 0) - 2.25) < 1e-15             # gamma_0 = p_0/n
    b = O.Basis(c=0.5, R=1, k_max=1, p=[25, 50], zeros=[], norm=[])
    lam = [np.array([3.0, 2.2]), np.array([g["selected"], g["rejected"]])]
    h = O.shrink_weights(lam, b, 100, 1.0, 1)
    assert h[1][0] > 0 and h[1][1] == 0
    assert abs(h[0][0] - 2.0 / 3.0) < 1e-15                            # soft: l = 2, h = l/(l+s)
    # spiked mode inverts lambda = (l + s)(1 + g s / l) exactly
    ell, s2, gam = 4.0, 1.0, 0.25
    lam_sp = (ell + s2) * (1 + gam * s2 / ell)
    h2 = O.shrink_weights([np.array([lam_sp]), np.array([lam_sp])], b, 100, s2, 2)
    assert abs(h2[1][0] - ell / (ell + s2)) < 1e-12


def test_mp_select_edges_and_white_noise():
    """Eq. (compselect) P:692 with gamma_0 = p_0/n, gamma_k = p_k/(2n): strict '>' at the edge, the same
    selection shrink_weights(mode 1) makes, and on pure white noise in coefficient space (a_0 ~ N(0, s2),
    a_k ~ CN(0, s2): C^(k) is a real Wishart with 2n samples, Marcenko-Pastur edge s2 (1 + sqrt(p_k/(2n)))^2)
    the largest noise eigenvalue sits at the edge (a gamma_k = p_k/n slip moves the edge by 20 %), no noise
    component is selected and a planted spike far above the BBP threshold is."""
    b = O.Basis(c=0.5, R=1, k_max=1, p=[25, 50], zeros=[], norm=[])
    lam = [np.array([3.0, 2.25, 2.2]), np.array([2.26, 2.25, 1.0])]
    sel = O.mp_select(lam, b, 100, 1.0)
    assert sel[0].tolist() == [True, False, False] and sel[1].tolist() == [True, False, False]
    h = O.shrink_weights(lam, b, 100, 1.0, 1)
    assert all(np.array_equal(s, hk > 0) for s, hk in zip(sel, h))
    rng = np.random.default_rng(17)
    p, n, s2 = 100, 500, 2.0
    bw = O.Basis(c=0.5, R=1, k_max=1, p=[p, p], zeros=[], norm=[])
    a0 = rng.normal(0, math.sqrt(s2), (p, n)) + 0j
    a1 = (rng.normal(0, math.sqrt(s2 / 2), (p, n)) + 1j * rng.normal(0, math.sqrt(s2 / 2), (p, n)))
    u = rng.standard_normal(p); u /= np.linalg.norm(u)
    spike = (rng.normal(0, math.sqrt(5 * s2 / 2), n) + 1j * rng.normal(0, math.sqrt(5 * s2 / 2), n))
    _, C = O.block_covariance([a0, a1])
    lam_n, _ = O.block_eig(C)
    edge0, edge1 = O.mp_edge(s2, p, n, 0), O.mp_edge(s2, p, n, 1)
    assert abs(edge0 - s2 * (1 + math.sqrt(0.2)) ** 2) < 1e-12 and abs(edge1 - s2 * (1 + math.sqrt(0.1)) ** 2) < 1e-12
    assert abs(lam_n[0][0] / edge0 - 1) < 0.05 and abs(lam_n[1][0] / edge1 - 1) < 0.05
    assert sum(int(s.sum()) for s in O.mp_select(lam_n, bw, n, s2)) <= 1
    _, Cs = O.block_covariance([a0, a1 + np.outer(u, spike)])
    lam_s, _ = O.block_eig(Cs)
    sel_s = O.mp_select(lam_s, bw, n, s2)
    assert sel_s[1][0] and int(sel_s[1].sum()) <= 2


def test_covariance_shard_partials_and_invariance():
    b = O.build_basis(0.5, 8)
    A = _random_A(b, 40, 8)
    m, C = O.block_covariance(A)
    parts = [O.covariance_partials([Ak[:, s:e] for Ak in A]) for s, e in ((0, 13), (13, 29), (29, 40))]
    S = [sum(p[0][k] for p in parts) for k in range(b.k_max + 1)]
    s0 = sum(p[1] for p in parts)
    m2, C2 = O.finalize_covariance(S, s0, sum(p[2] for p in parts))
    assert np.allclose(m, m2, atol=1e-13)
    assert all(np.allclose(x, y, atol=1e-12) for x, y in zip(C, C2))
    for T in (O.rotate_coeffs(A, 1.1), O.reflect_coeffs(A, 0.4)):
        _, C3 = O.block_covariance(T)
        assert all(np.allclose(x, y, atol=1e-12) for x, y in zip(C, C3))


# ---------------------------------------------------------------- Alg. 2 line 5: radial eigenfunctions
def test_radial_eigenfunctions_basis_and_permutation():
    """U = permutation: f^{k,l} is exactly the Bessel basis function N J_k(R_{k,pi(l)} xi / c) (Eq. (sPCArad)),
    evaluated here from scipy's jn_zeros / jv -- catches a transposed U (pi vs pi^-1) or a dropped norm."""
    b = O.build_basis(0.5, 16)
    xi, _, _ = O.polar_grid(b)
    rng = np.random.default_rng(3)
    U, perms = [], []
    for k in range(b.k_max + 1):
        pi = rng.permutation(b.p[k])
        P = np.zeros((b.p[k], b.p[k]))
        P[pi, np.arange(b.p[k])] = 1.0                 # u_l(q) = [q == pi(l)]
        U.append(P)
        perms.append(pi)
    f = O.radial_eigenfunctions(b, U)
    for k in (0, 1, 7, b.k_max):
        z = jn_zeros(k, b.p[k])
        for l in range(b.p[k]):
            q = perms[k][l]
            ref = jv(k, z[q] * xi / b.c) / (b.c * math.sqrt(math.pi) * abs(jv(k + 1, z[q])))
            assert np.allclose(f[k][l], ref, rtol=1e-10, atol=1e-12)


def test_radial_eigenfunctions_orthonormal_and_consistent():
    """For orthogonal U_k the f^{k,l} are orthonormal, 2 pi int_0^c f f' xi dxi = delta (Bessel orthonormality,
    P:87; 600-point GL rule, exact here), and sum_l c_{k,l} f^{k,l} = sum_q a_{k,q} N J_k(R_q xi/c) (Eq. (sPCAcoeff))."""
    b = O.build_basis(0.5, 12)
    rng = np.random.default_rng(5)
    U = [np.linalg.qr(rng.standard_normal((pk, pk)))[0] for pk in b.p]
    x, w = O.gauss_legendre(600, 0.0, b.c)
    f = O.radial_eigenfunctions(b, U, xi=x)
    for k in range(b.k_max + 1):
        G = 2 * np.pi * (f[k] * (x * w)[None, :]) @ f[k].T
        assert np.max(np.abs(G - np.eye(b.p[k]))) < 1e-11
    a = [rng.standard_normal((pk, 3)) + 1j * rng.standard_normal((pk, 3)) for pk in b.p]
    c = O.spca_coeffs(a, U)
    f0 = O.radial_eigenfunctions(b, [np.eye(pk) for pk in b.p], xi=x)   # the Bessel basis itself
    for k in (0, 2, b.k_max):
        assert np.allclose(f[k].T @ c[k], f0[k].T @ a[k], atol=1e-11)


# ---------------------------------------------------------------- NEXT-1: pixel synthesis and back-projection
def test_synthesize_pixels_recovery_and_rotation():
    """O.synthesize_pixels (Eq. (IFT_FB), reading Q2) is inverted by the oracle's expansion up to the truncation
    error of the finite grid, which shrinks with zero padding (prefactor, sign, orientation, q-parity pinned:
    the (-1)^q with the paper's q = 1..p_k); rot90 of the image = a_k e^{-ik pi/2} at odd L."""
    b = O.build_basis(0.5, 16)
    rng = np.random.default_rng(12)
    v = [np.exp(-b.zeros[k][: b.p[k]] ** 2 / 200.0) for k in range(b.k_max + 1)]
    a = [np.sqrt(v[0])[:, None] * rng.standard_normal((b.p[0], 3)) + 0j] + \
        [np.sqrt(vk / 2)[:, None] * (rng.standard_normal((len(vk), 3)) + 1j * rng.standard_normal((len(vk), 3)))
         for vk in v[1:]]
    errs = []
    for L in (32, 64):
        img = O.synthesize_pixels(a, b, L, mask=False)
        got = O.expand(img, b)
        errs.append(np.linalg.norm(O.to_flat(got) - O.to_flat(a)) / np.linalg.norm(O.to_flat(a)))
    assert errs[0] < 1e-2 and errs[1] < 0.3 * errs[0]
    img = O.synthesize_pixels(a, b, 33)
    rot = O.synthesize_pixels(O.rotate_coeffs(a, np.pi / 2), b, 33)
    assert np.allclose(rot, np.rot90(img, k=1, axes=(1, 2)), atol=1e-12 * np.abs(img).max())


def test_backproject_inverts_projection():
    """backproject(spca_coeffs(centred a, U), mean, U) = a for orthogonal U (Eq. (sPCAcoeff) P:364 inverted)."""
    b = O.build_basis(0.5, 12)
    rng = np.random.default_rng(13)
    a = [rng.standard_normal((pk, 4)) + 1j * rng.standard_normal((pk, 4)) for pk in b.p]
    a[0] = a[0].real + 0j
    mean, Ac = O.mean_and_center(a)
    U = [np.linalg.qr(rng.standard_normal((pk, pk)))[0] for pk in b.p]
    back = O.backproject(O.spca_coeffs(Ac, U), mean, U)
    for x, y in zip(back, a):
        assert np.allclose(x, y, atol=1e-12)


# ---------------------------------------------------------------- NEXT-2: parameter estimation
def test_noise_variance_white_noise_and_homogeneity():
    """Pure white noise sigma = 3 (n = 1000, L = 64): sigma^2 within 3 % of 9 (SPEC example; "sigma^2 = 9");
    doubling the amplitudes quadruples the estimate; constant images give 0."""
    rng = np.random.default_rng(1)
    st = 3.0 * rng.standard_normal((1000, 64, 64))
    s2 = O.estimate_noise_variance(st)
    assert abs(s2 - 9.0) <= 0.03 * 9.0
    assert abs(O.estimate_noise_variance(2 * st) - 4 * s2) <= 1e-9 * s2
    assert O.estimate_noise_variance(np.ones((5, 32, 32))) == 0.0


def test_support_and_bandlimit_phantoms():
    """Signal filling the disk of radius 20 (i.i.d. pixels inside, zero outside; negligible noise): R in [19, 22].
    A phantom band-limited to c = 0.25 (white noise low-passed by an ideal disk filter): c in [0.23, 0.28].
    Pure noise raises (SPEC examples)."""
    rng = np.random.default_rng(2)
    idx = np.arange(64) - 32
    disk = np.hypot(*np.meshgrid(idx, idx, indexing="ij")) <= 20
    st = rng.standard_normal((200, 64, 64)) * disk + 1e-3 * rng.standard_normal((200, 64, 64))
    R = O.estimate_support(st, O.estimate_noise_variance(st), 0.999)
    assert 19 <= R <= 22, R
    L = 64
    f = np.fft.fftfreq(L)
    mask = np.hypot(*np.meshgrid(f, f, indexing="ij")) <= 0.25
    band = np.real(np.fft.ifft2(np.fft.fft2(rng.standard_normal((300, L, L))) * mask))
    c = O.estimate_bandlimit(band, 0.0, 0.999)
    assert 0.23 <= c <= 0.28, c
    with pytest.raises(ValueError):
        O.estimate_support(rng.standard_normal((50, 32, 32)), 10.0, 0.999)
