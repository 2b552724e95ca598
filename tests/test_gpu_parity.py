"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded inputs.

Bars (BASELINE.json north_star): per-image coefficient relative l2 <= 1e-4 (reading Q12: k > 0 counted twice),
top-50 eigenvalues within 1e-4 relative, principal-subspace cosine >= 0.9999.  fp64 (C1) is held to 1e-9.
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
import paper_1412_0781_b200 as F
import synth

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0") if torch.cuda.is_available() else None
TOL32 = 1e-4


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g
    g.build()


def rel_l2_per_image(got, ref, basis):
    """Reading Q12: || a_gpu - a_orc || / || a_orc || per image, k > 0 rows weighted x2 (the +-k norm)."""
    wt = np.ones(ref.shape[0])
    wt[basis.p[0]:] = 2.0
    num = np.sqrt((wt[:, None] * np.abs(got - ref) ** 2).sum(0))
    den = np.sqrt((wt[:, None] * np.abs(ref) ** 2).sum(0))
    return num / den


def gpu_expand(plan, imgs_t):
    c = F.fbspca_expand(plan, imgs_t)
    torch.cuda.synchronize()
    return c.cpu().numpy().astype(np.complex128)


def blob_case(name, first, n, **kw):
    cfg = synth.config(name)
    imgs = synth.blob_images(cfg, first, n, device=DEV)
    return cfg, imgs


# ------------------------------------------------------------------ expansion (Alg. 1)
@pytest.mark.parametrize("name,n,max_batch", [("C2", 40, 4096), ("C2", 37, 16), ("C3", 12, 5)])
def test_expand_parity_blobs(name, n, max_batch):
    cfg, imgs = blob_case(name, 0, n)
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], device=0, max_batch=max_batch)
    got = gpu_expand(plan, imgs)
    basis = O.build_basis(cfg["c"], cfg["R"])
    ref = O.to_flat(O.expand(imgs.double().cpu().numpy(), basis))
    rel = rel_l2_per_image(got, ref, basis)
    assert rel.max() <= TOL32, f"max per-image rel l2 {rel.max():.3e}"
    assert np.all(got[: basis.p[0]].imag == 0)                    # Q8


def test_expand_parity_c1_fp64():
    imgs = synth.c1_images(256)
    plan = F.fbspca_plan(32, 0.5, 16, dtype=F.F64, device=0)
    got = gpu_expand(plan, torch.from_numpy(imgs).to(DEV))
    basis = O.build_basis(0.5, 16)
    ref = O.to_flat(O.expand(imgs, basis))
    rel = rel_l2_per_image(got, ref, basis)
    print("C1 fp64 max per-image rel l2", rel.max())
    assert rel.max() <= 1e-9


@pytest.mark.parametrize("L,R", [(33, 16), (20, 10)])
def test_expand_odd_and_small_L(L, R):
    rng = np.random.default_rng(L)
    imgs = rng.standard_normal((5, L, L)).astype(np.float32)
    plan = F.fbspca_plan(L, 0.5, R, device=0)
    got = gpu_expand(plan, torch.from_numpy(imgs).to(DEV))
    basis = O.build_basis(0.5, R)
    ref = O.to_flat(O.expand(imgs.astype(np.float64), basis))
    assert rel_l2_per_image(got, ref, basis).max() <= TOL32


def test_expand_single_image_and_errors():
    cfg, imgs = blob_case("C2", 7, 1)
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], device=0)
    got = gpu_expand(plan, imgs)
    basis = O.build_basis(cfg["c"], cfg["R"])
    ref = O.to_flat(O.expand(imgs.double().cpu().numpy(), basis))
    assert rel_l2_per_image(got, ref, basis).max() <= TOL32
    with pytest.raises(F.FbspcaError, match="ARG"):
        F.fbspca_expand(plan, imgs[:0])


def test_expand_rotation_reflection_on_gpu():
    """Eq. (rot)/(refl): rot90 -> a e^{-ik pi/2}, flip axis 0 -> conj(a), on the CUDA path (odd L)."""
    rng = np.random.default_rng(9)
    I = rng.standard_normal((1, 33, 33)).astype(np.float32)
    batch = np.concatenate([I, np.rot90(I, 1, axes=(1, 2)), I[:, ::-1, :]]).copy()
    plan = F.fbspca_plan(33, 0.5, 16, device=0)
    a = gpu_expand(plan, torch.from_numpy(batch).to(DEV))
    basis = O.build_basis(0.5, 16)
    A = O.from_flat(a, basis)
    scale = np.abs(a[:, 0]).max()
    for k in range(basis.k_max + 1):
        assert np.max(np.abs(A[k][:, 1] - A[k][:, 0] * np.exp(-1j * k * np.pi / 2))) <= 1e-4 * scale
        assert np.max(np.abs(A[k][:, 2] - np.conj(A[k][:, 0]))) <= 1e-4 * scale


@pytest.mark.parametrize("eps", [1e-5, 1e-4])
@pytest.mark.parametrize("name,n", [("C4", 2), ("C5", 1), ("T3", 1), ("RB", 2)])
def test_expand_parity_large_L(name, n, eps):
    cfg, imgs = blob_case(name, 0, n)
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], eps=eps, device=0, max_batch=64)
    assert plan.w == (5 if eps >= 1e-4 else 6)
    got = gpu_expand(plan, imgs)
    basis = O.build_basis(cfg["c"], cfg["R"])
    ref = O.to_flat(O.expand(imgs.double().cpu().numpy(), basis))
    rel = rel_l2_per_image(got, ref, basis)
    assert rel.max() <= TOL32, f"{name}: {rel.max():.3e}"


# ------------------------------------------------------------------ covariance / eig / projection (Alg. 2)
def _subspace_cos(Ug, Uo, lam_o, r):
    """sigma_min(U_gpu[:, :r]^T U_orc[:, :r]), r extended across near-ties (Q10)."""
    while r < len(lam_o) and abs(lam_o[r - 1] - lam_o[r]) <= 1e-3 * abs(lam_o[r - 1]):
        r += 1
    s = np.linalg.svd(Ug[:, :r].T @ Uo[:, :r], compute_uv=False)
    return s.min()


def test_spca_parity_c2_subset():
    cfg, imgs = blob_case("C2", 0, 600)
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], device=0, max_batch=256)
    coeffs = F.fbspca_expand(plan, imgs)
    blocks, mean = F.fbspca_covariance(plan, coeffs)
    evals, evecs = F.fbspca_eig(plan, blocks)
    sigma2 = (synth.blobs.noise_sigma(cfg, device=DEV)) ** 2
    out = F.fbspca_project(plan, coeffs, mean, evals, evecs, sigma2=sigma2, mode=1)
    torch.cuda.synchronize()
    basis = O.build_basis(cfg["c"], cfg["R"])
    A = O.expand(imgs.double().cpu().numpy(), basis)
    m_o, C_o = O.block_covariance(A)
    lam_o, U_o = O.block_eig(C_o)
    # covariance blocks
    C_g = F.unpack_blocks(plan, blocks.cpu().numpy())
    scale = max(np.abs(c).max() for c in C_o)
    assert max(np.abs(a - b).max() for a, b in zip(C_g, C_o)) <= 1e-4 * scale
    assert np.allclose(mean.cpu().numpy(), m_o, atol=1e-4 * np.abs(m_o).max())
    # top-50 eigenvalues (Q11 pooling)
    lam_g, U_g = F.split_eig(plan, evals.cpu().numpy(), evecs.cpu().numpy())
    pool_o = sorted(((-l, k, i) for k, lk in enumerate(lam_o) for i, l in enumerate(lk)))[:50]
    worst = max(abs(lam_g[k][i] - lam_o[k][i]) / abs(lam_o[k][i]) for _, k, i in pool_o)
    assert worst <= 1e-4, f"top-50 eigenvalue rel err {worst:.2e}"
    # principal subspaces per k
    for k in sorted({k for _, k, _ in pool_o}):
        r = sum(1 for _, kk, _ in pool_o if kk == k)
        assert _subspace_cos(U_g[k], U_o[k], lam_o[k], r) >= 0.9999
    # eigvec orthonormality on the GPU
    for Uk in U_g:
        assert np.allclose(Uk.T @ Uk, np.eye(Uk.shape[0]), atol=1e-10)
    # projection + MP/Wiener filter (mode 1) on well-separated leading components
    ref = O.project(A, m_o, U_o, lam_o, basis, sigma2, 1, A[0].shape[1])
    got = O.from_flat(out.cpu().numpy().astype(np.complex128), basis)
    for k in range(basis.k_max + 1):
        gaps = np.abs(np.diff(lam_o[k])) / np.maximum(np.abs(lam_o[k][:-1]), 1e-30)
        for l in range(min(3, basis.p[k])):
            if l < len(gaps) and gaps[l] > 1e-2 and (l == 0 or gaps[l - 1] > 1e-2):
                nrm = np.linalg.norm(ref[k][l]) + 1e-30
                assert np.linalg.norm(got[k][l] - ref[k][l]) <= 1e-3 * nrm + 1e-6 * np.linalg.norm(A[k])


def test_spca_parity_c1_fp64():
    imgs = synth.c1_images(256)
    plan = F.fbspca_plan(32, 0.5, 16, dtype=F.F64, device=0)
    coeffs = F.fbspca_expand(plan, torch.from_numpy(imgs).to(DEV))
    blocks, mean = F.fbspca_covariance(plan, coeffs)
    evals, evecs = F.fbspca_eig(plan, blocks)
    out = F.fbspca_project(plan, coeffs, mean, evals, evecs)
    torch.cuda.synchronize()
    basis = O.build_basis(0.5, 16)
    A = O.expand(imgs, basis)
    m_o, C_o = O.block_covariance(A)
    lam_o, U_o = O.block_eig(C_o)
    C_g = F.unpack_blocks(plan, blocks.cpu().numpy())
    scale = max(np.abs(c).max() for c in C_o)
    assert max(np.abs(a - b).max() for a, b in zip(C_g, C_o)) <= 1e-9 * scale
    lam_g, U_g = F.split_eig(plan, evals.cpu().numpy(), evecs.cpu().numpy())
    for lg, lo in zip(lam_g, lam_o):
        assert np.max(np.abs(lg - lo)) <= 1e-9 * max(1.0, np.abs(lo).max())
    got = O.from_flat(out.cpu().numpy(), basis)
    _, Ac = O.mean_and_center(A)
    for gk, ak in zip(got, Ac):      # orthonormal change of basis preserves per-image norms
        assert np.allclose(np.linalg.norm(gk, axis=0), np.linalg.norm(ak, axis=0), rtol=1e-8, atol=1e-12)


def test_eig_random_spd_blocks_vs_numpy():
    """K6 alone: feed packed random symmetric blocks (p up to 63) and compare with eigh."""
    plan = F.fbspca_plan(128, 0.5, 64, device=0)
    rng = np.random.default_rng(11)
    packed = np.zeros(plan.n_blk)
    mats = []
    for k in range(plan.k_max + 1):
        pk = int(plan.p[k])
        X = rng.standard_normal((pk, pk + 3))
        Cm = X @ X.T / (pk + 3) + np.diag(np.linspace(0, 1, pk))
        mats.append(Cm)
        packed[plan.blk_off[k]:plan.blk_off[k + 1]] = Cm[np.triu_indices(pk)]
    evals, evecs = F.fbspca_eig(plan, torch.from_numpy(packed).to(DEV))
    lam_g, U_g = F.split_eig(plan, evals.cpu().numpy(), evecs.cpu().numpy())
    lam_o, U_o = O.block_eig(mats)
    for Cm, lg, lo, Ug in zip(mats, lam_g, lam_o, U_g):
        assert np.max(np.abs(lg - lo)) <= 1e-11 * np.abs(lo).max()
        assert np.allclose(Ug @ np.diag(lg) @ Ug.T, Cm, atol=1e-11 * np.abs(Cm).max())


def test_covariance_virtual_shards_and_partial_api():
    """Sum of shard partials (shards aligned to the 4096-image accumulation batches) == the full partial."""
    cfg, imgs = blob_case("C2", 0, 10_000)
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], device=0)
    coeffs = F.fbspca_expand(plan, imgs)
    full = F.fbspca_covariance_partial(plan, coeffs).clone()
    parts = []
    for s, e in ((0, 4096), (4096, 8192), (8192, 10_000)):
        parts.append(F.fbspca_covariance_partial(plan, coeffs[:, s:e].contiguous()).clone())
    tot = sum(parts)
    assert torch.allclose(tot, full, rtol=1e-12, atol=1e-9)
    b1, m1 = F.fbspca_covariance_finalize(plan, tot)
    b2, m2 = F.fbspca_covariance(plan, coeffs)
    assert torch.allclose(b1, b2, rtol=1e-12, atol=1e-12) and torch.allclose(m1, m2)
    # PSD + symmetry of the finalised blocks
    for Ck in F.unpack_blocks(plan, b2.cpu().numpy()):
        assert np.linalg.eigvalsh(Ck).min() >= -1e-6 * np.abs(Ck).max()


def _oracle_cov_from_gpu_coeffs(coeffs, basis, chunk=8192):
    """fp64 oracle K5 (O.covariance_partials per chunk, O.finalize_covariance) on the GPU's coefficients."""
    n = coeffs.shape[1]
    S = s0 = None
    for c0 in range(0, n, chunk):
        A = O.from_flat(coeffs[:, c0:c0 + chunk].cpu().numpy().astype(np.complex128), basis)
        Sc, s0c, _ = O.covariance_partials(A)
        S = Sc if S is None else [a + b for a, b in zip(S, Sc)]
        s0 = s0c if s0 is None else s0 + s0c
    return O.finalize_covariance(S, s0, n)


def _spectral_checks(plan, blocks, mean, evals, evecs, m_o, C_o, tol_c=1e-4):
    lam_o, U_o = O.block_eig(C_o)
    C_g = F.unpack_blocks(plan, blocks.cpu().numpy())
    scale = max(np.abs(c).max() for c in C_o)
    err_c = max(np.abs(a - b).max() for a, b in zip(C_g, C_o)) / scale
    assert err_c <= tol_c, f"covariance blocks rel err {err_c:.2e}"
    assert np.allclose(mean.cpu().numpy(), m_o, rtol=1e-6, atol=1e-6 * np.abs(m_o).max())
    lam_g, U_g = F.split_eig(plan, evals.cpu().numpy(), evecs.cpu().numpy())
    pool_o = sorted(((-l, k, i) for k, lk in enumerate(lam_o) for i, l in enumerate(lk)))[:50]
    worst = max(abs(lam_g[k][i] - lam_o[k][i]) / abs(lam_o[k][i]) for _, k, i in pool_o)
    assert worst <= 1e-4, f"top-50 eigenvalue rel err {worst:.2e}"
    for k in sorted({k for _, k, _ in pool_o}):
        r = sum(1 for _, kk, _ in pool_o if kk == k)
        assert _subspace_cos(U_g[k], U_o[k], lam_o[k], r) >= 0.9999, f"subspace k={k}"
    return err_c, worst


def test_c5_full_size_sampled_expansion():
    """configs[4] at full size (50,000 images of 360 x 360) in bench.py's launch configuration (expand batches of
    min(50,000, 40 GB of ghat) = 25,806 images): the first and last image of each batch (the CTAs' first and ragged
    last pass) against the fp64 oracle."""
    cfg = synth.config("C5")
    n = cfg["n"]
    imgs = synth.blob_images(cfg, 0, n, device=DEV)
    probe = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], device=-1)
    batch = min(50000, int(40e9 // ((probe.k_max + 1) * 2 * probe.n_xi * 4)))
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], device=0, max_batch=batch)
    coeffs = F.fbspca_expand(plan, imgs)
    torch.cuda.synchronize()
    pick = [0, batch - 1, batch, n - 1]
    sample = imgs[pick].double().cpu().numpy()
    got = coeffs[:, pick].cpu().numpy().astype(np.complex128)
    del imgs, coeffs
    basis = O.build_basis(cfg["c"], cfg["R"])
    ref = O.to_flat(O.expand(sample, basis))
    rel = rel_l2_per_image(got, ref, basis)
    assert rel.max() <= TOL32, f"max per-image rel l2 {rel.max():.3e}"


@pytest.mark.parametrize("name,n", [("C4", 2048), ("C5", 1024), ("RB", 2048)])
def test_large_L_spectral_parity_subset(name, n):
    """configs[3] (L = 256), configs[4] (L = 360, p_k up to 179) and the ribosome shape: a larger subset than
    test_gpu_parity_full.py's 512 images through K1-K6, oracle K5/K6 on the GPU coefficients (checks K5-K6)."""
    cfg, imgs = blob_case(name, 0, n)
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], device=0, max_batch=512)
    coeffs = F.fbspca_expand(plan, imgs)
    blocks, mean = F.fbspca_covariance(plan, coeffs)
    evals, evecs = F.fbspca_eig(plan, blocks)
    torch.cuda.synchronize()
    basis = O.build_basis(cfg["c"], cfg["R"])
    m_o, C_o = _oracle_cov_from_gpu_coeffs(coeffs, basis)
    _spectral_checks(plan, blocks, mean, evals, evecs, m_o, C_o)


@pytest.mark.parametrize("name", ["C2", "C3", "C5"])
def test_radial_eigenfunctions_parity(name):
    """Alg. 2 line 5 (Eq. (sPCArad)): GPU f^{k,l}(xi_j) from the GPU eigenvectors vs the oracle's
    f^{k,l} from the same eigenvectors (fp64 both: 1e-10), on random SPD blocks."""
    cfg = synth.config(name)
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], device=0, max_batch=16)
    rng = np.random.default_rng(21)
    packed = np.zeros(plan.n_blk)
    for k in range(plan.k_max + 1):
        pk = int(plan.p[k])
        X = rng.standard_normal((pk, pk + 2))
        packed[plan.blk_off[k]:plan.blk_off[k + 1]] = (X @ X.T)[np.triu_indices(pk)]
    evals, evecs = F.fbspca_eig(plan, torch.from_numpy(packed).to(DEV))
    f = F.fbspca_radial_eigenfunctions(plan, evecs)
    torch.cuda.synchronize()
    _, U_g = F.split_eig(plan, evals.cpu().numpy(), evecs.cpu().numpy())
    basis = O.build_basis(cfg["c"], cfg["R"])
    f_o = O.radial_eigenfunctions(basis, U_g)
    got = f.cpu().numpy()
    for k in range(basis.k_max + 1):
        fk = got[plan.coef_off[k]:plan.coef_off[k + 1]]
        assert np.max(np.abs(fk - f_o[k])) <= 1e-10 * max(1.0, np.abs(f_o[k]).max()), f"k={k}"


# ------------------------------------------------------------------ NEXT-1: back to pixels (denoising)
@pytest.mark.parametrize("name,n", [("C1", 6), ("C2", 5), ("C3", 3)])
def test_synthesize_parity(name, n):
    """fbspca_synthesize (Eq. (IFT_FB), reading Q2) vs O.synthesize_pixels on the same random coefficients."""
    cfg = synth.config(name)
    dt = F.F64 if cfg["dtype"] == "f64" else F.F32
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], dtype=dt, device=0, max_batch=16)
    basis = O.build_basis(cfg["c"], cfg["R"])
    rng = np.random.default_rng(31)
    a = [rng.standard_normal((pk, n)) + 1j * rng.standard_normal((pk, n)) for pk in basis.p]
    a[0] = a[0].real + 0j
    flat = O.to_flat(a)
    ct = torch.from_numpy(flat.astype(np.complex128 if dt == F.F64 else np.complex64)).to(DEV)
    img = F.fbspca_synthesize(plan, ct)
    torch.cuda.synchronize()
    ref = O.synthesize_pixels(O.from_flat(flat.astype(np.complex64).astype(np.complex128) if dt == F.F32 else flat,
                                          basis), basis, cfg["L"])
    got = img.cpu().numpy().astype(np.float64)
    tol = 1e-10 if dt == F.F64 else 1e-5
    assert np.max(np.abs(got - ref)) <= tol * np.abs(ref).max()


def test_denoise_pipeline_parity_c2():
    """NEXT-1 end to end on C2 images: expand -> covariance -> eig -> project(mode 1: MP + Wiener) ->
    backproject -> synthesize, each GPU stage fed the previous GPU stage, vs the oracle stage on the same inputs."""
    cfg, imgs = blob_case("C2", 0, 600)
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], device=0, max_batch=256)
    coeffs = F.fbspca_expand(plan, imgs)
    blocks, mean = F.fbspca_covariance(plan, coeffs)
    evals, evecs = F.fbspca_eig(plan, blocks)
    sigma2 = float(synth.blobs.noise_sigma(cfg, device=DEV)) ** 2
    chat = F.fbspca_project(plan, coeffs, mean, evals, evecs, sigma2=sigma2, mode=1)
    ahat = F.fbspca_backproject(plan, chat, mean, evecs)
    den = F.fbspca_synthesize(plan, ahat[:, :8].contiguous())
    torch.cuda.synchronize()
    basis = O.build_basis(cfg["c"], cfg["R"])
    lam_g, U_g = F.split_eig(plan, evals.cpu().numpy(), evecs.cpu().numpy())
    c_g = O.from_flat(chat.cpu().numpy().astype(np.complex128), basis)
    a_ref = O.backproject(c_g, mean.cpu().numpy(), U_g)
    a_got = O.from_flat(ahat.cpu().numpy().astype(np.complex128), basis)
    for x, y in zip(a_got, a_ref):
        assert np.allclose(x, y, atol=1e-5 * max(1.0, np.abs(y).max()))
    ref = O.synthesize_pixels([x[:, :8] for x in O.from_flat(ahat.cpu().numpy().astype(np.complex128), basis)],
                              basis, cfg["L"])
    assert np.max(np.abs(den.cpu().numpy() - ref)) <= 1e-5 * np.abs(ref).max()
    # denoising reduces the error to the clean images inside the support (the paper's use case)
    clean = synth.blob_images(cfg, 0, 8, device=DEV, sigma_n=0.0).cpu().numpy()
    idx = np.arange(cfg["L"]) - cfg["L"] // 2
    disk = (idx[:, None] ** 2 + idx[None, :] ** 2) <= cfg["R"] ** 2
    noisy = imgs[:8].cpu().numpy()
    assert np.linalg.norm((den.cpu().numpy() - clean)[:, disk]) < 0.5 * np.linalg.norm((noisy - clean)[:, disk])


# ------------------------------------------------------------------ NEXT-2: parameter estimation
@pytest.mark.parametrize("name,n", [("C2", 3000), ("C3", 600)])
def test_estimate_params_parity(name, n):
    """fbspca_estimate_params vs the oracle's estimators on the same stack: sigma^2 to 1e-9 relative (fp64 sums),
    R and c identical (bin indices; a tie within 1e-9 of the 0.999 threshold would be reported)."""
    cfg, imgs = blob_case(name, 0, n)
    s2, R, c = F.fbspca_estimate_params(imgs, 0.999)
    st = imgs.double().cpu().numpy()
    s2_o = O.estimate_noise_variance(st)
    assert abs(s2 - s2_o) <= 1e-9 * abs(s2_o)
    assert R == O.estimate_support(st, s2_o, 0.999)
    assert c == O.estimate_bandlimit(st, s2_o, 0.999)
    # the blob model's noise level (reading Q15) is what the estimator recovers
    sig = float(synth.blobs.noise_sigma(cfg, device=DEV))
    assert abs(s2 - sig ** 2) <= 0.05 * sig ** 2


# ------------------------------------------------------------------ SVD route (Alg. 2 line 4)
@pytest.mark.parametrize("name,n", [("C1", 1), ("C1", 5), ("C2", 8), ("C2", 40), ("C3", 24), ("RB", 16)])
def test_svd_route_parity(name, n):
    """fbspca_svd vs O.svd_route on the same (GPU-expanded) coefficients: eigenvalues, mean, eigenvectors of
    simple eigenvalues, and a complete orthonormal basis with C^(k) U = U Lambda on the null space too."""
    if name == "C1":
        cfg, imgs = synth.config("C1"), torch.from_numpy(synth.c1_images(n)).to(DEV)
    else:
        cfg, imgs = blob_case(name, 0, n)
    dt = F.F64 if cfg["dtype"] == "f64" else F.F32
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], dtype=dt, device=0, max_batch=64)
    coeffs = F.fbspca_expand(plan, imgs)
    evals, evecs, mean = F.fbspca_svd(plan, coeffs)
    torch.cuda.synchronize()
    basis = O.build_basis(cfg["c"], cfg["R"])
    A = O.from_flat(coeffs.cpu().numpy().astype(np.complex128), basis)
    m_o, lam_o, U_o = O.svd_route(A)
    _, C_o = O.block_covariance(A)
    ev, vv = evals.cpu().numpy(), evecs.cpu().numpy()
    assert np.max(np.abs(mean.cpu().numpy() - m_o)) <= 1e-12 * max(1.0, np.abs(m_o).max())
    for k in range(basis.k_max + 1):
        pk = basis.p[k]
        lg = ev[plan.coef_off[k]:plan.coef_off[k] + pk]
        Ug = vv[plan.evec_off[k]:plan.evec_off[k] + pk * pk].reshape(pk, pk)
        scale = max(lam_o[k].max(), 1e-300)
        assert np.max(np.abs(lg - lam_o[k])) <= 1e-10 * scale, f"k={k}"
        assert np.max(np.abs(Ug.T @ Ug - np.eye(pk))) <= 1e-11, f"k={k}"
        assert np.max(np.abs(C_o[k] @ Ug - Ug * lg[None, :])) <= 1e-9 * scale, f"k={k}"
        for l in range(pk):
            gap = min([abs(lam_o[k][l] - lam_o[k][j]) for j in range(pk) if j != l] + [np.inf])
            if lam_o[k][l] > 1e-6 * scale and gap > 1e-4 * scale:
                assert np.max(np.abs(Ug[:, l] - U_o[k][:, l])) <= 1e-6, f"k={k} l={l}"


def test_svd_route_matches_eig_route():
    """n > p_k: fbspca_svd and fbspca_covariance + fbspca_eig give the same eigenvalues (C2, 200 images), to the
    covariance kernels' accuracy."""
    cfg, imgs = blob_case("C2", 0, 200)
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], device=0, max_batch=256)
    coeffs = F.fbspca_expand(plan, imgs)
    ev_s, _, mean_s = F.fbspca_svd(plan, coeffs)
    blocks, mean = F.fbspca_covariance(plan, coeffs)
    ev_e, _ = F.fbspca_eig(plan, blocks)
    torch.cuda.synchronize()
    a, b = ev_s.cpu().numpy(), ev_e.cpu().numpy()
    for k in range(plan.k_max + 1):
        sl = slice(plan.coef_off[k], plan.coef_off[k + 1])
        # the covariance route runs k >= 1 on tcgen05 3xTF32 (about 1e-6 relative, K5)
        assert np.max(np.abs(a[sl] - b[sl])) <= 1e-5 * max(b[sl].max(), 1e-300)
    assert torch.allclose(mean_s, mean.to(torch.float64), rtol=0, atol=1e-12)
