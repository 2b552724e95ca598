"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/fbspca.h declares, and its
host-side plan (census, GL rule, radial table, errors) agrees with the oracle.  No compute calls."""
import math
import os
import re

import numpy as np
import pytest
from scipy.special import jv

import oracle as O
import paper_1412_0781_b200 as F
from paper_1412_0781_b200._lib import LIB_PATH, SIGNATURES, FbspcaError, lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__ as g
    g.build()


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "fbspca.h")).read()
    declared = set(re.findall(r"\b(fbspca_[a-z_]+)\s*\(", hdr))
    declared = {d for d in declared if d not in ("fbspca_plan_t", "fbspca_stream_t")}
    assert declared, "no declarations parsed"
    L = lib()
    for name in sorted(declared):
        assert hasattr(L, name), f"{name} declared in fbspca.h but not exported by {LIB_PATH}"
    assert declared == set(SIGNATURES), "binding signatures out of sync with the header"
    assert b"sm_100a" in L.fbspca_version()


@pytest.mark.parametrize("L,R", [(32, 16), (33, 16), (64, 32), (128, 64)])
def test_host_plan_matches_oracle(L, R):
    pl = F.fbspca_plan(L, 0.5, R, device=-1)
    b = O.build_basis(0.5, R)
    assert pl.k_max == b.k_max and np.array_equal(pl.p, b.p)
    assert pl.n_xi == b.n_xi and pl.n_theta == b.n_theta
    zo = np.concatenate([z[:pk] for z, pk in zip(b.zeros, b.p)])
    assert np.max(np.abs(pl.zeros - zo)) < 1e-11
    xo, wo, _ = O.polar_grid(b)
    assert np.max(np.abs(pl.xi - xo)) < 1e-15 and np.max(np.abs(pl.wq - wo) / wo) < 1e-10
    assert np.array_equal(pl.coef_off, b.coef_off)
    assert pl.blk_off[-1] == sum(pk * (pk + 1) // 2 for pk in b.p)
    assert pl.n_theta % 2 == 0 and pl.M >= 2 * L


@pytest.mark.parametrize("L,c,R", [(240, 0.196, 98.0), (100, 0.3, 40.0)])
def test_host_plan_general_c(L, c, R):
    """c < 1/2 (the ribosome shape P:536: n_theta = ceil(16 c R) = 308 = 4 7 11, radix-7/11 angular FFTs)."""
    pl = F.fbspca_plan(L, c, R, device=-1)
    b = O.build_basis(c, R)
    assert pl.k_max == b.k_max and np.array_equal(pl.p, b.p)
    assert pl.n_xi == b.n_xi and pl.n_theta == b.n_theta
    xo, wo, _ = O.polar_grid(b)
    assert np.max(np.abs(pl.xi - xo)) < 1e-15


def test_plan_fft_size_error():
    with pytest.raises(FbspcaError, match="CONFIG"):       # n_theta = ceil(16 * 0.5 * 4.25) = 34 = 2 17
        F.fbspca_plan(16, 0.5, 4.25, device=-1)


def test_plan_window_and_phases():
    pl = F.fbspca_plan(128, 0.5, 64, device=-1)
    assert pl.w == 6 and abs(pl.beta - float(np.float32(2.3 * 6))) < 1e-12   # fp32 plans round beta to float (DESIGN Q16) and pl.M == 256
    assert 1 <= pl.n_phase <= 4 and pl.smem_bytes <= 227 * 1024
    pl64 = F.fbspca_plan(32, 0.5, 16, dtype=F.F64, device=-1)
    assert pl64.w == 13
    # eps >= 1e-4: w = 5 (compile-time-FFT and runtime-radix kernels alike); eps = 1e-6: w = 7
    pl5 = F.fbspca_plan(128, 0.5, 64, eps=1e-4, device=-1)
    assert pl5.w == 5 and pl5.M == 256 and abs(pl5.beta - float(np.float32(2.3 * 5))) < 1e-12
    assert pl5.n_phase == pl.n_phase and pl5.smem_bytes <= 227 * 1024
    assert F.fbspca_plan(64, 0.5, 32, eps=1e-4, device=-1).w == 5
    assert F.fbspca_plan(300, 0.5, 150, eps=1e-4, device=-1).w == 5
    assert F.fbspca_plan(32, 0.5, 16, eps=1e-4, device=-1).w == 5
    assert F.fbspca_plan(128, 0.25, 64, eps=1e-4, device=-1).w == 5
    assert F.fbspca_plan(240, 0.196, 98, eps=1e-4, device=-1).w == 5
    assert F.fbspca_plan(240, 0.196, 98, device=-1).w == 6
    assert F.fbspca_plan(128, 0.5, 64, eps=1e-6, device=-1).w == 7


@pytest.mark.parametrize("args,code", [
    ((64, 0.6, 32), "CONFIG"), ((64, 0.5, 40), "CONFIG"), ((64, 0.5, 1.5), "CONFIG"),
    ((64, 0.05, 10), "CONFIG"), ((2, 0.5, 1), "CONFIG"),
])
def test_plan_config_errors(args, code):
    with pytest.raises(FbspcaError, match=code):
        F.fbspca_plan(*args, device=-1)


def test_plan_eps_errors():
    with pytest.raises(FbspcaError, match="CONFIG"):
        F.fbspca_plan(64, 0.5, 32, eps=1e-8, device=-1)           # below the fp32 floor
    with pytest.raises(FbspcaError, match="CONFIG"):
        F.fbspca_plan(64, 0.5, 32, eps=1e-2, device=-1)
    F.fbspca_plan(64, 0.5, 32, eps=1e-8, dtype=F.F64, device=-1)


def test_host_only_plan_refuses_compute():
    import ctypes
    pl = F.fbspca_plan(32, 0.5, 16, device=-1)
    st = lib().fbspca_expand(ctypes.c_void_p(pl.handle), ctypes.c_void_p(16), 1, ctypes.c_void_p(16), None)
    assert st == 1 and b"host-only" in lib().fbspca_last_error()


def test_shard_range_partitions():
    for n in (1, 7, 100, 100_000):
        for world in (1, 2, 3, 8):
            spans = [F.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1


def test_unpack_blocks_layout():
    pl = F.fbspca_plan(32, 0.5, 16, device=-1)
    rng = np.random.default_rng(0)
    mats = []
    packed = np.zeros(pl.n_blk)
    for k in range(pl.k_max + 1):
        pk = int(pl.p[k])
        A = rng.standard_normal((pk, pk)); A = A + A.T
        mats.append(A)
        packed[pl.blk_off[k]:pl.blk_off[k + 1]] = A[np.triu_indices(pk)]
    got = F.unpack_blocks(pl, packed)
    assert all(np.array_equal(a, b) for a, b in zip(got, mats))


def _strided_angular(Fp, rs, k_max):
    """Eq. (1DFFT) on ring j sampled at every rs[j]-th angle: (2 pi s / n_theta) sum_{l = 0, s, 2s..} F e^{-ik theta_l},
    i.e. the (n_theta / s)-point DFT of the subsampled ring, indexed k mod (n_theta / s)."""
    n, n_xi, nt = Fp.shape
    out = np.empty((n, n_xi, k_max + 1), dtype=np.complex128)
    k = np.arange(k_max + 1)
    for j in range(n_xi):
        s = int(rs[j])
        nj = nt // s
        out[:, j, :] = (2 * np.pi / nj) * np.fft.fft(Fp[:, j, ::s], axis=-1)[:, k % nj]
    return out


def test_ring_stride_reading_against_oracle():
    """Reading Q21: the M = 256 plan samples inner rings at n_theta / s_j angles.  Against the oracle's
    exact direct sum (O5) on white-noise images (the most corner / high-angular content a square image has), ring j's
    Eq. (1DFFT) values for every k it feeds (k <= kneed(j), i.e. kj0[k] <= j) agree with the paper's n_theta-angle
    values to 1e-9 of the ring's largest value, and the Eq. (a) coefficients (K4's sum from kj0[k]) to 1e-8 rel l2 --
    four orders below the fp32 NUFFT error the path is held to.  Doubling any stride breaks the bound (the check has
    teeth: aliases of the ring's angular content land on the k it feeds)."""
    pl = F.fbspca_plan(128, 0.5, 64, device=-1)
    rs, kj0 = F.fbspca_plan_rings(pl)
    assert rs.max() >= 4 and rs.min() == 1 and np.all(np.diff(rs) <= 0)
    b = O.build_basis(0.5, 64)
    assert b.n_theta == pl.n_theta and b.k_max == pl.k_max
    imgs = np.random.default_rng(21).standard_normal((2, 128, 128))
    Fp = O.polar_ft_direct(imgs, b)
    g_full = O.angular_transform(Fp, b.k_max)
    g_str = _strided_angular(Fp, rs, b.k_max)
    kneed = np.array([max(k for k in range(b.k_max + 1) if kj0[k] <= j) for j in range(b.n_xi)])
    worst = 0.0
    for j in range(b.n_xi):
        scale = np.abs(g_full[:, j, :]).max()
        err = np.abs(g_str[:, j, :kneed[j] + 1] - g_full[:, j, :kneed[j] + 1]).max() / scale
        worst = max(worst, err)
    assert worst < 1e-9, worst
    # Eq. (a): K4 sums block k from ring kj0[k] on the strided rings
    table = O.radial_table(b)
    A_full = O.radial_quadrature(g_full, b, table)
    tab_cut = [t.copy() for t in table]
    for k in range(b.k_max + 1):
        tab_cut[k][:, :kj0[k]] = 0.0
    A_str = O.radial_quadrature(g_str, b, tab_cut)
    full, got = O.to_flat(A_full), O.to_flat(A_str)
    rel = np.linalg.norm(got - full, axis=0) / np.linalg.norm(full, axis=0)
    assert rel.max() < 1e-8, rel.max()
    # teeth: twice the plan's stride on the outermost ring of a stride class aliases visibly
    rs2 = rs.copy()
    j2 = int(np.nonzero(rs == 2)[0][-1])           # last ring the plan samples at every second angle
    rs2[j2] = 4
    g_bad = _strided_angular(Fp[:, j2:j2 + 1, :], rs2[j2:j2 + 1], b.k_max)
    bad = np.abs(g_bad[:, 0, :kneed[j2] + 1] - g_full[:, j2, :kneed[j2] + 1]).max() / np.abs(g_full[:, j2, :]).max()
    assert bad > 1e-6, bad
