"""Thin Python binding of the C ABI (include/fbspca.h): same names, argument marshalling only.

Torch is used for device memory and streams.  Every step of the hot path runs in libfbspca.so's
kernels; nothing here computes on the data.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import FbspcaError, check, lib

F32, F64 = 0, 1


def _stream_ptr(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def _ptr(t: torch.Tensor) -> int:
    if not t.is_cuda:
        raise FbspcaError("tensor must live on a CUDA device")
    if not t.is_contiguous():
        raise FbspcaError("tensor must be contiguous")
    return t.data_ptr()


@dataclass
class Plan:
    handle: int
    L: int
    c: float
    R: float
    dtype: int
    device: int
    n_xi: int
    n_theta: int
    k_max: int
    p: np.ndarray
    coef_off: np.ndarray
    blk_off: np.ndarray
    evec_off: np.ndarray
    M: int
    w: int
    beta: float
    n_phase: int
    smem_bytes: int
    zeros: np.ndarray
    xi: np.ndarray
    wq: np.ndarray

    @property
    def n_coef(self) -> int:
        return int(self.coef_off[-1])

    @property
    def n_blk(self) -> int:
        return int(self.blk_off[-1])

    @property
    def n_partial(self) -> int:
        return int(self.blk_off[-1]) + int(self.p[0]) + 1

    @property
    def real_dtype(self):
        return torch.float32 if self.dtype == F32 else torch.float64

    @property
    def complex_dtype(self):
        return torch.complex64 if self.dtype == F32 else torch.complex128

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                lib().fbspca_destroy(ctypes.c_void_p(self.handle))
            except Exception:
                pass
            self.handle = 0


def fbspca_plan(L: int, c: float, R: float, eps: float = 0.0, dtype: int = F32, device: int = 0,
                max_batch: int = 4096) -> Plan:
    h = ctypes.c_void_p()
    check(lib().fbspca_plan(int(L), float(c), float(R), float(eps), int(dtype), int(device), int(max_batch),
                            ctypes.byref(h)), "fbspca_plan")
    n_xi, n_theta, k_max = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    pk = ctypes.POINTER(ctypes.c_int)()
    co, bo, eo = (ctypes.POINTER(ctypes.c_int64)() for _ in range(3))
    check(lib().fbspca_plan_info(h, ctypes.byref(n_xi), ctypes.byref(n_theta), ctypes.byref(k_max), ctypes.byref(pk),
                                 ctypes.byref(co), ctypes.byref(bo), ctypes.byref(eo)), "fbspca_plan_info")
    nk = k_max.value + 1
    M, w, nph, smem = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    beta = ctypes.c_double()
    zp, xp, wp = (ctypes.POINTER(ctypes.c_double)() for _ in range(3))
    check(lib().fbspca_plan_detail(h, ctypes.byref(M), ctypes.byref(w), ctypes.byref(beta), ctypes.byref(nph),
                                   ctypes.byref(smem), ctypes.byref(zp), ctypes.byref(xp), ctypes.byref(wp)),
          "fbspca_plan_detail")
    p = np.ctypeslib.as_array(pk, shape=(nk,)).copy()
    coef_off = np.ctypeslib.as_array(co, shape=(nk + 1,)).copy()
    return Plan(handle=h.value, L=L, c=c, R=R, dtype=dtype, device=device, n_xi=n_xi.value,
                n_theta=n_theta.value, k_max=k_max.value, p=p, coef_off=coef_off,
                blk_off=np.ctypeslib.as_array(bo, shape=(nk + 1,)).copy(),
                evec_off=np.ctypeslib.as_array(eo, shape=(nk + 1,)).copy(),
                M=M.value, w=w.value, beta=beta.value, n_phase=nph.value, smem_bytes=smem.value,
                zeros=np.ctypeslib.as_array(zp, shape=(int(coef_off[-1]),)).copy(),
                xi=np.ctypeslib.as_array(xp, shape=(n_xi.value,)).copy(),
                wq=np.ctypeslib.as_array(wp, shape=(n_xi.value,)).copy())


def fbspca_plan_rings(plan: Plan):
    """(ring_stride[n_xi], k_first_ring[k_max + 1]) of the plan (include/fbspca.h: fbspca_plan_rings)."""
    rs = np.zeros(plan.n_xi, dtype=np.int32)
    kj = np.zeros(plan.k_max + 1, dtype=np.int32)
    check(lib().fbspca_plan_rings(ctypes.c_void_p(plan.handle), rs.ctypes.data, kj.ctypes.data), "fbspca_plan_rings")
    return rs, kj


def _on_plan_device(plan: Plan, *tensors):
    for t in tensors:
        if t.device.type != "cuda" or t.device.index != plan.device:
            raise FbspcaError(f"tensor on {t.device}, plan on cuda:{plan.device}")


def _check_coeffs(plan: Plan, coeffs: torch.Tensor, n: int, what: str = "coeffs"):
    """The C ABI takes ld = n: a (n_coef, n) complex tensor of the plan's precision, contiguous."""
    if tuple(coeffs.shape) != (plan.n_coef, n) or coeffs.dtype != plan.complex_dtype:
        raise FbspcaError(f"{what} must be ({plan.n_coef}, {n}) {plan.complex_dtype}, got {tuple(coeffs.shape)} "
                          f"{coeffs.dtype}")


def fbspca_expand(plan: Plan, images: torch.Tensor, coeffs: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """images (n, L, L) on the plan's device -> coefficients (n_coef, n) complex (coefficient layout)."""
    n = images.shape[0]
    if images.dtype != plan.real_dtype or tuple(images.shape[1:]) != (plan.L, plan.L):
        raise FbspcaError(f"images must be (n, {plan.L}, {plan.L}) {plan.real_dtype}")
    _on_plan_device(plan, images)
    if coeffs is None:
        coeffs = torch.empty((plan.n_coef, n), dtype=plan.complex_dtype, device=images.device)
    _check_coeffs(plan, coeffs, n)
    _on_plan_device(plan, coeffs)
    check(lib().fbspca_expand(ctypes.c_void_p(plan.handle), _ptr(images), n, _ptr(coeffs), _stream_ptr(stream)),
          "fbspca_expand")
    return coeffs


def fbspca_covariance(plan: Plan, coeffs: torch.Tensor, n_local: int | None = None, n_total: int | None = None,
                      comm: int | None = None, blocks=None, mean=None, stream=None):
    n_local = coeffs.shape[1] if n_local is None else n_local
    n_total = n_local if n_total is None else n_total
    _check_coeffs(plan, coeffs, n_local)
    _on_plan_device(plan, coeffs)
    dev = coeffs.device
    if blocks is None:
        blocks = torch.empty(plan.n_blk, dtype=torch.float64, device=dev)
    if mean is None:
        mean = torch.empty(int(plan.p[0]), dtype=torch.float64, device=dev)
    check(lib().fbspca_covariance(ctypes.c_void_p(plan.handle), _ptr(coeffs), n_local, n_total,
                                  ctypes.c_void_p(comm or 0), _ptr(blocks), _ptr(mean), _stream_ptr(stream)),
          "fbspca_covariance")
    return blocks, mean


def fbspca_covariance_partial(plan: Plan, coeffs: torch.Tensor, partial=None, stream=None) -> torch.Tensor:
    _check_coeffs(plan, coeffs, coeffs.shape[1])
    if partial is None:
        partial = torch.empty(plan.n_partial, dtype=torch.float64, device=coeffs.device)
    check(lib().fbspca_covariance_partial(ctypes.c_void_p(plan.handle), _ptr(coeffs), coeffs.shape[1], _ptr(partial),
                                          _stream_ptr(stream)), "fbspca_covariance_partial")
    return partial


def fbspca_covariance_accumulate(plan: Plan, coeffs: torch.Tensor, partial: torch.Tensor, stream=None):
    check(lib().fbspca_covariance_accumulate(ctypes.c_void_p(plan.handle), _ptr(coeffs), coeffs.shape[1],
                                             _ptr(partial), _stream_ptr(stream)), "fbspca_covariance_accumulate")
    return partial


def fbspca_allreduce_partial(plan: Plan, partial: torch.Tensor, comm: int | None, stream=None):
    check(lib().fbspca_allreduce_partial(ctypes.c_void_p(plan.handle), _ptr(partial), ctypes.c_void_p(comm or 0),
                                         _stream_ptr(stream)), "fbspca_allreduce_partial")
    return partial


def fbspca_covariance_finalize(plan: Plan, partial: torch.Tensor, stream=None):
    blocks = torch.empty(plan.n_blk, dtype=torch.float64, device=partial.device)
    mean = torch.empty(int(plan.p[0]), dtype=torch.float64, device=partial.device)
    check(lib().fbspca_covariance_finalize(ctypes.c_void_p(plan.handle), _ptr(partial), _ptr(blocks), _ptr(mean),
                                           _stream_ptr(stream)), "fbspca_covariance_finalize")
    return blocks, mean


def fbspca_eig(plan: Plan, blocks: torch.Tensor, stream=None):
    evals = torch.empty(plan.n_coef, dtype=torch.float64, device=blocks.device)
    evecs = torch.empty(int(plan.evec_off[-1]), dtype=torch.float64, device=blocks.device)
    check(lib().fbspca_eig(ctypes.c_void_p(plan.handle), _ptr(blocks), _ptr(evals), _ptr(evecs), _stream_ptr(stream)),
          "fbspca_eig")
    return evals, evecs


def fbspca_svd(plan: Plan, coeffs: torch.Tensor, stream=None):
    """Alg. 2 line 4 via the SVD of A_k (the n < p_k route): (evals, evecs, mean) as fbspca_eig."""
    n = coeffs.shape[1]
    evals = torch.empty(plan.n_coef, dtype=torch.float64, device=coeffs.device)
    evecs = torch.empty(int(plan.evec_off[-1]), dtype=torch.float64, device=coeffs.device)
    mean = torch.empty(int(plan.p[0]), dtype=torch.float64, device=coeffs.device)
    check(lib().fbspca_svd(ctypes.c_void_p(plan.handle), _ptr(coeffs), n, _ptr(mean), _ptr(evals), _ptr(evecs),
                           _stream_ptr(stream)), "fbspca_svd")
    return evals, evecs, mean


def fbspca_radial_eigenfunctions(plan: Plan, evecs: torch.Tensor, stream=None) -> torch.Tensor:
    """Alg. 2 line 5: f^{k,l}(xi_j) as a (sum_k p_k) x n_xi fp64 tensor (row coef_off[k] + l)."""
    f = torch.empty((plan.n_coef, plan.n_xi), dtype=torch.float64, device=evecs.device)
    check(lib().fbspca_radial_eigenfunctions(ctypes.c_void_p(plan.handle), _ptr(evecs), _ptr(f), _stream_ptr(stream)),
          "fbspca_radial_eigenfunctions")
    return f


def fbspca_backproject(plan: Plan, c: torch.Tensor, mean, evecs, out=None, stream=None) -> torch.Tensor:
    """NEXT-1: a_k = U_k c_k (+ mean at k = 0), coefficient layout in and out."""
    n = c.shape[1]
    if out is None:
        out = torch.empty_like(c)
    check(lib().fbspca_backproject(ctypes.c_void_p(plan.handle), _ptr(c), n, _ptr(mean), _ptr(evecs), _ptr(out),
                                   _stream_ptr(stream)), "fbspca_backproject")
    return out


def fbspca_synthesize(plan: Plan, coeffs: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    """NEXT-1: n x L x L images from FB coefficients (Eq. (IFT_FB), reading Q2), zero outside r <= R."""
    n = coeffs.shape[1]
    if out is None:
        dt = torch.float32 if plan.dtype == F32 else torch.float64
        out = torch.empty((n, plan.L, plan.L), dtype=dt, device=coeffs.device)
    check(lib().fbspca_synthesize(ctypes.c_void_p(plan.handle), _ptr(coeffs), n, _ptr(out), _stream_ptr(stream)),
          "fbspca_synthesize")
    return out


def fbspca_estimate_params(images: torch.Tensor, fraction: float = 0.999):
    """NEXT-2: (sigma2, R, c) of an n x L x L stack on its CUDA device (see include/fbspca.h)."""
    n, L, L2 = images.shape
    assert L == L2 and images.is_cuda and images.is_contiguous()
    dt = F32 if images.dtype == torch.float32 else F64
    s2, R, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    check(lib().fbspca_estimate_params(L, dt, images.device.index, _ptr(images), n, float(fraction), ctypes.byref(s2),
                                       ctypes.byref(R), ctypes.byref(c)), "fbspca_estimate_params")
    return s2.value, R.value, c.value


def fbspca_project(plan: Plan, coeffs: torch.Tensor, mean, evals, evecs, sigma2: float = 0.0, mode: int = 0,
                   n_total: int | None = None, out=None, stream=None) -> torch.Tensor:
    n = coeffs.shape[1]
    n_total = n if n_total is None else n_total
    if out is None:
        out = torch.empty_like(coeffs)
    check(lib().fbspca_project(ctypes.c_void_p(plan.handle), _ptr(coeffs), n, _ptr(mean), _ptr(evals), _ptr(evecs),
                               float(sigma2), int(mode), int(n_total), _ptr(out), _stream_ptr(stream)),
          "fbspca_project")
    return out


def fbspca_step(plan: Plan, images: torch.Tensor, coeffs: torch.Tensor, blocks: torch.Tensor, mean: torch.Tensor,
                n_total: int | None = None, comm: int | None = None, use_graph: bool = False, stream=None):
    """expand + covariance (+ all-reduce) + finalise as one call; use_graph replays a captured CUDA graph."""
    n = images.shape[0]
    n_total = n if n_total is None else n_total
    _check_coeffs(plan, coeffs, n)
    _on_plan_device(plan, images, coeffs, blocks, mean)
    check(lib().fbspca_step(ctypes.c_void_p(plan.handle), _ptr(images), n, n_total, ctypes.c_void_p(comm or 0),
                            _ptr(coeffs), _ptr(blocks), _ptr(mean), int(bool(use_graph)), _stream_ptr(stream)),
          "fbspca_step")
    return blocks, mean


def fbspca_comm_wait(comm: int, stream=None, timeout_s: float = 0.0):
    check(lib().fbspca_comm_wait(ctypes.c_void_p(comm), _stream_ptr(stream), float(timeout_s)), "fbspca_comm_wait")


def fbspca_nccl_unique_id() -> bytes:
    buf = (ctypes.c_char * 128)()
    check(lib().fbspca_nccl_unique_id(buf), "fbspca_nccl_unique_id")
    return bytes(buf)


def fbspca_comm_init(unique_id: bytes, nranks: int, rank: int) -> int:
    buf = (ctypes.c_char * 128).from_buffer_copy(unique_id)
    comm = ctypes.c_void_p()
    check(lib().fbspca_comm_init(buf, nranks, rank, ctypes.byref(comm)), "fbspca_comm_init")
    return comm.value


def fbspca_comm_destroy(comm: int):
    check(lib().fbspca_comm_destroy(ctypes.c_void_p(comm)), "fbspca_comm_destroy")


def fbspca_set_timing(plan: Plan, enabled: bool = True):
    check(lib().fbspca_set_timing(ctypes.c_void_p(plan.handle), int(enabled)), "fbspca_set_timing")


def fbspca_get_timing(plan: Plan) -> dict:
    cnt = ctypes.c_int()
    names = ctypes.POINTER(ctypes.c_char_p)()
    ms = ctypes.POINTER(ctypes.c_float)()
    check(lib().fbspca_get_timing(ctypes.c_void_p(plan.handle), ctypes.byref(cnt), ctypes.byref(names),
                                  ctypes.byref(ms)), "fbspca_get_timing")
    n = cnt.value
    return {names[i].decode(): (float(ms[i]), int(ms[n + i])) for i in range(n)}


# ---------------------------------------------------------------- host-side layout helpers (no compute)
def split_blocks(plan: Plan, coeffs: torch.Tensor) -> list:
    """Coefficient layout -> list over k of (p_k, n) views."""
    return [coeffs[int(plan.coef_off[k]):int(plan.coef_off[k + 1])] for k in range(plan.k_max + 1)]


def unpack_blocks(plan: Plan, packed: np.ndarray) -> list:
    """Packed upper triangles (fp64) -> list of symmetric (p_k, p_k) numpy arrays."""
    out = []
    for k in range(plan.k_max + 1):
        pk = int(plan.p[k])
        seg = packed[int(plan.blk_off[k]):int(plan.blk_off[k + 1])]
        C = np.zeros((pk, pk))
        iu = np.triu_indices(pk)
        C[iu] = seg
        C = C + np.triu(C, 1).T
        out.append(C)
    return out


def split_eig(plan: Plan, evals: np.ndarray, evecs: np.ndarray):
    lam, U = [], []
    for k in range(plan.k_max + 1):
        pk = int(plan.p[k])
        lam.append(evals[int(plan.coef_off[k]):int(plan.coef_off[k + 1])])
        U.append(evecs[int(plan.evec_off[k]):int(plan.evec_off[k + 1])].reshape(pk, pk))
    return lam, U


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [s, e) of n images for rank r of world."""
    base, rem = divmod(n, world)
    s = rank * base + min(rank, rem)
    return s, s + base + (1 if rank < rem else 0)
