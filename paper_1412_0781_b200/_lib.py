"""ctypes loader for libfbspca.so (the C ABI in include/fbspca.h).  No fallback: if the library is
missing or fails to load, every call raises."""
from __future__ import annotations

import ctypes
import glob
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# FBSPCA_LIB: load a variant build instead (A/B experiments, paper_1412_0781_b200/build.py --lib ... -D ...)
LIB_PATH = os.environ.get("FBSPCA_LIB") or os.path.join(_HERE, "lib", "libfbspca.so")

_lib = None

c_int, c_double, c_int64, c_void_p, c_char_p = ctypes.c_int, ctypes.c_double, ctypes.c_int64, ctypes.c_void_p, ctypes.c_char_p
P_int = ctypes.POINTER(ctypes.c_int)
P_int64 = ctypes.POINTER(ctypes.c_int64)
P_double = ctypes.POINTER(ctypes.c_double)

# name -> (restype, argtypes)
SIGNATURES = {
    "fbspca_plan": (c_int, [c_int, c_double, c_double, c_double, c_int, c_int, c_int64, ctypes.POINTER(c_void_p)]),
    "fbspca_plan_info": (c_int, [c_void_p, P_int, P_int, P_int, ctypes.POINTER(P_int), ctypes.POINTER(P_int64),
                                 ctypes.POINTER(P_int64), ctypes.POINTER(P_int64)]),
    "fbspca_plan_detail": (c_int, [c_void_p, P_int, P_int, P_double, P_int, P_int, ctypes.POINTER(P_double),
                                   ctypes.POINTER(P_double), ctypes.POINTER(P_double)]),
    "fbspca_plan_rings": (c_int, [c_void_p, c_void_p, c_void_p]),
    "fbspca_expand": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "fbspca_covariance": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "fbspca_covariance_partial": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "fbspca_covariance_finalize": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "fbspca_covariance_accumulate": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "fbspca_allreduce_partial": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "fbspca_eig": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "fbspca_svd": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "fbspca_radial_eigenfunctions": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "fbspca_backproject": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "fbspca_synthesize": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "fbspca_estimate_params": (c_int, [c_int, c_int, c_int, c_void_p, c_int64, c_double, P_double, P_double, P_double]),
    "fbspca_project": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_double, c_int, c_int64,
                               c_void_p, c_void_p]),
    "fbspca_nccl_unique_id": (c_int, [c_void_p]),
    "fbspca_comm_init": (c_int, [c_void_p, c_int, c_int, ctypes.POINTER(c_void_p)]),
    "fbspca_comm_destroy": (c_int, [c_void_p]),
    "fbspca_comm_wait": (c_int, [c_void_p, c_void_p, c_double]),
    "fbspca_step": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                            c_void_p]),
    "fbspca_set_timing": (c_int, [c_void_p, c_int]),
    "fbspca_get_timing": (c_int, [c_void_p, P_int, ctypes.POINTER(ctypes.POINTER(c_char_p)),
                                  ctypes.POINTER(ctypes.POINTER(ctypes.c_float))]),
    "fbspca_destroy": (None, [c_void_p]),
    "fbspca_last_error": (c_char_p, []),
    "fbspca_version": (c_char_p, []),
}


class FbspcaError(RuntimeError):
    pass


def _preload_nccl():
    """Make NCCL resolvable for the library's dlopen("libnccl.so.2"): prefer the torch-bundled one."""
    try:
        import nvidia.nccl  # noqa: F401
        for p in glob.glob(os.path.join(os.path.dirname(nvidia.nccl.__file__), "lib", "libnccl.so*")):
            ctypes.CDLL(p, mode=ctypes.RTLD_GLOBAL)
            return
    except Exception:
        pass


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FbspcaError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        _preload_nccl()
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int, what: str):
    if status != 0:
        msg = lib().fbspca_last_error().decode(errors="replace")
        names = {1: "ARG", 2: "CONFIG", 3: "CUDA", 4: "NCCL", 5: "NUMERIC"}
        raise FbspcaError(f"{what}: FBSPCA_ERR_{names.get(status, status)}: {msg}")
