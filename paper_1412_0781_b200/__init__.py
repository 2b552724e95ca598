"""B200-native Fast Fourier-Bessel steerable PCA (arXiv 1412.0781): C-ABI library + thin binding."""
from .fbspca import (  # noqa: F401
    F32, F64, Plan, fbspca_comm_destroy, fbspca_comm_init, fbspca_covariance, fbspca_covariance_finalize,
    fbspca_covariance_partial, fbspca_covariance_accumulate, fbspca_allreduce_partial, fbspca_eig, fbspca_svd, fbspca_expand, fbspca_get_timing, fbspca_nccl_unique_id, fbspca_plan, fbspca_plan_rings,
    fbspca_backproject, fbspca_estimate_params, fbspca_project, fbspca_radial_eigenfunctions, fbspca_synthesize, fbspca_set_timing, fbspca_step, fbspca_comm_wait, shard_range, split_blocks, split_eig,
    unpack_blocks,
)
from ._lib import FbspcaError, LIB_PATH  # noqa: F401
