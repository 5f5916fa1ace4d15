"""B200-native hot path of p2TDVP (Secular et al., arXiv:1912.06127).

The compute lives in libtdvp.so (CUDA, sm_100a; C-ABI in include/tdvp.h);
this package is the thin ctypes binding.  No CPU fallback exists.
"""
from .tdvp import (  # noqa: F401
    Tdvp, TdvpError, lib, plan, partition, balanced_partition, nccl_unique_id, apply_heff2, apply_heff1, env_left, env_right,
    expm_lanczos_dense, svd_split, zgemm, LIB_PATH,
)
