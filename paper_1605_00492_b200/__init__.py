"""B200-native tensor-product multigrid for the thin-shell pressure Helmholtz
problem of arXiv:1605.00492 (Mitchell & Mueller).

The compute path is the CUDA library ``libhmg.so`` (sm_100a) behind the C-ABI
of ``include/hmg.h``; this package is a thin ctypes binding (argument
marshalling only).  There is no CPU fallback: importing works without a GPU,
but every call that computes needs the CUDA library and a device.
"""
from .binding import (HmgError, Hierarchy, MGParams, STATUS, band_apply, band_factor, band_solve, lib_path,
                      load_library, nccl_unique_id, p_prolong_add, p_restrict, partition_plan)

__all__ = ["HmgError", "Hierarchy", "MGParams", "STATUS", "band_apply", "band_factor", "band_solve", "lib_path",
           "load_library", "nccl_unique_id", "p_prolong_add", "p_restrict", "partition_plan"]
