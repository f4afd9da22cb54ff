"""B200-native AIM-accelerated EFIE matvec + GMRES (arXiv 1712.02443, §V).

Thin Python binding over the C ABI in include/aim.h (libaim_b200.so, built
in-tree for sm_100a).  PyTorch is used for device memory and streams only;
every step of the operator runs in the library's CUDA kernels.
"""
from .api import AimPlan, AimSlabPlan, AimError, launch_count, slab_partition, nccl_unique_id, EXPORT  # noqa: F401
