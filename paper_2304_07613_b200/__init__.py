"""B200-native grouped n:m hot path of STen (arXiv 2304.07613).

The product is the C-ABI library ``libsten.so`` (include/sten.h) with its
sm_100a kernels; ``sten`` is the thin ctypes binding and ``parallel`` the
torch.distributed partition of the SpMM.  Nothing here imports ``oracle/``.
"""
from .sten import (  # noqa: F401
    ALGO_AUTO, ALGO_MMA_SYNC, ALGO_SIMT, ALGO_TCGEN05, StenError, densify, launch_count, load,
    make_plan, sparse_linear_host, sparse_linear_host_workspace_size, sparsify_grouped_nm,
    spmm_grouped_nm, spmm_plan,
)
