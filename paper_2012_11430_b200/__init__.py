"""paper_2012_11430_b200 — B200 (sm_100a) hot path of the parallel multivariate matrix-pencil
Prony method (arXiv 2012.11430): S_l = U* T_l V Sigma^-1 with T_l generated implicitly from
the sample grid, the Vandermonde A = [z_j^k] and the least-squares products A conj(A)^T,
A conj(f), behind a C ABI (include/prony.h, libprony.so) with this thin ctypes binding.

There is no CPU fallback: importing works anywhere, every compute call needs the built
libprony.so and a CUDA device and raises otherwise.
"""
from .binding import (  # noqa: F401
    EXPORTS, ExecInfo, make_exec_info, MAX_D, MAX_M, PRONY_ERR_CUDA, PRONY_ERR_INVALID, PRONY_ERR_RANGE, PRONY_ERR_SINGULAR,
    PRONY_ERR_UNIMPLEMENTED, PRONY_ERR_WORKSPACE, PRONY_OK, UNITS_L_MAJOR, UNITS_ROW_MAJOR, WS_LS,
    WS_PENCIL_HOST, WS_PROJECT, PronyError, alloc_workspace, build_pencil, device_info, lib, ls_solve,
    pencil_host, project, status_string, toeplitz_apply, vandermonde_ls, workspace_size,
    WS_APPLY, WS_DIAG, WS_PROJECT_MU, project_mu, diagonalize, PRONY_ERR_RANK, PRONY_ERR_NOT_CONVERGED, WS_BUILD,
    WS_LANCZOS, lanczos_svd, pencil_host_part, UNITS_SHARED, HostContext, pencil, WS_PENCIL,
)
from . import sharding  # noqa: F401

__all__ = ["project", "vandermonde_ls", "ls_solve", "pencil", "pencil_host", "pencil_host_part", "HostContext", "build_pencil", "lanczos_svd", "diagonalize",
           "project_mu", "toeplitz_apply", "workspace_size",
           "alloc_workspace", "device_info", "status_string", "PronyError", "sharding"]
