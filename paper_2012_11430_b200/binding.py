"""Thin ctypes binding of libprony.so (include/prony.h). Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels. Tensors are torch tensors
on a CUDA device (torch supplies device memory and the current stream); there is no CPU
fallback — without the built library or a CUDA device every call raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PRONY_LIB") or os.path.join(_HERE, "libprony.so")  # PRONY_LIB: A/B builds

PRONY_OK = 0
PRONY_ERR_INVALID = 1
PRONY_ERR_RANGE = 2
PRONY_ERR_SINGULAR = 3
PRONY_ERR_RANK = 4
PRONY_ERR_NOT_CONVERGED = 5
PRONY_ERR_CUDA = 6
PRONY_ERR_UNIMPLEMENTED = 7
PRONY_ERR_WORKSPACE = 8

WS_PROJECT, WS_LS, WS_PENCIL_HOST, WS_BUILD, WS_APPLY, WS_DIAG, WS_PROJECT_MU, WS_LANCZOS, WS_PENCIL = range(9)
UNITS_L_MAJOR, UNITS_ROW_MAJOR, UNITS_SHARED = 0, 1, 2
MAX_D, MAX_M = 8, 128

# every symbol include/prony.h declares (checked by tests/test_abi.py)
EXPORTS = ("prony_abi_version", "prony_status_string", "prony_device_info", "prony_workspace_size",
           "prony_project", "prony_project_ex", "prony_vandermonde_ls", "prony_vandermonde_ls_ex", "prony_ls_solve",
           "prony_toeplitz_apply", "prony_pencil_host", "prony_build_pencil", "prony_diagonalize",
           "prony_project_mu", "prony_lanczos_svd", "prony_pencil_host_part", "prony_host_context_create",
           "prony_host_context_destroy", "prony_pencil_host_ctx", "prony_pencil_host_part_ctx", "prony_pencil")


class ExecInfo(ctypes.Structure):
    """prony_exec_info (include/prony.h): events around the dominant kernel + launch record."""
    _fields_ = [("ev_main_begin", ctypes.c_void_p), ("ev_main_end", ctypes.c_void_p), ("launches", ctypes.c_int32),
                ("main_grid", ctypes.c_int32 * 3), ("main_block", ctypes.c_int32), ("split_k", ctypes.c_int32),
                ("main_flops", ctypes.c_double), ("ev_wait_u", ctypes.c_void_p)]


def make_exec_info(ev_begin=None, ev_end=None, ev_wait_u=None) -> ExecInfo:
    """ev_*: torch.cuda.Event already created (recorded once). ev_wait_u (prony_project_ex): an event the call's
    stream waits on before the reduction that first reads U."""
    info = ExecInfo()
    info.ev_main_begin = ev_begin.cuda_event if ev_begin is not None else None
    info.ev_main_end = ev_end.cuda_event if ev_end is not None else None
    info.ev_wait_u = ev_wait_u.cuda_event if ev_wait_u is not None else None
    return info


class PronyError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        super().__init__(f"{what}: {status_string(code)} (status {code})")


_lib = None


def lib() -> ctypes.CDLL:
    """Load libprony.so (built in-tree by __graft_entry__.build()). Raises if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
        L.prony_abi_version.restype = i32
        L.prony_status_string.restype = ctypes.c_char_p
        L.prony_status_string.argtypes = [i32]
        L.prony_device_info.argtypes = [vp, vp, vp]
        L.prony_workspace_size.argtypes = [i32, i32, i32, i32, ctypes.POINTER(sz)]
        L.prony_project.argtypes = [i32, i32, i32, vp, vp, vp, vp, i64, i64, i32, vp, vp, sz, vp, vp]
        L.prony_vandermonde_ls.argtypes = [i32, i32, i32, vp, vp, i64, i64, vp, vp, vp, vp, vp, vp, sz, vp, vp]
        L.prony_project_ex.argtypes = L.prony_project.argtypes + [vp]
        L.prony_vandermonde_ls_ex.argtypes = L.prony_vandermonde_ls.argtypes + [vp]
        L.prony_ls_solve.argtypes = [i32, i32, vp, vp, vp, vp, vp, vp, sz, vp, vp]
        L.prony_toeplitz_apply.argtypes = [i32, i32, vp, i32, i32, vp, i32, i32, vp, i32, vp, sz, vp]
        L.prony_pencil_host.argtypes = [i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp, vp]
        L.prony_build_pencil.argtypes = [i32, i32, i32, vp, ctypes.c_uint64, ctypes.c_double, i32, vp, vp, vp, vp, vp,
                                         vp, vp, sz, vp, vp]
        L.prony_diagonalize.argtypes = [i32, i32, vp, vp, vp, vp, vp, vp, sz, vp, vp]
        L.prony_project_mu.argtypes = [i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp, vp]
        L.prony_pencil_host_part.argtypes = [i32, i32, i32, vp, vp, vp, vp, vp, i64, i64, i64, i64, vp, vp, vp, vp, sz,
                                             vp, vp]
        L.prony_lanczos_svd.argtypes = [i32, i32, vp, i32, ctypes.c_double, ctypes.c_uint64, i32, vp, vp, vp, vp, vp,
                                        vp, sz, vp]
        L.prony_host_context_create.argtypes = [ctypes.POINTER(vp)]
        L.prony_host_context_destroy.argtypes = [vp]
        L.prony_pencil_host_ctx.argtypes = [vp] + L.prony_pencil_host.argtypes
        L.prony_pencil_host_part_ctx.argtypes = [vp] + L.prony_pencil_host_part.argtypes
        L.prony_pencil.argtypes = [vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp, vp, vp, vp]
        for f in ("prony_device_info", "prony_workspace_size", "prony_project", "prony_vandermonde_ls", "prony_ls_solve",
                  "prony_project_ex", "prony_vandermonde_ls_ex", "prony_toeplitz_apply", "prony_diagonalize",
                  "prony_project_mu", "prony_pencil_host_part", "prony_lanczos_svd", "prony_host_context_create",
                  "prony_host_context_destroy", "prony_pencil_host_ctx", "prony_pencil_host_part_ctx",
                  "prony_pencil_host", "prony_build_pencil", "prony_pencil"):
            getattr(L, f).restype = i32
        _lib = L
    return _lib


def status_string(code: int) -> str:
    return lib().prony_status_string(int(code)).decode()


def _check(rc: int, what: str) -> None:
    if rc != PRONY_OK:
        raise PronyError(rc, what)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dev_tensor(t, dtype, name):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA torch tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def device_info():
    sms, a, b = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _check(lib().prony_device_info(ctypes.byref(sms), ctypes.byref(a), ctypes.byref(b)), "prony_device_info")
    return sms.value, (a.value, b.value)


def workspace_size(kind: int, d: int, n: int, m: int) -> int:
    out = ctypes.c_size_t()
    _check(lib().prony_workspace_size(kind, d, n, m, ctypes.byref(out)), "prony_workspace_size")
    return out.value


def alloc_workspace(kind: int, d: int, n: int, m: int, device=None) -> torch.Tensor:
    nbytes = workspace_size(kind, d, n, m)
    return torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device or "cuda")


def unit_count(d: int, n: int, unit_order: int) -> int:
    """Size of the unit space of prony_project: d N (L_MAJOR, ROW_MAJOR) or (n+2)^d (SHARED)."""
    return (n + 2) ** d if unit_order == UNITS_SHARED else d * (n + 1) ** d


def project(grid, U, V, sigma, d: int, n: int, m: int, unit_begin: int = 0, unit_end: int | None = None,
            unit_order: int = UNITS_SHARED, out=None, workspace=None, dev_status=None, stream=None, info=None):
    """S_l = U* T_l V Sigma^-1 over units [unit_begin, unit_end) -> (d, m, m) complex128.
    The default order SHARED computes all d pencils from one extended product (F8)."""
    _dev_tensor(grid, torch.complex128, "grid")
    _dev_tensor(U, torch.complex128, "U")
    _dev_tensor(V, torch.complex128, "V")
    _dev_tensor(sigma, torch.float64, "sigma")
    if unit_end is None:
        unit_end = unit_count(d, n, unit_order)
    if out is None:
        out = torch.empty((d, m, m), dtype=torch.complex128, device=grid.device)
    _dev_tensor(out, torch.complex128, "out")
    if workspace is None:
        workspace = alloc_workspace(WS_PROJECT, d, n, m, grid.device)
    rc = lib().prony_project_ex(d, n, m, _ptr(grid), _ptr(U), _ptr(V), _ptr(sigma), int(unit_begin),
                                int(unit_end), int(unit_order), _ptr(out), _ptr(workspace), workspace.numel(),
                                _ptr(dev_status), _stream(stream), None if info is None else ctypes.byref(info))
    _check(rc, "prony_project")
    return out


def vandermonde_ls(z, grid, d: int, n: int, m: int, col_begin: int = 0, col_end: int | None = None,
                   want_A: bool = False, want_solution: bool = True, out=None, workspace=None, dev_status=None,
                   stream=None, info=None):
    """A = [z_j^k], G = A conj(A)^T, b = A conj(f) (+ c, t over the full range) -> dict of tensors."""
    N = (n + 1) ** d
    _dev_tensor(z, torch.complex128, "z")
    _dev_tensor(grid, torch.complex128, "grid")
    if col_end is None:
        col_end = N
    dev = grid.device
    if out is None:
        out = {}
    G = out.get("G")
    if G is None:
        G = torch.empty((m, m), dtype=torch.complex128, device=dev)
    b = out.get("b")
    if b is None:
        b = torch.empty(m, dtype=torch.complex128, device=dev)
    A = out.get("A")
    if want_A and A is None:
        A = torch.empty((m, col_end - col_begin), dtype=torch.complex128, device=dev)
    full = col_begin == 0 and col_end == N
    c = t = None
    if full and want_solution:
        c = out.get("c")
        if c is None:
            c = torch.empty(m, dtype=torch.complex128, device=dev)
        t = out.get("t")
        if t is None:
            t = torch.empty((m, d), dtype=torch.float64, device=dev)
    if workspace is None:
        workspace = alloc_workspace(WS_LS, d, n, m, dev)
    rc = lib().prony_vandermonde_ls_ex(d, n, m, _ptr(z), _ptr(grid), int(col_begin), int(col_end),
                                       _ptr(A if want_A else None), _ptr(G), _ptr(b), _ptr(c), _ptr(t),
                                       _ptr(workspace), workspace.numel(), _ptr(dev_status), _stream(stream),
                                       None if info is None else ctypes.byref(info))
    _check(rc, "prony_vandermonde_ls")
    res = {"G": G, "b": b}
    if want_A:
        res["A"] = A
    if c is not None:
        res["c"] = c
        res["t"] = t
    return res


def ls_solve(G, b, z, d: int, m: int, want_t: bool = True, workspace=None, dev_status=None, stream=None, out=None):
    """c = conj(G^-1 b) (Cholesky) and t = (-arg z/2pi) mod 1 for already-reduced G, b.
    out: optional dict with preallocated "c" (m,) complex128 / "t" (m, d) float64 device tensors."""
    _dev_tensor(G, torch.complex128, "G")
    _dev_tensor(b, torch.complex128, "b")
    _dev_tensor(z, torch.complex128, "z")
    dev = G.device
    out = out or {}
    c = out.get("c")
    if c is None:
        c = torch.empty(m, dtype=torch.complex128, device=dev)
    _dev_tensor(c, torch.complex128, "c")
    t = out.get("t") if want_t else None
    if want_t and t is None:
        t = torch.empty((m, d), dtype=torch.float64, device=dev)
    if workspace is None:
        workspace = torch.empty(m * m * 16 + m * 16 + 512, dtype=torch.uint8, device=dev)
    rc = lib().prony_ls_solve(d, m, _ptr(G), _ptr(b), _ptr(z), _ptr(c), _ptr(t), _ptr(workspace), workspace.numel(),
                              _ptr(dev_status), _stream(stream))
    _check(rc, "prony_ls_solve")
    return c, t


def project_mu(grid, U, V, sigma, mu, d: int, n: int, m: int, out=None, workspace=None, stream=None):
    """C_mu = U* B_mu V Sigma^-1, B_mu = sum_l mu_l T_l: one projection on the combined grid."""
    for t_, nm in ((grid, "grid"), (U, "U"), (V, "V"), (mu, "mu")):
        _dev_tensor(t_, torch.complex128, nm)
    _dev_tensor(sigma, torch.float64, "sigma")
    if out is None:
        out = torch.empty((m, m), dtype=torch.complex128, device=grid.device)
    if workspace is None:
        workspace = alloc_workspace(WS_PROJECT_MU, d, n, m, grid.device)
    rc = lib().prony_project_mu(d, n, m, _ptr(grid), _ptr(U), _ptr(V), _ptr(sigma), _ptr(mu), _ptr(out),
                                _ptr(workspace), workspace.numel(), None, _stream(stream))
    _check(rc, "prony_project_mu")
    return out


def toeplitz_apply(grid, X, d: int, n: int, ell: int = 0, conj: bool = False, out=None, workspace=None,
                   stream=None):
    """Y = T_l X (l = 1..d), T X (l = 0) or T^H X (l = 0, conj) with the implicit gather."""
    _dev_tensor(grid, torch.complex128, "grid")
    if not (isinstance(X, torch.Tensor) and X.is_cuda and X.dtype == torch.complex128 and X.dim() == 2
            and X.stride(1) == 1):
        raise TypeError("X must be a CUDA complex128 matrix with unit column stride")
    N, r = X.shape
    if out is None:
        out = torch.empty((N, r), dtype=torch.complex128, device=X.device)
    if workspace is None:
        workspace = alloc_workspace(WS_APPLY, d, n, 1, X.device)
    rc = lib().prony_toeplitz_apply(d, n, _ptr(grid), int(ell), int(bool(conj)), _ptr(X), X.stride(0), r, _ptr(out),
                                    out.stride(0), _ptr(workspace), workspace.numel(), _stream(stream))
    _check(rc, "prony_toeplitz_apply")
    return out


def pencil(grid, U, V, sigma, z, d: int, n: int, m: int, out: dict, workspace, context=None, dev_status=None,
           stream=None, info_p=None, info_l=None):
    """One full pencil on DEVICE buffers in one C call (prony_pencil): S_1..S_d on `stream`, the LS products,
    c and t concurrently on the context's side stream. out: preallocated device tensors "S" (d,m,m), "G" (m,m),
    "b" (m,), "c" (m,), "t" (m,d); workspace >= WS_PENCIL. Asynchronous; returns `out`."""
    for name, x, shape in (("S", out["S"], (d, m, m)), ("G", out["G"], (m, m)), ("b", out["b"], (m,)),
                           ("c", out["c"], (m,))):
        _dev_tensor(x, torch.complex128, name)
        if tuple(x.shape) != shape:
            raise ValueError(f"out[{name!r}] must have shape {shape}, got {tuple(x.shape)}")
    _dev_tensor(out["t"], torch.float64, "t")
    if tuple(out["t"].shape) != (m, d):
        raise ValueError(f"out['t'] must have shape {(m, d)}")
    for name, x in (("grid", grid), ("U", U), ("V", V), ("z", z)):
        _dev_tensor(x, torch.complex128, name)
    _dev_tensor(sigma, torch.float64, "sigma")
    rc = lib().prony_pencil(None if context is None else context.handle, d, n, m, _ptr(grid), _ptr(U), _ptr(V),
                            _ptr(sigma), _ptr(z), _ptr(out["S"]), _ptr(out["G"]), _ptr(out["b"]), _ptr(out["c"]),
                            _ptr(out["t"]), _ptr(workspace), workspace.numel(), _ptr(dev_status), _stream(stream),
                            None if info_p is None else ctypes.byref(info_p),
                            None if info_l is None else ctypes.byref(info_l))
    _check(rc, "prony_pencil")
    return out


class HostContext:
    """prony_host_context: the side streams / events of the host-input pencil, created once on the current
    device and reused by pencil_host / pencil_host_part calls that pass it (destroyed with the object)."""

    def __init__(self):
        h = ctypes.c_void_p()
        _check(lib().prony_host_context_create(ctypes.byref(h)), "prony_host_context_create")
        self.handle = h

    def close(self):
        if self.handle is not None and self.handle.value:
            _check(lib().prony_host_context_destroy(self.handle), "prony_host_context_destroy")
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pencil_host(grid, U, V, sigma, z, d: int, n: int, m: int, workspace=None, outputs=None, stream=None,
                context: HostContext | None = None):
    """Full pencil from HOST (numpy or pinned CPU torch) buffers: H2D copies, prony_project over
    [0, dN), prony_vandermonde_ls over [0, N), D2H copies, stream sync. Returns dict of host arrays.
    context: a HostContext whose streams / events the call reuses (None: created per call)."""
    import numpy as np

    def host_ptr(a):
        if isinstance(a, torch.Tensor):
            assert not a.is_cuda and a.is_contiguous()
            return ctypes.c_void_p(a.data_ptr())
        return a.ctypes.data_as(ctypes.c_void_p)

    if outputs is None:
        outputs = {
            "S": np.empty((d, m, m), np.complex128), "G": np.empty((m, m), np.complex128),
            "b": np.empty(m, np.complex128), "c": np.empty(m, np.complex128), "t": np.empty((m, d), np.float64),
        }
    if workspace is None:
        workspace = alloc_workspace(WS_PENCIL_HOST, d, n, m)
    st = ctypes.c_int32(0)
    rc = lib().prony_pencil_host_ctx(None if context is None else context.handle, d, n, m, host_ptr(grid), host_ptr(U),
                                     host_ptr(V), host_ptr(sigma), host_ptr(z),
                                 host_ptr(outputs["S"]), host_ptr(outputs["G"]), host_ptr(outputs["b"]),
                                 host_ptr(outputs["c"]), host_ptr(outputs["t"]), _ptr(workspace), workspace.numel(),
                                 ctypes.byref(st), _stream(stream))
    _check(rc, "prony_pencil_host")
    outputs["status"] = st.value
    return outputs


def pencil_host_part(grid, U, V, sigma, z, d: int, n: int, m: int, unit_begin: int, unit_end: int, col_begin: int,
                     col_end: int, S, G, b, workspace=None, dev_status=None, stream=None,
                     context: HostContext | None = None):
    """One rank's partial pencil from HOST inputs (pinned CPU torch tensors for overlap): SHARED units
    [unit_begin, unit_end), LS columns [col_begin, col_end); partial S, G, b land in the given DEVICE
    tensors. Asynchronous on `stream`."""
    def host_ptr(a):
        if not (isinstance(a, torch.Tensor) and not a.is_cuda and a.is_contiguous()):
            raise TypeError("host inputs must be contiguous CPU tensors")
        return ctypes.c_void_p(a.data_ptr())

    for name, x in (("S", S), ("G", G), ("b", b)):
        _dev_tensor(x, torch.complex128, name)
    if workspace is None:
        workspace = alloc_workspace(WS_PENCIL_HOST, d, n, m, S.device)
    rc = lib().prony_pencil_host_part_ctx(None if context is None else context.handle, d, n, m, host_ptr(grid),
                                          host_ptr(U), host_ptr(V), host_ptr(sigma), host_ptr(z),
                                      int(unit_begin), int(unit_end), int(col_begin), int(col_end), _ptr(S), _ptr(G),
                                      _ptr(b), _ptr(workspace), workspace.numel(), _ptr(dev_status), _stream(stream))
    _check(rc, "prony_pencil_host_part")
    return S, G, b


def build_pencil(grid, d: int, n: int, m: int, seed: int = 0, tol: float | None = None, max_iter: int = 4,
                 workspace=None, stream=None, check: bool = True):
    """Algorithm 1 lines 1-3 on the device: block power reduced SVD of T (Alg. 3) and
    S_l = U* T_l V Sigma^-1. tol defaults to N eps_M. Synchronous. Returns a dict with
    S (d,m,m), U, V (N,m), sigma (m,), rank, resid, status (PRONY_OK / _RANK / _NOT_CONVERGED)."""
    _dev_tensor(grid, torch.complex128, "grid")
    N = (n + 1) ** d
    if tol is None:
        tol = N * 2.220446049250313e-16
    dev = grid.device
    S = torch.empty((d, m, m), dtype=torch.complex128, device=dev)
    U = torch.empty((N, m), dtype=torch.complex128, device=dev)
    V = torch.empty((N, m), dtype=torch.complex128, device=dev)
    s = torch.empty(m, dtype=torch.float64, device=dev)
    rank = ctypes.c_int32(0)
    resid = ctypes.c_double(-1.0)
    if workspace is None:
        workspace = alloc_workspace(WS_BUILD, d, n, m, dev)
    rc = lib().prony_build_pencil(d, n, m, _ptr(grid), int(seed), float(tol), int(max_iter), _ptr(S), _ptr(U), _ptr(V),
                                  _ptr(s), ctypes.byref(rank), ctypes.byref(resid), _ptr(workspace), workspace.numel(),
                                  None, _stream(stream))
    if check and rc not in (PRONY_OK, PRONY_ERR_NOT_CONVERGED, PRONY_ERR_RANK):
        _check(rc, "prony_build_pencil")
    return {"S": S, "U": U, "V": V, "sigma": s, "rank": rank.value, "resid": resid.value, "status": rc}


def lanczos_svd(grid, d: int, n: int, max_rank: int, tol: float | None = None, seed: int = 0, ldo: int | None = None,
                workspace=None, stream=None, check: bool = True):
    """Rank-revealing reduced SVD of T by Lanczos bidiagonalization with full reorthogonalization
    (Alg. 2), m unknown. tol defaults to N eps_M (the noise-free tolerance of P:172/P:581).
    Synchronous. Returns a dict with U, V (N, ldo), sigma (ldo,) [first min(rank, ldo) valid], rank,
    steps, status (PRONY_OK / PRONY_ERR_NOT_CONVERGED when max_rank steps ran out)."""
    _dev_tensor(grid, torch.complex128, "grid")
    N = (n + 1) ** d
    if tol is None:
        tol = N * 2.220446049250313e-16
    if ldo is None:
        ldo = max_rank
    dev = grid.device
    U = torch.zeros((N, ldo), dtype=torch.complex128, device=dev)
    V = torch.zeros((N, ldo), dtype=torch.complex128, device=dev)
    s = torch.zeros(ldo, dtype=torch.float64, device=dev)
    rank = ctypes.c_int32(0)
    steps = ctypes.c_int32(0)
    if workspace is None:
        workspace = alloc_workspace(WS_LANCZOS, d, n, max_rank, dev)
    rc = lib().prony_lanczos_svd(d, n, _ptr(grid), int(max_rank), float(tol), int(seed), int(ldo), _ptr(U), _ptr(V),
                                 _ptr(s), ctypes.byref(rank), ctypes.byref(steps), _ptr(workspace), workspace.numel(),
                                 _stream(stream))
    if check and rc not in (PRONY_OK, PRONY_ERR_NOT_CONVERGED):
        _check(rc, "prony_lanczos_svd")
    return {"U": U, "V": V, "sigma": s, "rank": rank.value, "steps": steps.value, "status": rc}


def diagonalize(S, mu, d: int, m: int, workspace=None, dev_status=None, stream=None):
    """Algorithm 1 lines 4-6 on the device: C_mu = sum mu_l S_l, W = eigenvectors, z = diag(W^-1 S_l W),
    t = (-arg z / 2 pi) mod 1. Returns (z (m,d), t (m,d), W (m,m))."""
    _dev_tensor(S, torch.complex128, "S")
    _dev_tensor(mu, torch.complex128, "mu")
    dev = S.device
    z = torch.empty((m, d), dtype=torch.complex128, device=dev)
    t = torch.empty((m, d), dtype=torch.float64, device=dev)
    W = torch.empty((m, m), dtype=torch.complex128, device=dev)
    if workspace is None:
        workspace = alloc_workspace(WS_DIAG, d, m, m, dev)
    rc = lib().prony_diagonalize(d, m, _ptr(S), _ptr(mu), _ptr(z), _ptr(t), _ptr(W), _ptr(workspace),
                                 workspace.numel(), _ptr(dev_status), _stream(stream))
    _check(rc, "prony_diagonalize")
    return z, t, W
