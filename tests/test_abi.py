"""The C ABI library builds, loads on a CPU-only box and exports every symbol include/prony.h
declares; argument validation happens synchronously before any CUDA call."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pb():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2012_11430_b200 as pb
    return pb


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "prony.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(prony_\w+)\s*\(", src, flags=re.M)))


def test_header_symbols_exported(pb):
    syms = declared_symbols()
    assert len(syms) >= 8
    L = ctypes.CDLL(pb.binding.LIB_PATH)
    for s in syms:
        assert hasattr(L, s), f"libprony.so does not export {s}"
    assert set(syms) == set(pb.EXPORTS)


def test_exported_symbols_are_c_abi(pb):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", pb.binding.LIB_PATH], capture_output=True, text=True).stdout
    names = {l.split()[-1] for l in out.splitlines() if " T " in l}
    for s in declared_symbols():
        assert s in names   # unmangled => extern "C"


def test_abi_version_and_status_strings(pb):
    hdr = open(os.path.join(ROOT, "include", "prony.h")).read()
    assert pb.lib().prony_abi_version() == int(re.search(r"#define PRONY_ABI_VERSION (\d+)", hdr).group(1)) == 6
    for code in range(0, 9):
        assert len(pb.status_string(code)) > 0
    assert pb.status_string(12345) == "unknown status"


def test_validation_before_any_cuda_call(pb):
    L = pb.lib()
    null = None
    # d = 0 -> INVALID; m > 128 -> RANGE; (2n+2)^d >= 2^31 -> RANGE; null pointers -> INVALID
    assert L.prony_project(0, 4, 2, null, null, null, null, 0, 1, 0, null, null, 0, null, null) == pb.PRONY_ERR_INVALID
    assert L.prony_project(2, 4, 129, null, null, null, null, 0, 1, 0, null, null, 0, null, null) == pb.PRONY_ERR_RANGE
    assert L.prony_project(4, 200, 3, null, null, null, null, 0, 1, 0, null, null, 0, null, null) == pb.PRONY_ERR_RANGE
    assert L.prony_project(2, 1, 5, null, null, null, null, 0, 1, 0, null, null, 0, null, null) == pb.PRONY_ERR_RANGE
    assert L.prony_project(2, 4, 3, null, null, null, null, 0, 1, 0, null, null, 0, null, null) == pb.PRONY_ERR_INVALID
    assert L.prony_vandermonde_ls(2, 4, 3, null, null, 0, 25, null, null, null, null, null, null, 0, null,
                                  null) == pb.PRONY_ERR_INVALID
    assert L.prony_ls_solve(0, 3, null, null, null, null, null, null, 0, null, null) == pb.PRONY_ERR_INVALID
    sz = ctypes.c_size_t()
    assert L.prony_workspace_size(0, 9, 4, 3, ctypes.byref(sz)) == pb.PRONY_ERR_INVALID
    assert L.prony_build_pencil(2, 4, 3, null, 0, 0.0, 1, null, null, null, null, null, null, null, 0, null,
                                null) == pb.PRONY_ERR_INVALID
    assert L.prony_diagonalize(0, 3, null, null, null, null, null, null, 0, null, null) == pb.PRONY_ERR_INVALID
    assert L.prony_toeplitz_apply(2, 4, null, 3, 0, null, 1, 1, null, 1, null, 0, null) == pb.PRONY_ERR_INVALID
    # lanczos: null grid -> INVALID; max_rank above the Jacobi limit or above N -> RANGE (pointers non-null)
    assert L.prony_lanczos_svd(2, 4, null, 5, 0.0, 0, 5, null, null, null, null, null, null, 0,
                               null) == pb.PRONY_ERR_INVALID
    buf = (ctypes.c_double * 64)()
    p = ctypes.c_void_p(ctypes.addressof(buf))
    r = ctypes.c_int32()
    assert L.prony_lanczos_svd(2, 4, p, 26, 0.0, 0, 5, p, p, p, ctypes.byref(r), None, p, 0,
                               null) == pb.PRONY_ERR_RANGE
    assert L.prony_lanczos_svd(2, 4, p, 5, 0.0, 0, 6, p, p, p, ctypes.byref(r), None, p, 0,
                               null) == pb.PRONY_ERR_INVALID
    assert L.prony_workspace_size(pb.WS_LANCZOS, 2, 20, 256, ctypes.byref(sz)) == pb.PRONY_ERR_RANGE
    # the diagonalization's workspace does not depend on n: a huge n is fine, m is still checked
    assert L.prony_workspace_size(pb.WS_DIAG, 8, 100000, 40, ctypes.byref(sz)) == pb.PRONY_OK and sz.value > 0
    assert L.prony_workspace_size(pb.WS_DIAG, 8, 1, 129, ctypes.byref(sz)) == pb.PRONY_ERR_RANGE
    # host context: null out-pointer / null context
    assert L.prony_host_context_create(None) == pb.PRONY_ERR_INVALID
    assert L.prony_host_context_destroy(None) == pb.PRONY_ERR_INVALID
    assert L.prony_pencil_host_ctx(None, 0, 4, 2, *([None] * 11), 0, None, None) == pb.PRONY_ERR_INVALID


def test_misaligned_pointer_rejected(pb):
    L = pb.lib()
    buf = (ctypes.c_double * 64)()
    base = ctypes.addressof(buf)
    p = ctypes.c_void_p(base + 8 if base % 16 == 0 else base)   # 8-byte aligned, not 16
    q = ctypes.c_void_p(base + 256 - base % 256 if False else base)
    rc = L.prony_project(2, 4, 3, p, p, p, p, 0, 1, 0, p, q, 0, None, None)
    assert rc == pb.PRONY_ERR_INVALID


def test_no_cpu_fallback_without_gpu(pb):
    """Every compute entry point refuses CPU tensors (there is no CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(TypeError):
        pb.project(torch.zeros(4, dtype=torch.complex128), None, None, None, 1, 1, 1)
