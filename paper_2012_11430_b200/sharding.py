"""Multi-GPU sharding of the pencil.

S_l = sum_g U[R_g]^* T_l[R_g, :] V Sigma^-1 is linear in any partition of the rows k of T_l
and of l, and G = sum_g A[:, K_g] A[:, K_g]^H, b likewise over the columns k. So each rank
takes a contiguous, equal slice of the unit space (default: the SHARED order, rows k' of the
extended block T_E, each standing for row k' - e_l of every T_l; or [0, dN) l-major / row-major,
see prony_unit_order) and of the columns [0, N), computes partial S (Sigma^-1 already applied),
G and b with its own GPU, and ONE all_reduce(SUM) of the packed [S_1..S_d, G, b]
((d+1) m^2 + m complex128, 470 KB at d=2, m=100) over NCCL completes the pencil on every
rank; the m x m Cholesky solve for c then runs locally (prony_ls_solve).

This module is host logic only (ranges, packing, the collective); the arithmetic is in the
CUDA library. It is exercised on CPU with gloo (tests/test_sharding.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def split_range(total: int, parts: int, idx: int) -> tuple[int, int]:
    """Contiguous near-equal split of [0, total) into `parts`; slice `idx`."""
    return total * idx // parts, total * (idx + 1) // parts


UNITS_L_MAJOR, UNITS_ROW_MAJOR, UNITS_SHARED = 0, 1, 2


def unit_count(d: int, n: int, order: int) -> int:
    return (n + 2) ** d if order == UNITS_SHARED else d * (n + 1) ** d


def unit_range(d: int, n: int, world: int, rank: int, order: int = UNITS_SHARED) -> tuple[int, int]:
    return split_range(unit_count(d, n, order), world, rank)


def shared_u_rows(d: int, n: int, e0: int, e1: int) -> tuple[int, int]:
    """Rows [lo, hi) of U that the SHARED units [e0, e1) pair with (k = k' - e_l in I_n, any l): the
    range prony_pencil_host_part copies (mirrors its host-side computation)."""
    def krow(e, ell):
        c = []
        for _ in range(d):
            c.append(e % (n + 2))
            e //= n + 2
        c = c[::-1]
        c[ell] -= 1
        if min(c) < 0 or max(c) > n:
            return -1
        k = 0
        for ci in c:
            k = k * (n + 1) + ci
        return k
    lo, hi = None, -1
    for ell in range(d):
        for e in range(e0, e1):
            k = krow(e, ell)
            if k >= 0:
                lo = k if lo is None else min(lo, k)
                break
        for e in range(e1 - 1, e0 - 1, -1):
            k = krow(e, ell)
            if k >= 0:
                hi = max(hi, k + 1)
                break
    return (0, 0) if hi < 0 else (lo, hi)


def column_range(d: int, n: int, world: int, rank: int) -> tuple[int, int]:
    N = (n + 1) ** d
    return split_range(N, world, rank)


def default_unit_order(d: int, world: int) -> int:
    """SHARED for every world size: one extended product serves all l ((n+2)^d rows of work instead
    of d (n+1)^d), and a contiguous slice of it is a balanced row block on every rank."""
    return UNITS_SHARED


def pack(S: torch.Tensor, G: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """[S_1..S_d, G, b] flattened into one complex128 buffer (one collective)."""
    return torch.cat([S.reshape(-1), G.reshape(-1), b.reshape(-1)])


def unpack(buf: torch.Tensor, d: int, m: int):
    s = d * m * m
    return buf[:s].view(d, m, m), buf[s:s + m * m].view(m, m), buf[s + m * m:s + m * m + m]


def allreduce_pencil(S: torch.Tensor, G: torch.Tensor, b: torch.Tensor, group=None):
    """Sum the per-rank partial pencils: one all_reduce(SUM) of the packed buffer.
    complex128 is reduced as its float64 view (sum of complex = sum of re and im parts)."""
    d, m, _ = S.shape
    buf = pack(S, G, b)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(torch.view_as_real(buf), op=dist.ReduceOp.SUM, group=group)
    return unpack(buf, d, m)


class DistributedPencil:
    """One pencil sharded over the ranks of the default process group (strong scaling of a single
    pencil): rank r computes the partial pencil of its unit range and the partial LS
    products of its column range on its own GPU (libprony), one all_reduce(SUM) of the packed
    [S, G, b] completes them on every rank, and prony_ls_solve gives c, t locally.
    Workspaces and output buffers are allocated once (no allocation per call)."""

    def __init__(self, d: int, n: int, m: int, device, world: int = 1, rank: int = 0, unit_order: int | None = None):
        from . import binding as pb
        self.pb = pb
        self.d, self.n, self.m = d, n, m
        self.world, self.rank = world, rank
        self.order = default_unit_order(d, world) if unit_order is None else unit_order
        self.u0, self.u1 = unit_range(d, n, world, rank, self.order)
        self.c0, self.c1 = column_range(d, n, world, rank)
        self.ws_p = pb.alloc_workspace(pb.WS_PROJECT, d, n, m, device)
        self.ws_l = pb.alloc_workspace(pb.WS_LS, d, n, m, device)
        self.S = torch.empty((d, m, m), dtype=torch.complex128, device=device)
        self.G = torch.empty((m, m), dtype=torch.complex128, device=device)
        self.b = torch.empty(m, dtype=torch.complex128, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        # the LS step is independent of the projection: it runs on a side stream and fills the SMs
        # the projection's last wave leaves idle
        self.side = torch.cuda.Stream(device=device)
        self.ev_in = torch.cuda.Event()
        self.ev_ls = torch.cuda.Event()

    def __call__(self, grid, U, V, sigma, z, stream=None, info_p=None, info_l=None):
        pb, d, n, m = self.pb, self.d, self.n, self.m
        main = stream if stream is not None else torch.cuda.current_stream()
        self.ev_in.record(main)
        pb.project(grid, U, V, sigma, d, n, m, self.u0, self.u1, self.order, out=self.S, workspace=self.ws_p,
                   stream=main, info=info_p)
        full = self.world == 1
        self.side.wait_event(self.ev_in)
        res = pb.vandermonde_ls(z, grid, d, n, m, self.c0, self.c1, want_solution=full,
                                out={"G": self.G, "b": self.b}, workspace=self.ws_l, dev_status=self.status,
                                stream=self.side, info=info_l)
        self.ev_ls.record(self.side)
        main.wait_event(self.ev_ls)
        if full:
            return self.S, res["c"], res["t"]
        Sr, Gr, br = allreduce_pencil(self.S, self.G, self.b)
        c, t = pb.ls_solve(Gr.contiguous(), br.contiguous(), z, d, m, dev_status=self.status, stream=main)
        return Sr, c, t

    def from_host(self, grid_h, U_h, V_h, sigma_h, z_h, z_dev, stream=None):
        """End to end from HOST inputs (page-locked CPU tensors): this rank's partial pencil through
        prony_pencil_host_part (grid, V and only the U rows its unit slab pairs with are copied; the copy
        of V overlaps the projection), then the all-reduce and the local m x m solve. SHARED order only.
        z_dev: the nodes on the device (the solve's t); the LS products read z from z_h."""
        pb, d, n, m = self.pb, self.d, self.n, self.m
        if self.order != UNITS_SHARED:
            raise ValueError("from_host needs the SHARED unit order")
        main = stream if stream is not None else torch.cuda.current_stream()
        if not hasattr(self, "ws_h"):
            self.ws_h = pb.alloc_workspace(pb.WS_PENCIL_HOST, d, n, m, self.S.device)
        pb.pencil_host_part(grid_h, U_h, V_h, sigma_h, z_h, d, n, m, self.u0, self.u1, self.c0, self.c1, self.S,
                            self.G, self.b, workspace=self.ws_h, dev_status=self.status, stream=main)
        Sr, Gr, br = allreduce_pencil(self.S, self.G, self.b)
        c, t = pb.ls_solve(Gr.contiguous(), br.contiguous(), z_dev, d, m, dev_status=self.status, stream=main)
        return Sr, c, t
