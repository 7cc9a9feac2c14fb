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


def host_rows(d: int, n: int, world: int, rank: int, order: int = UNITS_SHARED):
    """What rank `rank` copies from its host in the scatter mode of DistributedPencil.from_host: rows
    [v0, v1) of V (a padded equal split of N: chunk = ceil(N / world) rows per rank) and rows [ulo, uhi)
    of U (those its unit slab pairs with; all of U for the per-l orders). Returns (chunk, (v0, v1), (ulo, uhi))."""
    N = (n + 1) ** d
    chunk = -(-N // world)
    v0, v1 = min(rank * chunk, N), min((rank + 1) * chunk, N)
    if order == UNITS_SHARED:
        u0, u1 = unit_range(d, n, world, rank, order)
        ulo, uhi = shared_u_rows(d, n, u0, u1)
    else:
        ulo, uhi = 0, N
    return chunk, (v0, v1), (ulo, uhi)


def h2d_bytes(d: int, n: int, m: int, world: int, rank: int, order: int = UNITS_SHARED, scatter_v: bool = True) -> int:
    """Host -> device bytes of one rank per pencil in from_host: the grid, V (its slice, or all of it),
    the U rows of its slab, sigma, z."""
    N = (n + 1) ** d
    _, (v0, v1), (ulo, uhi) = host_rows(d, n, world, rank, order)
    vrows = (v1 - v0) if scatter_v else N
    return ((2 * n + 2) ** d + (vrows + (uhi - ulo)) * m + m * d) * 16 + m * 8


def allgather_rows(buf: torch.Tensor, world: int, rank: int, mine: torch.Tensor | None = None,
                   collective: bool | None = None) -> None:
    """buf: (chunk * world, ...); this rank's rows are in `mine` (chunk, ...) — or already at
    [rank * chunk, (rank + 1) * chunk) of buf when mine is None. Afterwards every rank holds all of them
    in buf (one all_gather, out of place from `mine`). collective=False (default at world 1): a local copy."""
    chunk = buf.shape[0] // world
    if mine is None:
        mine = buf[rank * chunk:(rank + 1) * chunk].clone()
    if not (world > 1 if collective is None else collective):
        buf.copy_(mine)
        return
    real = (lambda x: torch.view_as_real(x)) if buf.is_complex() else (lambda x: x)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(real(buf), real(mine))
    else:
        parts = list(buf.view(world, chunk, *buf.shape[1:]).unbind(0))
        dist.all_gather([real(p) for p in parts], real(mine))


class DistributedPencil:
    """One pencil sharded over the ranks of the default process group (strong scaling of a single
    pencil): rank r computes the partial pencil of its unit range and the partial LS
    products of its column range on its own GPU (libprony), one all_reduce(SUM) of the packed
    [S, G, b] completes them on every rank, and prony_ls_solve gives c, t locally.
    Workspaces and output buffers are allocated once (no allocation per call). Every call runs on
    `stream` (default: the current stream): the projection, the packing, the collective and the solve
    are all ordered on it; the LS products run on a side stream that joins it before the collective."""

    def __init__(self, d: int, n: int, m: int, device, world: int = 1, rank: int = 0, unit_order: int | None = None,
                 collective: bool | None = None):
        """collective: run the partial path with its collectives (default: world > 1). collective=True at
        world 1 drives the N > 1 code path, NCCL calls included, on a one-rank process group (tested)."""
        from . import binding as pb
        self.pb = pb
        self.d, self.n, self.m = d, n, m
        self.N = (n + 1) ** d
        self.world, self.rank = world, rank
        self.collective = world > 1 if collective is None else collective
        self.device = torch.device(device)
        self.order = default_unit_order(d, world) if unit_order is None else unit_order
        self.u0, self.u1 = unit_range(d, n, world, rank, self.order)
        self.c0, self.c1 = column_range(d, n, world, rank)
        self.ws_p = pb.alloc_workspace(pb.WS_PROJECT, d, n, m, device)
        self.ws_l = pb.alloc_workspace(pb.WS_LS, d, n, m, device)
        # S, G, b are views of ONE packed buffer: the kernels write their partials straight into it and the
        # all-reduce runs in place (no pack / unpack copies)
        self.buf = torch.empty(d * m * m + m * m + m, dtype=torch.complex128, device=device)
        self.S, self.G, self.b = unpack(self.buf, d, m)
        self.c = torch.empty(m, dtype=torch.complex128, device=device)
        self.t = torch.empty((m, d), dtype=torch.float64, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        # the projection runs on a HIGH-priority stream, the LS step on a normal-priority side stream: the LS
        # CTAs fill the SMs the projection's last wave leaves idle without delaying any projection CTA
        self.hi = torch.cuda.Stream(device=device, priority=-1)
        self.ctx = None  # prony_host_context of the single-rank one-call path (created on first use)
        self.outs = {"S": self.S, "G": self.G, "b": self.b, "c": self.c, "t": self.t}
        self.side = torch.cuda.Stream(device=device)
        self.ev_in = torch.cuda.Event()
        self.ev_ls = torch.cuda.Event()
        # recorded by the library right after k_project (N > 1): the LS branch's all-reduce of [G, b] waits
        # for it, so no rank's NCCL kernel occupies SMs (spinning on its peers) while projections still run
        self.ev_proj = torch.cuda.Event()
        self.ev_proj.record(torch.cuda.current_stream(self.device))  # materialize the handle
        # recorded by the library right BEFORE k_project (after the prep kernels): the LS branch starts there, so
        # in back-to-back calls its CTAs cannot take the SMs ahead of k_project's first wave
        self.ev_pbeg = torch.cuda.Event()
        self.ev_pbeg.record(torch.cuda.current_stream(self.device))

    def __call__(self, grid, U, V, sigma, z, stream=None, ev_project=None, ev_ls=None, ev_comm=None, ev_wait_u=None):
        """Device-resident inputs -> (S, c, t) (views of this object's buffers, valid until the next call).
        Ordered after prior work on `stream` (default: the current stream), which is ordered after all of it
        on return. ev_project / ev_ls: optional (begin, end) timing torch.cuda.Events the library records
        around k_project / k_vls (each already recorded once so its handle exists); ev_comm: optional
        (begin, end) events recorded around the collective of S; ev_wait_u: optional event after which U is complete
        (a copy still in flight on another stream): only the reduction, the first kernel reading U, waits for it.

        N > 1: the LS branch (side stream, released right before k_project, which runs on a HIGHER-priority
        stream) gets SMs only once k_project's CTA queue is drained — in its last wave — and all-reduces its G, b
        and solves for c, t there, so the NCCL kernel and the one-CTA solve use the SMs the last wave leaves idle
        instead of following k_project; the projection stream then runs k_reduce_ws, k_finalize and the
        all-reduce of S."""
        pb, d, n, m = self.pb, self.d, self.n, self.m
        main = stream if stream is not None else torch.cuda.current_stream(self.device)
        full = not self.collective
        pe = ev_project if ev_project is not None else (self.ev_pbeg, self.ev_proj)
        info_p = pb.make_exec_info(pe[0], pe[1], ev_wait_u)
        info_l = pb.make_exec_info(*ev_ls) if ev_ls is not None else pb.make_exec_info()
        if full and self.order == UNITS_SHARED:
            # one C call (prony_pencil): the projection on `main`, the LS step on the context's side stream
            if self.ctx is None:
                self.ctx = pb.HostContext()
                self.ws_pencil = pb.alloc_workspace(pb.WS_PENCIL, d, n, m, self.device)
            if ev_wait_u is not None:  # prony_pencil has no U hook: the whole call waits for U
                main.wait_event(ev_wait_u)
            # prony_pencil zeroes the status word in its first kernel (no separate reset launch)
            pb.pencil(grid, U, V, sigma, z, d, n, m, self.outs, self.ws_pencil, context=self.ctx,
                      dev_status=self.status, stream=main, info_p=info_p, info_l=info_l)
            self._note(info_p, info_l, 0)
            return self.S, self.c, self.t
        hi, side = self.hi, self.side
        hi.wait_stream(main)
        with torch.cuda.stream(hi):
            self.status.zero_()
            self.ev_in.record(hi)
            pb.project(grid, U, V, sigma, d, n, m, self.u0, self.u1, self.order, out=self.S, workspace=self.ws_p,
                       dev_status=self.status, stream=hi, info=info_p)
        side.wait_event(self.ev_in)
        side.wait_event(pe[0])  # recorded by the library right before k_project (stale only if it had no rows)
        with torch.cuda.stream(side):
            res = pb.vandermonde_ls(z, grid, d, n, m, self.c0, self.c1, want_solution=full,
                                    out={"G": self.G, "b": self.b, "c": self.c, "t": self.t}, workspace=self.ws_l,
                                    dev_status=self.status, stream=side, info=info_l)
            if not full:
                self._allreduce(self.buf[d * m * m:])            # G, b (in k_project's last wave)
                pb.ls_solve(self.G, self.b, z, d, m, dev_status=self.status, stream=side,
                            out={"c": self.c, "t": self.t})
            self.ev_ls.record(side)
        with torch.cuda.stream(hi):
            if not full:
                if ev_comm is not None:
                    ev_comm[0].record(hi)
                self._allreduce(self.buf[:d * m * m])            # S
                if ev_comm is not None:
                    ev_comm[1].record(hi)
            hi.wait_event(self.ev_ls)
        main.wait_stream(hi)
        self._note(info_p, info_l, 0 if full else 1)
        return self.S, (res["c"] if full else self.c), (res["t"] if full else self.t)

    def _note(self, info_p, info_l, extra):
        """Launch record of the last call (the bench's gpu_launches and roofline fields): libprony kernels
        launched (+ the separate k_solve at N > 1), the dominant kernel's flops (ZGEMM convention), grid, split-K."""
        self.last_launches = info_p.launches + info_l.launches + extra
        self.last_main_flops = info_p.main_flops
        self.last_grid = list(info_p.main_grid)
        self.last_split_k = info_p.split_k

    def _allreduce(self, x):
        if self.collective and dist.is_available() and dist.is_initialized():
            dist.all_reduce(torch.view_as_real(x), op=dist.ReduceOp.SUM)

    def _reduce_and_solve(self, z, st, ev_comm=None):
        pb, d, m = self.pb, self.d, self.m
        if ev_comm is not None:
            ev_comm[0].record(st)
        self._allreduce(self.buf)
        if ev_comm is not None:
            ev_comm[1].record(st)
        c, t = pb.ls_solve(self.G, self.b, z, d, m, dev_status=self.status, stream=st, out={"c": self.c, "t": self.t})
        return self.S, c, t

    # ------------------------------------------------------------------ end to end from host buffers
    def h2d_bytes(self, scatter_v: bool = True) -> int:
        return h2d_bytes(self.d, self.n, self.m, self.world, self.rank, self.order, scatter_v)

    def from_host(self, grid_h, U_h, V_h, sigma_h, z_h, stream=None, scatter_v: bool = True, ev_comm=None):
        """End to end from HOST inputs (page-locked CPU tensors) -> (S, c, t) on the device.

        scatter_v=True (default for world > 1): PCIe is the scarce link and NVLink the abundant one, so
        each rank copies only ITS 1/world slice of V's rows (plus the grid, the U rows its unit slab pairs
        with, sigma and z) from its host, and one all_gather over NVLink assembles V on every rank; then
        the device path of __call__. Per-rank H2D: (N/world + U slab) m + box complex values instead of
        (N + U slab) m + box.
        scatter_v=False: prony_pencil_host_part (C ABI): the full V and the grid per rank, V's copy
        overlapped with the projection (SHARED order only)."""
        pb, d, n, m = self.pb, self.d, self.n, self.m
        main = stream if stream is not None else torch.cuda.current_stream(self.device)
        dev = self.device
        if not hasattr(self, "dz"):
            chunk = -(-self.N // self.world)
            self.dz = torch.empty((m, d), dtype=torch.complex128, device=dev)
            self.dgrid = torch.empty((2 * n + 2) ** d, dtype=torch.complex128, device=dev)
            self.dsig = torch.empty(m, dtype=torch.float64, device=dev)
            self.dU = torch.zeros((self.N, m), dtype=torch.complex128, device=dev)
            self.dVpad = torch.zeros((chunk * self.world, m), dtype=torch.complex128, device=dev)
            self.dVmine = torch.zeros((chunk, m), dtype=torch.complex128, device=dev)
            self.su = torch.cuda.Stream(device=dev)  # U rows behind V's slice, overlapped with the projection
            self.ev_vcopied = torch.cuda.Event()
            self.ev_ucopied = torch.cuda.Event()
        with torch.cuda.stream(main):
            self.dz.copy_(z_h, non_blocking=True)
            if not scatter_v:
                if self.order != UNITS_SHARED:
                    raise ValueError("scatter_v=False needs the SHARED unit order")
                if not hasattr(self, "ws_h"):
                    self.ws_h = pb.alloc_workspace(pb.WS_PENCIL_HOST, d, n, m, dev)
                    self.hctx = pb.HostContext()
                if not self.collective:
                    raise ValueError("scatter_v=False is the N > 1 partial path")
                self.status.zero_()
                pb.pencil_host_part(grid_h, U_h, V_h, sigma_h, z_h, d, n, m, self.u0, self.u1, self.c0, self.c1,
                                    self.S, self.G, self.b, workspace=self.ws_h, dev_status=self.status, stream=main,
                                    context=self.hctx)
                return self._reduce_and_solve(self.dz, main, ev_comm)
            if not hasattr(self, "rows_h"):  # a Python scan over the unit range: computed once, not per call
                self.rows_h = host_rows(d, n, self.world, self.rank, self.order)
            chunk, (v0, v1), (ulo, uhi) = self.rows_h
            self.dgrid.copy_(grid_h, non_blocking=True)
            self.dsig.copy_(sigma_h, non_blocking=True)
            if v1 > v0:
                self.dVmine[:v1 - v0].copy_(V_h[v0:v1], non_blocking=True)
            self.ev_vcopied.record(main)
        # the U rows cross the link after V's slice (so they do not slow it down) on their own stream; only the
        # reduction at the end of the projection waits for them (prony_exec_info.ev_wait_u)
        self.su.wait_event(self.ev_vcopied)
        with torch.cuda.stream(self.su):
            if uhi > ulo:
                self.dU[ulo:uhi].copy_(U_h[ulo:uhi], non_blocking=True)
            self.ev_ucopied.record(self.su)
        with torch.cuda.stream(main):
            allgather_rows(self.dVpad, self.world, self.rank, self.dVmine, collective=self.collective)
            V = self.dVpad[:self.N]
        return self(self.dgrid, self.dU, V, self.dsig, self.dz, stream=main, ev_comm=ev_comm, ev_wait_u=self.ev_ucopied)
