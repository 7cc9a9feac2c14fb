"""bench.py — pencils/s and FP64 TFLOP/s of the hot path (S_1..S_d + Vandermonde/LS), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--cfg cfg4] [--impl ours|reference]

A step is one whole pencil of the headline workload (BASELINE.json configs[3], "cfg4": d=2,
n=200, N=40401, m=100, complex-Gaussian noise sigma=1e-6): prony_project over this rank's
units + prony_vandermonde_ls over its columns (+ the NCCL all-reduce of the packed partials
and the m x m solve when N > 1). Inputs are resident in HBM; L2 is flushed (a 256 MiB write)
before every timed step, outside the timed interval. Timing: CUDA events per step on the
launching stream, barrier + synchronize around the loop, max over ranks.

e2e: the same pencil through the C ABI with HOST buffers (prony_pencil_host: pinned host ->
device copies of grid, U, V, sigma, z, the device path, device -> host copies of S, G, b, c, t).

--impl reference: the CPU oracle (oracle/, plain C, all host cores) on a bounded sample of the
same workload per step, extrapolated to pencils/s (this tier has no installable reference).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workload as W  # noqa: E402

METRIC = "pencils/s and FP64 TFLOP/s (% peak) for S_1..S_d+LS, d=2 N=40401 m=100, 1/2/4/8 GPUs"
UNIT = "pencils/s"


def pencil_flops(d, N, m):
    """Algorithmic flops of one pencil: d(8mN^2 + 8Nm^2) + 8m^2 N + 8mN."""
    return d * (8.0 * m * N * N + 8.0 * N * m * m) + 8.0 * m * m * N + 8.0 * m * N


# ------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        loaded = [s for s, p in zip(sm, power) if p > 300.0] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------ reference arm
def run_reference(args, cfg):
    """The oracle, as it stands, on host cores: each step = a bounded sample of one pencil
    (rows [0, R) of T_1 V plus U^* for the pencil part; columns [0, C) of A, G, b for LS),
    extrapolated to a full pencil."""
    import oracle
    oracle.build()
    prob = W.make_problem(cfg)
    c = prob.cfg
    d, n, m, N = c.d, c.n, c.m, c.N
    # calibrate the sample to ~3 s of project work per step (on a warm call: the first one pays the
    # OpenMP pool start-up)
    oracle.project_rows(prob.grid, prob.U, prob.V, prob.sigma, d, n, 1, 0, 8)
    R = min(N, 64)
    t0 = time.perf_counter()
    oracle.project_rows(prob.grid, prob.U, prob.V, prob.sigma, d, n, 1, 0, R)
    per_row = (time.perf_counter() - t0) / R
    R = int(max(8, min(N, 3.0 / max(per_row, 1e-9))))
    Cc = min(N, 4096)

    def step():
        t0 = time.perf_counter()
        oracle.project_rows(prob.grid, prob.U, prob.V, prob.sigma, d, n, 1, 0, R)
        t_proj = time.perf_counter() - t0
        t0 = time.perf_counter()
        A = oracle.vandermonde(prob.z, d, n, 0, Cc)
        oracle.ls_products(A, prob.grid, d, n, 0, Cc)
        t_ls = time.perf_counter() - t0
        return t_proj * (d * N / R) + t_ls * (N / Cc)

    for _ in range(args.warmup):
        step()
    est = [step() for _ in range(args.steps)]
    sec = statistics.median(est)
    value = 1.0 / sec
    sample = (f"per step: oracle_project_rows rows [0,{R}) of T_1 (of d*N={d * N} row-units) + "
              f"vandermonde+ls_products on columns [0,{Cc}) of N={N}; extrapolated linearly to one pencil")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{c.name}: d={d} n={n} N={N} m={m} noise={c.noise}", "d": d, "n": n, "N": N, "m": m,
                   "parallelism": "host threads (OpenMP)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "tflops": pencil_flops(d, N, m) * value / 1e12,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(prob, budget_s=16.0):
    """cpu_baseline leg (rank 0, N=1): the oracle on a bounded sample of the bench workload."""
    import oracle
    oracle.build()
    c = prob.cfg
    d, n, m, N = c.d, c.n, c.m, c.N
    # calibrate the row count on a warm call (the first one pays the OpenMP pool start-up), aiming at
    # ~0.8 * budget_s of projection work in the measured sample
    oracle.project_rows(prob.grid, prob.U, prob.V, prob.sigma, d, n, 1, 0, 8)
    R = 64
    t0 = time.perf_counter()
    oracle.project_rows(prob.grid, prob.U, prob.V, prob.sigma, d, n, 1, 0, R)
    per_row = (time.perf_counter() - t0) / R
    R = int(max(8, min(N, 0.8 * budget_s / max(per_row, 1e-9))))
    t0 = time.perf_counter()
    oracle.project_rows(prob.grid, prob.U, prob.V, prob.sigma, d, n, 1, 0, R)
    t_proj = time.perf_counter() - t0
    Cc = min(N, 8192)
    t0 = time.perf_counter()
    A = oracle.vandermonde(prob.z, d, n, 0, Cc)
    oracle.ls_products(A, prob.grid, d, n, 0, Cc)
    t_ls = time.perf_counter() - t0
    sec = t_proj * (d * N / R) + t_ls * (N / Cc)
    return {"value": 1.0 / sec, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
            "sample": (f"oracle_project_rows on rows [0,{R}) of T_1 ({t_proj:.1f} s) + vandermonde/ls_products on "
                       f"columns [0,{Cc}) ({t_ls:.1f} s), extrapolated to one pencil of {c.name} "
                       f"({d * N} row-units, {N} columns): {sec:.0f} s per pencil")}


# ------------------------------------------------------------------------------------ our arm
def zgemm_peak_tflops(torch, n=4096, reps=5):
    """cuBLAS ZGEMM (complex128) throughput measured now: the FP64-tensor roofline denominator."""
    a = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    b = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    c = torch.empty_like(a)
    for _ in range(2):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b, out=c)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    del a, b, c
    return 8.0 * n ** 3 / (best * 1e-3) / 1e12


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2012_11430_b200 as pb
    from paper_2012_11430_b200 import sharding

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # gloo: functional check of the N>1 path with several ranks on one GPU (no waiting kernels)
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local)

    prob = W.make_problem(cfg)
    c = prob.cfg
    d, n, m, N = c.d, c.n, c.m, c.N
    tg = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    grid, U, V, sigma, z = tg(prob.grid), tg(prob.U), tg(prob.V), tg(prob.sigma), tg(prob.z)
    order_arg = {"l-major": 0, "row-major": 1, "shared": 2}[args.units]
    pencil = sharding.DistributedPencil(d, n, m, dev, world, rank, unit_order=order_arg)
    order = pencil.order
    st = pencil.status
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def new_events(k):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        for e in evs:
            e.record(stream)  # force creation so .cuda_event is a live handle
        return evs

    def step(info_p=None, info_l=None):
        return pencil(grid, U, V, sigma, z, stream=stream, info_p=info_p, info_l=info_l)

    # warm-up (also validates the device status once)
    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    assert int(st.item()) == 0, f"device status {int(st.item())}"

    K = args.steps
    ev_s, ev_e = new_events(K), new_events(K)
    ev_ps, ev_pe = new_events(K), new_events(K)
    ev_ls, ev_le = new_events(K), new_events(K)
    infos_p = [pb.make_exec_info(ev_ps[i], ev_pe[i]) for i in range(K)]
    infos_l = [pb.make_exec_info(ev_ls[i], ev_le[i]) for i in range(K)]
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(K):
        flush.fill_(i & 0xFF)                  # L2 flush outside the timed interval
        ev_s[i].record(stream)
        step(infos_p[i], infos_l[i])
        ev_e[i].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()

    step_ms = [ev_s[i].elapsed_time(ev_e[i]) for i in range(K)]
    proj_ms = [ev_ps[i].elapsed_time(ev_pe[i]) for i in range(K)]
    vls_ms = [ev_ls[i].elapsed_time(ev_le[i]) for i in range(K)]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms, sum(proj_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms_max = float(t[0])
    launches_per_step = infos_p[0].launches + infos_l[0].launches + (1 if world > 1 else 0)

    # ---- end to end from pinned host buffers: N = 1 through the C-ABI host call prony_pencil_host;
    # N > 1 through the sharded public API (pinned H2D of the inputs on every rank, the pencil, D2H of
    # S, c, t on rank 0), the whole interval timed on the device (max over ranks)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    hg, hU, hV, hs, hz = pin(prob.grid), pin(prob.U), pin(prob.V), pin(prob.sigma), pin(prob.z)
    h2d = sum(x.numel() * x.element_size() for x in (hg, hU, hV, hs, hz))
    Ke = max(2, min(K, 5))
    e_ms = []
    if world == 1:
        outs = {k: torch.empty(s, dtype=dt).pin_memory() for k, s, dt in
                [("S", (d, m, m), torch.complex128), ("G", (m, m), torch.complex128), ("b", (m,), torch.complex128),
                 ("c", (m,), torch.complex128), ("t", (m, d), torch.float64)]}
        ws_h = pb.alloc_workspace(pb.WS_PENCIL_HOST, d, n, m, dev)
        for _ in range(max(args.warmup, 3)):  # e2e warm-up: same count as the device loop
            pb.pencil_host(hg, hU, hV, hs, hz, d, n, m, workspace=ws_h, outputs=outs, stream=stream)
        for i in range(Ke):
            flush.fill_(i & 0xFF)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = pb.pencil_host(hg, hU, hV, hs, hz, d, n, m, workspace=ws_h, outputs=outs, stream=stream)
            e1.record(stream)
            e1.synchronize()
            assert r["status"] == 0
            e_ms.append(e0.elapsed_time(e1))
        d2h = sum(x.numel() * x.element_size() for x in outs.values() if isinstance(x, torch.Tensor)) + 4
        api = "prony_pencil_host (C ABI, pinned host buffers)"
        del ws_h
    else:
        dg, dU, dV, ds, dz = (torch.empty_like(x, device=dev) for x in (hg, hU, hV, hs, hz))
        hS = torch.empty((d, m, m), dtype=torch.complex128).pin_memory()
        hc = torch.empty(m, dtype=torch.complex128).pin_memory()
        ht = torch.empty((m, d), dtype=torch.float64).pin_memory()

        shared = pencil.order == sharding.UNITS_SHARED
        if shared:  # per rank: grid, V, sigma, z (+ z for the solve) and only the U rows its slab pairs with
            ulo, uhi = sharding.shared_u_rows(d, n, pencil.u0, pencil.u1)
            h2d_rank = (hg.numel() + hV.numel() + 2 * hz.numel() + (uhi - ulo) * m) * 16 + hs.numel() * 8
        else:
            h2d_rank = h2d
        hb = torch.tensor([float(h2d_rank)], dtype=torch.float64, device=dev)
        dist.all_reduce(hb, op=dist.ReduceOp.SUM)
        h2d_total = int(hb.item())

        def e2e_step():
            if shared:
                dz.copy_(hz, non_blocking=True)
                Sx, cx, tx = pencil.from_host(hg, hU, hV, hs, hz, dz, stream=stream)
            else:
                for dst, src in ((dg, hg), (dU, hU), (dV, hV), (ds, hs), (dz, hz)):
                    dst.copy_(src, non_blocking=True)
                Sx, cx, tx = pencil(dg, dU, dV, ds, dz, stream=stream)
            if rank == 0:
                hS.copy_(Sx, non_blocking=True)
                hc.copy_(cx, non_blocking=True)
                ht.copy_(tx, non_blocking=True)

        for _ in range(max(args.warmup, 3)):
            e2e_step()
        torch.cuda.synchronize()
        for i in range(Ke):
            flush.fill_(i & 0xFF)
            torch.cuda.synchronize()
            dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            e2e_step()
            e1.record(stream)
            e1.synchronize()
            e_ms.append(e0.elapsed_time(e1))
        d2h = (hS.numel() + hc.numel()) * 16 + ht.numel() * 8
        api = ("sharding.DistributedPencil.from_host -> prony_pencil_host_part (pinned H2D per rank, V copy "
               "overlapped, all-reduce, D2H on rank 0)" if shared else
               "sharding.DistributedPencil (pinned H2D per rank, all-reduce, D2H on rank 0)")
    te = torch.tensor([sum(e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = {"value": Ke / (float(te[0]) * 1e-3), "unit": UNIT,
           "h2d_bytes_per_step": h2d if world == 1 else h2d_total,
           "d2h_bytes_per_step": d2h, "ms_per_step": float(te[0]) / Ke, "api": api}

    # ---- roofline of the dominant kernel (k_project), measured live above
    flops_proj = infos_p[0].main_flops
    proj_avg_s = statistics.mean(proj_ms) * 1e-3
    peak = zgemm_peak_tflops(torch) if rank == 0 else None

    if rank == 0:
        value = K / (total_ms_max * 1e-3)   # one pencil per step, sharded over the ranks
        ms_per_step = total_ms_max / K
        F = pencil_flops(d, N, m)
        traffic = None
        prof = os.path.join(ROOT, "profiles", "r01_ncu_project.json")
        if os.path.exists(prof):
            try:
                traffic = json.load(open(prof)).get("dram_bytes_per_launch")
            except (OSError, ValueError):
                traffic = None
        achieved = flops_proj / proj_avg_s / 1e12
        cm = 1.0 if os.environ.get("PRONY_CMUL", "3m").startswith("4") else 0.75
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",  # one pencil per step at every N (fixed total work)
            "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded planted exponential sum, complex Gaussian noise 1e-6)",
            "config": {"workload": f"{c.name}: d={d} n={n} N={N} m={m} noise={c.noise} (BASELINE configs[{int(c.name[3:]) - 1}])",
                       "d": d, "n": n, "N": N, "m": m, "parallelism": f"dp{world} ({['l-major', 'row-major', 'shared'][order]} units)",
                       "l2": "flushed (256 MiB write) before every timed step, outside the timed interval",
                       "pencils_per_step": 1, "comm": "1 x all_reduce(SUM) of packed [S,G,b] per step" if world > 1 else "none"},
            "tflops": F * value / 1e12,
            "pct_peak": (F * value / 1e12) / (peak * world) if peak else None,
            "flop_accounting": ("tflops/pct_peak count the paper's d(8mN^2+8Nm^2)+8m^2N+8mN per pencil; with "
                                "shared units one extended product T_E V ((n+2)^d rows) replaces the d products "
                                "T_l V (d(n+1)^d rows), DESIGN.md F8; roofline.achieved counts the flops of the "
                                "product k_project actually computes (8 m N rows), as a 4M ZGEMM would"),
            "roofline": {"bound": "tensor", "kernel": "k_project (complex FP64 DMMA, implicit Toeplitz gather)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                         "traffic": traffic,
                         "peak_source": "cuBLAS ZGEMM 4096^3 complex128 measured in this run (MEASURED_PEAKS.json has no FP64 entry; a bf16-peak x nominal-ratio figure would understate the FP64 pipe)",
                         "frac_of": "measured",
                         "flops_per_launch": flops_proj, "avg_launch_ms": proj_avg_s * 1e3,
                         # 3M executes 3 of 4 real products, on NP = 8 ceil(m/8) padded columns:
                         "executed_tflops": achieved * cm * (8 * ((m + 7) // 8)) / m,
                         "executed_frac": (achieved * cm * (8 * ((m + 7) // 8)) / m) / peak if peak else None,
                         "cmul": "4M" if cm == 1.0 else "3M",
                         # also against the planning figure 148 SM x 128 FP64 flop/clk x 1.965 GHz
                         "planning_peak": 37.2, "executed_frac_vs_planning": (achieved * cm * (8 * ((m + 7) // 8)) / m) / 37.2,
                         "share_of_step": sum(proj_ms) / sum(step_ms),
                         "grid": list(infos_p[0].main_grid), "split_k": infos_p[0].split_k},
            "kernels_ms": {"k_project": statistics.mean(proj_ms), "k_vls": statistics.mean(vls_ms)},
            "gpu_launches": launches_per_step * K,
            "clocks": clk,
            "e2e": e2e,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_sample(prob)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cfg", default="cfg4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--units", default="shared", choices=["shared", "l-major", "row-major"],
                    help="prony_unit_order of the projection (shared: one extended product for all l, F8)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = W.CONFIGS[args.cfg]
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        run_reference(args, cfg)
        return
    from paper_2012_11430_b200 import _build
    _build.build()
    run_ours(args, cfg)


if __name__ == "__main__":
    main()
