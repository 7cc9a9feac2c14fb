"""bench.py — pencils/s and FP64 TFLOP/s of the hot path (S_1..S_d + Vandermonde/LS), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--cfg cfg4] [--units shared|l-major|row-major]
                    [--impl ours|reference] [--dist-backend nccl|gloo]

A step is one whole pencil of the headline workload (BASELINE.json configs[3], "cfg4": d=2,
n=200, N=40401, m=100, complex-Gaussian noise sigma=1e-6): prony_project over this rank's
units + prony_vandermonde_ls over its columns (+ the NCCL all-reduce of the packed partials
and the m x m solve when N > 1). Inputs are resident in HBM; L2 is flushed (a 256 MiB write)
before every timed step, outside the timed interval. Timing: CUDA events per step on the
launching stream, barrier + synchronize around the loop, max over ranks.

--gpus N > 1 without a torchrun environment re-executes itself under
`python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1`, so the
driver's `python bench.py --gpus N` and its torchrun form run the same N-rank job.

e2e: the same pencil end to end from pinned HOST buffers — N = 1 through the C ABI
(prony_pencil_host); N > 1 through sharding.DistributedPencil.from_host (each rank copies its slice
of V, its U rows and the grid; V is all-gathered over NVLink; all-reduce; D2H of S, c, t on rank 0).

--impl reference: the CPU oracle (oracle/, plain C, all host cores) on a bounded sample of the
same workload per step, extrapolated to pencils/s (this tier has no installable reference).
"""
from __future__ import annotations

import argparse
import fcntl
import hashlib
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
# sources of k_project: an ncu capture is used for roofline.traffic only if it was taken on these
KPROJECT_SOURCES = ["paper_2012_11430_b200/csrc/project.cu", "paper_2012_11430_b200/csrc/project.cuh",
                    "paper_2012_11430_b200/csrc/engine.cuh", "paper_2012_11430_b200/csrc/common.cuh"]
TRAFFIC_PROFILE = os.path.join(ROOT, "profiles", "ncu_k_project_current.json")


def paper_pencil_flops(d, N, m):
    """The paper's formulation: d separate products T_l V and U^* (T_l V), ZGEMM
    convention (8 real flops per complex MAC): d(8mN^2 + 8Nm^2) + 8m^2 N + 8mN."""
    return d * (8.0 * m * N * N + 8.0 * N * m * m) + 8.0 * m * m * N + 8.0 * m * N


def source_stamp(paths=KPROJECT_SOURCES):
    h = hashlib.sha1()
    for p in paths:
        with open(os.path.join(ROOT, p), "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


# ------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms during the timed region."""
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
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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


# ------------------------------------------------------------------------------------ the oracle on host cores
def oracle_pencil_sample(prob, budget_s):
    """The oracle, as it stands, on a bounded sample of one pencil: rows [0, R) of T_1 through
    oracle_project_rows (naive T_1 V then U^*, the O(N^2 m) part) and columns [0, C) through
    oracle_vandermonde + oracle_ls_products; R is calibrated on a warm call to ~0.8 budget_s.
    Returns (seconds per pencil extrapolated linearly to d*N rows and N columns, sample description)."""
    import oracle
    c = prob.cfg
    d, n, m, N = c.d, c.n, c.m, c.N
    oracle.project_rows(prob.grid, prob.U, prob.V, prob.sigma, d, n, 1, 0, min(8, N))  # warm the thread pool
    R = min(N, 64)
    t0 = time.perf_counter()
    oracle.project_rows(prob.grid, prob.U, prob.V, prob.sigma, d, n, 1, 0, R)
    per_row = (time.perf_counter() - t0) / R
    R = int(max(1, min(N, 0.8 * budget_s / max(per_row, 1e-9))))
    t0 = time.perf_counter()
    oracle.project_rows(prob.grid, prob.U, prob.V, prob.sigma, d, n, 1, 0, R)
    t_proj = time.perf_counter() - t0
    Cc = min(N, 8192)
    t0 = time.perf_counter()
    A = oracle.vandermonde(prob.z, d, n, 0, Cc)
    oracle.ls_products(A, prob.grid, d, n, 0, Cc)
    t_ls = time.perf_counter() - t0
    sec = t_proj * (d * N / R) + t_ls * (N / Cc)
    sample = (f"oracle_project_rows on rows [0,{R}) of T_1 ({t_proj:.1f} s) + vandermonde/ls_products on columns "
              f"[0,{Cc}) ({t_ls:.2f} s), extrapolated linearly to one pencil of {c.name} ({d * N} T_l rows, {N} "
              f"columns): {sec:.1f} s per pencil")
    return sec, sample, t_proj + t_ls


def host_info():
    import oracle
    return {"nproc": os.cpu_count(), "omp_num_threads": os.environ.get("OMP_NUM_THREADS"),
            "threads_used": oracle.num_threads()}


def cpu_baseline(prob, budget_s=16.0):
    """cpu_baseline leg (rank 0, N=1): the oracle on all host cores on a bounded sample of the bench workload,
    plus the small configs cfg1/cfg2 on ONE core (same bounded sampling, ~3 s each)."""
    import oracle
    oracle.build()
    sec, sample, _ = oracle_pencil_sample(prob, budget_s)
    info = host_info()
    small = {}
    threads = oracle.num_threads()
    try:
        oracle.set_num_threads(1)
        for name in ("cfg1", "cfg2"):
            p = W.make_problem(name)
            s1, _, _ = oracle_pencil_sample(p, 3.0)
            small[name] = {"value": 1.0 / s1, "unit": UNIT, "cores": 1}
    finally:
        oracle.set_num_threads(threads)
    return {"value": 1.0 / sec, "unit": UNIT, "cores": info["threads_used"], "kind": "oracle", "sample": sample,
            **info, "small_configs_1core": small}


def run_reference(args, cfg):
    """Reference arm: the oracle, as it stands, on host cores; each step = a bounded sample of the same kind as
    the cpu_baseline leg (~7 s of CPU work: large enough that the oracle's per-call marshalling of U, V does not
    inflate the extrapolation; a 3 s sample read ~20% slower than cpu_baseline's 12 s one). A step computes a
    known fraction of one pencil (the sampled rows and columns), so ms_per_step is the measured time of that
    sample and value = fraction / step time = pencils/s."""
    import oracle
    oracle.build()
    prob = W.make_problem(cfg)
    c = prob.cfg
    d, n, m, N = c.d, c.n, c.m, c.N
    est, step_s, sample = [], [], ""
    for i in range(args.warmup + args.steps):
        sec, sample, t_step = oracle_pencil_sample(prob, 8.0)
        if i >= args.warmup:
            est.append(sec)
            step_s.append(t_step)
    sec = statistics.median(est)
    value = 1.0 / sec
    ms_step = statistics.median(step_s) * 1e3
    info = host_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "pencils_per_step": ms_step * 1e-3 / sec,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{c.name}: d={d} n={n} N={N} m={m} noise={c.noise}", "d": d, "n": n, "N": N, "m": m,
                   "parallelism": "host threads (OpenMP)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["threads_used"], "kind": "oracle",
                         "sample": "per step: " + sample, **info},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "paper_equivalent_tflops": paper_pencil_flops(d, N, m) * value / 1e12,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------ our arm
def zgemm_peak_tflops(torch, index, n=4096, reps=40):
    """cuBLAS ZGEMM (complex128, 4 real DMMA products) throughput measured now, best of `reps`: the
    FP64-tensor roofline denominator (real FP64 flop/s), with the SM clocks sampled while it runs."""
    a = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    b = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    c = torch.empty_like(a)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    clocks = ClockSampler(index)
    clocks.start()
    best = 1e30
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b, out=c)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    clk = clocks.stop()
    del a, b, c
    return 8.0 * n ** 3 / (best * 1e-3) / 1e12, clk


def stamped_traffic():
    """roofline.traffic: dram bytes per k_project launch from the committed ncu --set full summary, used
    only if that capture was taken on the current k_project sources (source stamp match)."""
    try:
        j = json.load(open(TRAFFIC_PROFILE))
    except (OSError, ValueError):
        return None, "no capture"
    if j.get("source_stamp") != source_stamp():
        return None, f"stale capture ({j.get('source_stamp')} != {source_stamp()})"
    return j.get("dram_bytes_per_launch"), os.path.relpath(TRAFFIC_PROFILE, ROOT)


def other_configs(names, dev, peak, steps=10, warmup=3):
    """The other BASELINE configs through the same device path on this GPU (parity cases, not bench lines), so
    the driver's own run records them too: pencils/s, ms per pencil, k_project ms and its fraction of the
    measured FP64 peak (real 3M flops). Same timing rules: warm-up, L2 flushed before each step, CUDA events."""
    import torch

    from paper_2012_11430_b200 import sharding
    out = {}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    for name in names:
        prob = W.make_problem(W.CONFIGS[name])
        c = prob.cfg
        tg = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        args = [tg(x) for x in (prob.grid, prob.U, prob.V, prob.sigma, prob.z)]
        pencil = sharding.DistributedPencil(c.d, c.n, c.m, dev)
        for _ in range(warmup):
            pencil(*args, stream=stream)
        torch.cuda.synchronize()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
        for e in ev:
            for x in e:
                x.record(stream)
        torch.cuda.synchronize()
        for i in range(steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record(stream)
            pencil(*args, stream=stream, ev_project=(ev[i][2], ev[i][3]))
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        assert int(pencil.status.item()) == 0, f"{name}: device status {int(pencil.status.item())}"
        step = sum(e[0].elapsed_time(e[1]) for e in ev) / steps
        proj = sum(e[2].elapsed_time(e[3]) for e in ev) / steps
        achieved = 6.0 * (pencil.last_main_flops / 8.0) / (proj * 1e-3) / 1e12
        out[name] = {"workload": f"d={c.d} n={c.n} N={c.N} m={c.m} noise={c.noise}", "pencils_per_s": 1e3 / step,
                     "ms_per_step": step, "k_project_ms": proj,
                     "k_project_frac": achieved / peak if peak else None}
        del pencil, args
    del flush
    return out


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
    # --force-dist: the N > 1 code path (process group, collectives, per-rank gather) on a one-rank group
    dist_on = world > 1 or args.force_dist
    if dist_on:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if "MASTER_PORT" not in os.environ:
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
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
    pencil = sharding.DistributedPencil(d, n, m, dev, world, rank, unit_order=order_arg, collective=dist_on)
    order = pencil.order
    st = pencil.status
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def new_events(k):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        for e in evs:
            e.record(stream)  # force creation so .cuda_event is a live handle
        return evs

    # warm-up (also validates the device status once)
    for _ in range(max(args.warmup, 0)):
        pencil(grid, U, V, sigma, z, stream=stream)
    torch.cuda.synchronize()
    assert int(st.item()) == 0, f"device status {int(st.item())}"

    K = args.steps
    ev_s, ev_e = new_events(K), new_events(K)
    ev_ps, ev_pe = new_events(K), new_events(K)
    ev_ls, ev_le = new_events(K), new_events(K)
    ev_cs, ev_ce = new_events(K), new_events(K)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(K):
        flush.fill_(i & 0xFF)                  # L2 flush outside the timed interval
        ev_s[i].record(stream)
        pencil(grid, U, V, sigma, z, stream=stream, ev_project=(ev_ps[i], ev_pe[i]), ev_ls=(ev_ls[i], ev_le[i]),
               ev_comm=(ev_cs[i], ev_ce[i]) if dist_on else None)
        ev_e[i].record(stream)
    torch.cuda.synchronize()
    if dist_on:
        dist.barrier()
    clk = clocks.stop()
    assert int(st.item()) == 0, f"device status {int(st.item())}"

    step_ms = [ev_s[i].elapsed_time(ev_e[i]) for i in range(K)]
    proj_ms = [ev_ps[i].elapsed_time(ev_pe[i]) for i in range(K)]
    vls_ms = [ev_ls[i].elapsed_time(ev_le[i]) for i in range(K)]
    comm_ms = [ev_cs[i].elapsed_time(ev_ce[i]) for i in range(K)] if dist_on else [0.0] * K
    mine = torch.tensor([sum(step_ms), statistics.mean(proj_ms), statistics.mean(vls_ms), statistics.mean(comm_ms),
                         statistics.mean(step_ms)], dtype=torch.float64, device=dev)
    if dist_on:
        allr = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(allr, mine)
        per_rank = [x.tolist() for x in allr]
    else:
        per_rank = [mine.tolist()]
    total_ms_max = max(r[0] for r in per_rank)
    launches_per_step = pencil.last_launches

    # ---- end to end from pinned host buffers
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    hg, hU, hV, hs, hz = pin(prob.grid), pin(prob.U), pin(prob.V), pin(prob.sigma), pin(prob.z)
    h2d_full = sum(x.numel() * x.element_size() for x in (hg, hU, hV, hs, hz))
    Ke = max(2, min(K, 5))
    e_ms = []
    if not dist_on:
        outs = {k: torch.empty(s, dtype=dt).pin_memory() for k, s, dt in
                [("S", (d, m, m), torch.complex128), ("G", (m, m), torch.complex128), ("b", (m,), torch.complex128),
                 ("c", (m,), torch.complex128), ("t", (m, d), torch.float64)]}
        ws_h = pb.alloc_workspace(pb.WS_PENCIL_HOST, d, n, m, dev)
        hctx = pb.HostContext()   # side streams / events created once, not per call
        for _ in range(max(args.warmup, 3)):
            pb.pencil_host(hg, hU, hV, hs, hz, d, n, m, workspace=ws_h, outputs=outs, stream=stream, context=hctx)
        for i in range(Ke):
            flush.fill_(i & 0xFF)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = pb.pencil_host(hg, hU, hV, hs, hz, d, n, m, workspace=ws_h, outputs=outs, stream=stream, context=hctx)
            e1.record(stream)
            e1.synchronize()
            assert r["status"] == 0
            e_ms.append(e0.elapsed_time(e1))
        d2h = sum(x.numel() * x.element_size() for x in outs.values() if isinstance(x, torch.Tensor)) + 4
        h2d_rank = [h2d_full]
        api = "prony_pencil_host_ctx (C ABI, pinned host buffers, one prony_host_context)"
        hctx.close()
        del ws_h
    else:
        hS = torch.empty((d, m, m), dtype=torch.complex128).pin_memory()
        hc = torch.empty(m, dtype=torch.complex128).pin_memory()
        ht = torch.empty((m, d), dtype=torch.float64).pin_memory()
        h2d_rank = [sharding.h2d_bytes(d, n, m, world, r, order, scatter_v=True) for r in range(world)]

        def e2e_step():
            Sx, cx, tx = pencil.from_host(hg, hU, hV, hs, hz, stream=stream, scatter_v=True)
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
        api = ("sharding.DistributedPencil.from_host (per rank: pinned H2D of the grid, its 1/N slice of V and its "
               "U rows; all_gather of V over the device interconnect; pencil; all-reduce; D2H of S, c, t on rank 0)")
    te = torch.tensor([sum(e_ms)], dtype=torch.float64, device=dev)
    if dist_on:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = {"value": Ke / (float(te[0]) * 1e-3), "unit": UNIT, "h2d_bytes_per_step": sum(h2d_rank),
           "h2d_bytes_per_rank": h2d_rank, "d2h_bytes_per_step": d2h, "ms_per_step": float(te[0]) / Ke, "api": api}

    peak = peak_clk = None
    if rank == 0:
        peak, peak_clk = zgemm_peak_tflops(torch, local)

    if rank == 0:
        value = K / (total_ms_max * 1e-3)   # one pencil per step, sharded over the ranks
        ms_per_step = total_ms_max / K
        cm = 1.0 if os.environ.get("PRONY_CMUL", "3m").startswith("4") else 0.75
        # complex MACs of the pencil as this implementation computes it (per rank: k_project's product over
        # its E rows; the reduce U^* Y over those rows for every l; the LS products over its columns)
        cmac_proj = pencil.last_main_flops / 8.0
        rows = cmac_proj / (m * N)
        cmac_step = cmac_proj + d * m * m * rows + m * m * N / world + m * N / world
        real_per_cmac = 8.0 * cm                         # 3M: 3 real products = 6 real flops per complex MAC
        proj_avg_s = statistics.mean(proj_ms) * 1e-3
        achieved = real_per_cmac * cmac_proj / proj_avg_s / 1e12
        # DMMA work actually issued per k-step and 16-row tile, in real products: 3 per full 8-column n-tile
        # (3M), 2 for a last n-tile with <= 4 valid columns (packed, DESIGN.md v9), 3 otherwise; the useful
        # work is 3 m / 8 (4M: 4 per tile, 4 m / 8)
        ntile, w = (m + 7) // 8, m % 8
        if cm == 1.0:
            issued, useful = 4.0 * ntile, 4.0 * m / 8.0
        else:
            issued, useful = 3.0 * (ntile - 1) + (2.0 if 0 < w <= 4 else 3.0), 3.0 * m / 8.0
        executed = achieved * issued / useful
        traffic, traffic_src = stamped_traffic()
        tflops = real_per_cmac * cmac_step * world * value / 1e12
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",  # one pencil per step at every N
            "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded planted exponential sum, complex Gaussian noise 1e-6)",
            "config": {"workload": f"{c.name}: d={d} n={n} N={N} m={m} noise={c.noise} (BASELINE configs[{int(c.name[3:]) - 1}])",
                       "d": d, "n": n, "N": N, "m": m, "parallelism": f"dp{world} ({['l-major', 'row-major', 'shared'][order]} units)",
                       "l2": "flushed (256 MiB write) before every timed step, outside the timed interval",
                       "pencils_per_step": 1,
                       "comm": "1 x all_reduce(SUM) of packed [S,G,b] per step" if dist_on else "none",
                       "dist_backend": args.dist_backend if dist_on else None},
            # physical rates: real FP64 flops the implementation executes per pencil (3M products) / time
            "tflops": tflops,
            "pct_peak": tflops / (peak * world) if peak else None,
            "paper_equivalent_tflops": paper_pencil_flops(d, N, m) * value / 1e12,
            "flop_accounting": ("tflops = real FP64 flops executed per pencil / step time: complex MACs of the "
                                "shared-row product T_E V ((n+2)^d rows, DESIGN.md F8) + U^*Y for every l + the LS "
                                "products, x6 real flops per complex MAC (3M); pct_peak = tflops / (measured ZGEMM "
                                "x N GPUs), a fraction. paper_equivalent_tflops = the paper's d separate ZGEMM-"
                                "convention products (SURVEY §8(d) F) per second: not a hardware rate."),
            "roofline": {"bound": "tensor", "kernel": "k_project (complex FP64 DMMA, implicit Toeplitz gather)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "algorithmic_flops_per_launch": real_per_cmac * cmac_proj,
                         "flops_definition": ("6 real flops per complex MAC (3M: 3 real DMMA products) x m N rows; "
                                              "the ZGEMM convention (8 per complex MAC) is achieved_zgemm_convention"),
                         "achieved_zgemm_convention": 8.0 * cmac_proj / proj_avg_s / 1e12,
                         "executed_tflops": executed, "executed_frac": executed / peak if peak else None,
                         "peak_source": ("cuBLAS ZGEMM 4096^3 complex128 measured in this run, best of 40 (real FP64 "
                                         "flop/s; MEASURED_PEAKS.json has no FP64 entry)"),
                         "peak_clocks": peak_clk, "frac_of": "measured",
                         "planning_peak": 37.2, "frac_vs_planning": achieved / 37.2,
                         "avg_launch_ms": proj_avg_s * 1e3, "cmul": "4M" if cm == 1.0 else "3M",
                         "share_of_step": sum(proj_ms) / sum(step_ms),
                         "grid": pencil.last_grid, "split_k": pencil.last_split_k},
            "kernels_ms": {"k_project": statistics.mean(proj_ms), "k_vls": statistics.mean(vls_ms),
                           "outside_k_project": statistics.mean(step_ms) - statistics.mean(proj_ms),
                           "note": "k_vls = the event interval around k_vls on the LS side stream, released right "
                                   "before k_project: its CTAs wait for the SMs k_project's last wave leaves idle, "
                                   "so the interval spans that wait (its own run time is ~0.13 ms at cfg4)"},
            "per_rank": [{"rank": r, "step_ms": x[4], "k_project_ms": x[1], "k_vls_ms": x[2], "allreduce_ms": x[3]}
                         for r, x in enumerate(per_rank)],
            "gpu_launches": launches_per_step * K,
            "clocks": clk,
            "e2e": e2e,
        }
        if world == 1 and not args.no_other_configs and c.name == "cfg4":
            try:  # informational: never let it cost the headline line
                line["other_configs"] = other_configs([k for k in ("cfg2", "cfg3", "cfg5") if k in W.CONFIGS], dev,
                                                      peak)
            except Exception as exc:  # noqa: BLE001
                line["other_configs"] = {"error": f"{type(exc).__name__}: {exc}"}
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(prob)
        print(json.dumps(line), flush=True)
    if dist_on:
        dist.barrier()
        dist.destroy_process_group()


def relaunch_under_torchrun(args_argv, gpus):
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-exec as an N-rank torchrun job on this node."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *args_argv]
    os.execv(sys.executable, cmd)


def build_locked():
    """Build libprony.so once per node: every rank takes the same file lock; the first builds, the others
    find the library fresh (no concurrent nvcc into the same objects)."""
    from paper_2012_11430_b200 import _build
    import oracle
    lock = os.path.join(ROOT, "paper_2012_11430_b200", ".build.lock")
    with open(lock, "w") as f:
        fcntl.flock(f, fcntl.LOCK_EX)
        _build.build()
        oracle.build()
        fcntl.flock(f, fcntl.LOCK_UN)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cfg", default="cfg4", choices=sorted(W.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the cfg2/cfg3/cfg5 device timings attached to the cfg4 line at N = 1")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--cmul", choices=["3m", "4m"], default=None,
                    help="complex products of the DMMA engine: 3M (Gauss, default) or 4M (sets PRONY_CMUL)")
    ap.add_argument("--force-dist", action="store_true",
                    help="test hook: run the N > 1 path (process group + collectives) even with one rank")
    ap.add_argument("--units", default="shared", choices=["shared", "l-major", "row-major"],
                    help="prony_unit_order of the projection (shared: one extended product for all l, F8)")
    args = ap.parse_args()
    if args.cmul:
        os.environ["PRONY_CMUL"] = args.cmul  # read by the library at each launch (and by torchrun children)
    if args.warmup < 3:
        args.warmup = 3
    cfg = W.CONFIGS[args.cfg]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(sys.argv[1:], args.gpus)
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        run_reference(args, cfg)
        return
    if args.gpus > 1 and args.dist_backend == "nccl":
        # the NCCL INIT log (ranks, channels, NVLS) on stderr, for the driver's rank check
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    build_locked()
    run_ours(args, cfg)


if __name__ == "__main__":
    main()
