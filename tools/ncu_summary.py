"""Summarize an ncu --set full report: key metrics, stall breakdown, top stall instructions."""
import csv
import io
import json
import subprocess
import sys


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, out_json=None, top=12, stamp=False):
    raw = ncu_csv(rep, "--page", "raw")
    hdr, vals = raw[0], raw[2]
    g = dict(zip(hdr, vals))
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "l1tex__t_bytes.sum", "lts__t_bytes.sum", "smsp__inst_executed.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__shared_mem_per_block_dynamic"]
    summ = {k: g.get(k) for k in keys}
    units = dict(zip(hdr, raw[1]))
    stalls = {h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(v)
              for h, v in g.items() if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("ratio")}
    stalls = dict(sorted(((k, v) for k, v in stalls.items() if v > 0.01), key=lambda kv: -kv[1]))
    print(json.dumps({k: f"{v} {units.get(k, '')}" for k, v in summ.items()}, indent=1))
    print("stalls per issued instruction:", json.dumps(stalls))
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    sh, data = src[1], src[2:]
    si = sh.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[si]) for r in data if r[si].isdigit())
    ranked = sorted(data, key=lambda r: -(int(r[si]) if r[si].isdigit() else 0))[:top]
    for r in ranked:
        s = int(r[si])
        print(f"{r[0][-5:]} {100 * s / tot:5.1f}%  {r[1].strip()[:90]}")
    if out_json:
        dur_ns = float(g["gpu__time_duration.sum"])
        rd = float(g["dram__bytes_read.sum"]) * (1e6 if units["dram__bytes_read.sum"] == "Mbyte" else (1e9 if units["dram__bytes_read.sum"] == "Gbyte" else 1))
        wr = float(g["dram__bytes_write.sum"]) * (1e6 if units["dram__bytes_write.sum"] == "Mbyte" else (1e9 if units["dram__bytes_write.sum"] == "Gbyte" else 1))
        extra = {}
        if stamp:
            sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
            import bench
            extra["source_stamp"] = bench.source_stamp()
        json.dump({**extra, "report": rep, "duration_ms": dur_ns / 1e6 if units["gpu__time_duration.sum"] == "ns" else dur_ns,
                   "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
                   "metrics": summ, "stalls_per_issue": stalls}, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    main(args[0], args[1] if len(args) > 1 else None, stamp="--stamp" in sys.argv)
