"""Summarize an ncu --metrics gpu__time_duration.sum launch list (CSV): per-kernel count/total/share."""
import csv
import sys


def main(path, skip_foreign=False):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot, cnt = {}, {}
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        if skip_foreign and not name.startswith("prony::"):
            continue
        v = float(r[vi].replace(",", ""))
        tot[name] = tot.get(name, 0) + v
        cnt[name] = cnt.get(name, 0) + 1
    s = sum(tot.values())
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k[:48]:48s} n={cnt[k]:4d} avg={tot[k] / cnt[k] / 1e3:10.3f} us share={100 * tot[k] / s:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], "--prony" in sys.argv)
