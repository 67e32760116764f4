"""Summarise ncu output for profiles/ (run on the CPU host, reading files gpurun brought back).

  python scripts/ncu_summary.py launches <launch-list.csv>        # per-kernel totals and shares
  python scripts/ncu_summary.py full <report.ncu-rep> [regex]      # key metrics per profiled launch
"""
import collections
import csv
import re
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui] if ui is not None else "nsecond"
        v *= {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}.get(unit, 1.0)
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("(anonymous namespace)::", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for _, t in agg.values())
    print(f"| kernel | launches | total ms | share | mean us |\n|---|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k[:80]}` | {n} | {t / 1e6:.3f} | {100 * t / tot:.1f}% | {t / n / 1e3:.1f} |")
    print(f"\n{sum(n for n, _ in agg.values())} launches, {tot / 1e6:.3f} ms (ncu gpu__time_duration, cold-cache, serialised)")


METRICS = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread", "launch__grid_size",
           "sm__warps_active.avg.pct_of_peak_sustained_active"]


def full(path, regex=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    idx = {m: h.index(m) for m in METRICS if m in h}
    print("| kernel | " + " | ".join(f"{m} ({units[idx[m]]})" for m in idx) + " |")
    print("|---" * (len(idx) + 1) + "|")
    for r in rows[2:]:
        name = re.sub(r"\(.*", "", r[h.index("Kernel Name")]).replace("void ", "")
        if regex and not re.search(regex, name):
            continue
        print(f"| `{name[:60]}` | " + " | ".join(r[i] for i in idx.values()) + " |")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
