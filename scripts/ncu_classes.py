"""Per-kernel-class summary of an ncu metrics CSV of one bench step (TP_PROFILE_RANGE=1 capture):
launches, time, share, DRAM bytes per launch, time-weighted tensor-pipe activity, plus the
individual kernels ranked by time. Classes follow bench.py (forward GEMMs = K-major GEMMs before
the last cross-entropy launch, dX after it, dW = MN-major GEMMs).

  python scripts/ncu_classes.py metrics.csv [--traffic profiles/traffic.json] [--md out.md]
"""
import argparse
import collections
import csv
import json
import re


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ID, K, MN, MV, MU = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    ks = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= MV:
            continue
        k = ks.setdefault(int(r[ID]), {"name": re.sub(r"\(.*", "", r[K]).replace("void ", "")
                                       .replace("(anonymous namespace)::", "").replace("unnamed>::", "")})
        v = float(r[MV].replace(",", ""))
        if r[MN] == "gpu__time_duration.sum":
            v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(r[MU], 1)
        if r[MN].startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[MU], 1)
        k[r[MN]] = v
    return list(ks.values())


def cls(i, k, last_ce):
    n = k["name"]
    if "gemm_sm100" in n:
        if re.search(r"<\d+, \d+, (1|true), (1|true)\b", n):
            return "gemm_dw"
        return "gemm_fwd" if i < last_ce else "gemm_dx"
    if "attn_fwd" in n:
        return "attn_fwd"
    if "attn_bwd" in n or "bwd_stage" in n or "dq_convert" in n or "dkv_finalize" in n:
        return "attn_bwd"
    if "ln_" in n:
        return "layernorm"
    if "embed" in n:
        return "embed"
    if "ce_" in n:
        return "cross_entropy"
    return "misc"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--traffic", default="")
    ap.add_argument("--md", default="")
    a = ap.parse_args()
    L = load(a.csv)
    last_ce = max(i for i, k in enumerate(L) if "ce_" in k["name"])
    agg = collections.defaultdict(collections.Counter)
    per = collections.defaultdict(collections.Counter)
    for i, k in enumerate(L):
        c = cls(i, k, last_ce)
        t = k["gpu__time_duration.sum"]
        for d in (agg[c],):
            d["n"] += 1
            d["ns"] += t
            d["dram"] += k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
            d["tp"] += k.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0) * t
        per[k["name"]]["n"] += 1
        per[k["name"]]["ns"] += t
    tot = sum(d["ns"] for d in agg.values())
    out = ["| class | launches | ncu ms | share | DRAM MB / launch | tensor-pipe active % (time-weighted) |",
           "|---|---|---|---|---|---|"]
    for c, d in sorted(agg.items(), key=lambda x: -x[1]["ns"]):
        out.append(f"| {c} | {d['n']} | {d['ns'] / 1e6:.2f} | {100 * d['ns'] / tot:.1f}% | "
                   f"{d['dram'] / d['n'] / 1e6:.1f} | {d['tp'] / d['ns']:.1f} |")
    out += ["", f"{len(L)} launches, {tot / 1e6:.2f} ms (ncu gpu__time_duration, serialised)", "",
            "| kernel | launches | total ms | share | mean us |", "|---|---|---|---|---|"]
    for n, d in sorted(per.items(), key=lambda x: -x[1]["ns"]):
        out.append(f"| `{n[:70]}` | {d['n']} | {d['ns'] / 1e6:.3f} | {100 * d['ns'] / tot:.1f}% | "
                   f"{d['ns'] / d['n'] / 1e3:.1f} |")
    text = "\n".join(out)
    print(text)
    if a.md:
        open(a.md, "w").write(text + "\n")
    if a.traffic:
        json.dump({c: round(d["dram"] / d["n"]) for c, d in agg.items()}, open(a.traffic, "w"), indent=1)


if __name__ == "__main__":
    main()
