"""Per-kernel DRAM bytes and durations per launch from ncu CSV captures -> profiles/ncu_traffic.json.

usage: python tools/ncu_traffic.py CONFIG capture.csv [CONFIG capture.csv ...]
Each capture: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--clock-control none --csv --log-file capture.csv python bench.py ... (one config).  Launches are
grouped by kernel class (the bench's profile ids); the per-launch mean over the pass kernels is
stored under "CONFIG:class" (the setup launches of bn_set_tile are excluded from "counts" for
SWAP captures, where the counts kernel never runs inside a pass)."""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_traffic.json")
CLASSES = [("k_gram", "gram"), ("k_lut", "lut"), ("k_decide", "decide"), ("k_finish_gather", "commit"),
           ("k_finish", "commit"), ("k_pass_tail", "tail"), ("k_paper_gather", "gather"), ("k_counts", "counts"),
           ("k_narrow_pack", "pack"), ("k_narrow_range", "range")]


def rows(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.reader(lines[start:]))


def parse(path):
    r = rows(path)
    h = r[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = defaultdict(dict)
    names = {}
    for x in r[1:]:
        try:
            per[x[ii]][x[mi]] = float(x[vi].replace(",", ""))
        except ValueError:
            continue
        names[x[ii]] = x[ki]
    agg = defaultdict(lambda: defaultdict(list))
    for i, m in per.items():
        cls = next((c for pref, c in CLASSES if pref in names[i]), None)
        if cls is None:
            continue
        for k, v in m.items():
            agg[cls][k].append(v)
    return agg


def main():
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    args = sys.argv[1:]
    for cfg, path in zip(args[0::2], args[1::2]):
        for cls, m in parse(path).items():
            rd, wr = m.get("dram__bytes_read.sum", []), m.get("dram__bytes_write.sum", [])
            t = m.get("gpu__time_duration.sum", [])
            if not rd:
                continue
            n = len(rd)
            out[f"{cfg}:{cls}"] = {"dram_bytes_per_launch": (sum(rd) + sum(wr)) / n, "read": sum(rd) / n,
                                   "write": sum(wr) / n, "ncu_us_per_launch": sum(t) / len(t) / 1e3 if t else None,
                                   "launches": n, "source": os.path.relpath(path, ROOT)}
    json.dump(out, open(OUT, "w"), indent=1, sort_keys=True)
    print(json.dumps(out, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()


def summary_md(path):
    """Markdown table of the launch list: per kernel class launches, mean and total ncu time, share."""
    agg = parse(path)
    tot = sum(sum(m.get("gpu__time_duration.sum", [])) for m in agg.values())
    out = ["| kernel class | launches | mean us | total us | share | DRAM MB / launch |", "|---|---|---|---|---|---|"]
    for cls, m in sorted(agg.items(), key=lambda kv: -sum(kv[1].get("gpu__time_duration.sum", []))):
        t = m.get("gpu__time_duration.sum", [])
        if not t:
            continue
        dr = (sum(m.get("dram__bytes_read.sum", [])) + sum(m.get("dram__bytes_write.sum", []))) / len(t) / 1e6
        out.append(f"| {cls} | {len(t)} | {sum(t) / len(t) / 1e3:.1f} | {sum(t) / 1e3:.1f} | {sum(t) / tot:.3f} | {dr:.1f} |")
    return "\n".join(out)
