"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum
--csv): count, total and mean time, and share of the listed time.
   python tools/launch_summary.py launches.csv OUT.json [name-filter-substr]"""
import csv
import json
import re
import sys
from collections import defaultdict


def short(name):
    m = re.search(r"(somb::\w+|at::\w+::\w+|\w+_kernel\w*|nccl\w+)", name)
    base = m.group(1) if m else name[:60]
    t = re.search(r"<([^<>]*)>", name)
    return base + (f"<{t.group(1)}>" if t and base.startswith("somb::") else "")


def main():
    path, out = sys.argv[1], sys.argv[2]
    keep = sys.argv[3] if len(sys.argv) > 3 else ""
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum" or keep not in r["Kernel Name"]:
            continue
        k = short(r["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += float(r["Metric Value"].replace(",", "")) / 1e6
    tot = sum(v[1] for v in agg.values())
    res = {"source": path, "total_ms": tot, "kernels": sorted(
        ({"kernel": k, "launches": v[0], "total_ms": round(v[1], 4), "mean_ms": round(v[1] / v[0], 4),
          "share": round(v[1] / tot, 4)} for k, v in agg.items()), key=lambda e: -e["total_ms"])}
    json.dump(res, open(out, "w"), indent=1)
    for e in res["kernels"][:12]:
        print(e)


if __name__ == "__main__":
    main()
