#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into per-kernel totals:

    python profiles/launch_summary.py gpurun_out/launches_128k.csv profiles/r01_launches_128k.json "what"

ncu serialises launches and runs them cold-cache, so compare SHARES, not absolute times."""
import csv
import json
import sys


def main(src, out, what):
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    h = rows[0]
    ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    k = {}
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].replace("(anonymous namespace)::", "")[:60]
        v = float(r[iv].replace(",", ""))
        e = k.setdefault(name, {"launches": 0, "total_ms": 0.0})
        e["launches"] += 1
        unit = r[h.index("Metric Unit")]
        e["total_ms"] += v * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3}.get(unit, 1.0)
    tot = sum(e["total_ms"] for e in k.values())
    for e in k.values():
        e["total_ms"] = round(e["total_ms"], 3)
        e["share"] = round(e["total_ms"] / tot, 4)
    res = {"what": what, "kernels": dict(sorted(k.items(), key=lambda x: -x[1]["total_ms"])), "total_ms": round(tot, 3)}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
