#!/usr/bin/env python
"""Warp-stall samples of one kernel in an .ncu-rep, aggregated by CUDA source line.

    python profiles/ncu_lines.py REPORT.ncu-rep OBJECT.o KERNEL_SUBSTRING [N]

The SASS page of the report carries absolute addresses; the line table comes from
`nvdisasm -g` of the same build's cubin (extracted from OBJECT.o), so the object
must be the one that was profiled.
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main(rep, obj, kname, n=30):
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True, check=True).stdout
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, capture_output=True, check=True)
        cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
        dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(td, cub)], capture_output=True, text=True,
                             check=True).stdout.split("\n")
    start = [i for i, l in enumerate(dis) if kname in l and "----" in l][0]
    amap, loc = {}, "?"
    for l in dis[start + 1:]:
        if "----" in l and ".text." in l:
            break
        m = re.search(r'//## File ".*/([\w.]+)", line (\d+)', l)
        if m:
            loc = f"{m.group(1)}:{m.group(2)}"
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            amap[int(m.group(1), 16)] = (loc, m.group(2).strip()[:48])
    rows = list(csv.reader(io.StringIO(sass)))
    h = rows[1]
    ia, isamp = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
    cols = {c: h.index(c) for c in h if c.startswith("stall_") and "Not Issued" not in c}
    base = int(rows[2][ia], 16)
    agg, tot = {}, 0.0
    for r in rows[2:]:
        try:
            a = int(r[ia], 16) - base
        except ValueError:
            continue
        s = float(r[isamp] or 0)
        tot += s
        loc_, ins = amap.get(a, ("?", "?"))
        d = agg.setdefault(loc_, {"n": 0.0, "ins": ins})
        d["n"] += s
        for c, i in cols.items():
            d[c] = d.get(c, 0.0) + float(r[i] or 0)
    print(f"total samples {tot:.0f}")
    for loc_, d in sorted(agg.items(), key=lambda x: -x[1]["n"])[:n]:
        top = sorted(((v, c) for c, v in d.items() if c.startswith("stall_")), reverse=True)[:3]
        print(f"{d['n'] / tot * 100:5.1f}% {loc_:20s} {d['ins']:48s}",
              " ".join(f"{c[6:]}={v / max(d['n'], 1) * 100:.0f}%" for v, c in top))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 30)


def instr_by_pipe(rep, obj, kname):
    """Executed warp-instructions of one kernel, by SASS opcode (for issue-slot budgets)."""
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(sass)))
    h = rows[1]
    isrc, iex = h.index("Source"), h.index("Instructions Executed")
    ops = {}
    for r in rows[2:]:
        try:
            n = float(r[iex] or 0)
        except ValueError:
            continue
        op = r[isrc].strip().split()
        if not op:
            continue
        o = op[0] if not op[0].startswith("@") else op[1]
        o = o.split(".")[0]
        ops[o] = ops.get(o, 0) + n
    return ops
