#!/usr/bin/env python
"""Summarise an `ncu --set full` report (.ncu-rep) into the JSON kept under profiles/.

    python profiles/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_attn_bwd_v3_32k.json "note"

Extracts, per profiled launch: duration, DRAM bytes (read+write = the `traffic`
of bench.py's roofline object), L2 bytes, tensor-pipe / issue / pipe utilisation,
occupancy and registers, plus the top stall reasons from the source page.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__cycles_elapsed.avg.per_second", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__cycles_active.avg", "sm__cycles_elapsed.avg",
]


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True, check=True).stdout


def main(rep, out, note=""):
    raw = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    hdr, units, rows = raw[0], raw[1], raw[2:]
    launches = []
    for r in rows:
        d = {"kernel": r[hdr.index("Kernel Name")][:120]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = {"value": r[i], "unit": units[i]}
        launches.append(d)
    src = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    stalls = {}
    if len(src) > 2:
        h = src[1]
        cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
        tot = 0.0
        for r in src[2:]:
            for i in cols:
                try:
                    v = float(r[i] or 0) if i < len(r) else 0.0
                except ValueError:       # header rows of the next kernel's section
                    v = 0.0
                stalls[h[i]] = stalls.get(h[i], 0.0) + v
                tot += v
        stalls = {k: round(v / tot, 4) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:10]} if tot else {}
    json.dump({"report": rep, "note": note, "launches": launches, "stall_share_top10": stalls}, open(out, "w"), indent=1)
    print(json.dumps(launches[0], indent=1)[:2000])
    print(stalls)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
