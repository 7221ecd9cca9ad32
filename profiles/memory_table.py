#!/usr/bin/env python
"""Per-rank chunk-buffer memory of the UPipe layer at the BASELINE configs' CP degrees, from the library's own
workspace planner (upipe_workspace_size; host-only, no GPU needed):

    python profiles/memory_table.py > profiles/r02_memory_table.txt

For each shape: the forward and backward workspace of UPipe (U) and of chunk = all-heads Ulysses (U = Hq) in
the overlapped schedule (pass 0/1, the default for C > 1), the sequential one (pass 2/3, the paper's single
buffer set) and the direct-to-peer one (pass 4/5: receive buffers only). "chunk" = the
backward workspace minus the U-independent pre-allocated gradient buffer (DESIGN A21, A30). The reduction is
1 - UPipe / Ulysses; the paper's target is 1 - U/H, which the Q path meets exactly and the K/V
path cannot go below one KV head per device under GQA (DESIGN A22)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_21196_b200 import upipe as U  # noqa: E402

GiB = 2.0 ** 30
SHAPES = [  # (name, S, Hq, Hkv, d, D, C, U)
    ("Llama3-8B 128K", 131072, 32, 8, 128, 4096, 8, 8),
    ("Llama3-8B 128K", 131072, 32, 8, 128, 4096, 8, 16),
    ("Llama3-8B 1M", 1048576, 32, 8, 128, 4096, 1, 8),
    ("Llama3-8B 1M", 1048576, 32, 8, 128, 4096, 2, 8),
    ("Llama3-8B 1M", 1048576, 32, 8, 128, 4096, 4, 8),
    ("Llama3-8B 1M", 1048576, 32, 8, 128, 4096, 8, 8),
    ("Llama3-8B 5M", 5242880, 32, 8, 128, 4096, 8, 8),
    ("32B-class 1M", 1048576, 64, 8, 128, 5120, 8, 8),
    ("MHA control 1M", 1048576, 32, 32, 128, 4096, 8, 8),
]


def ws(C, S_l, Hq, Hkv, d, D, Uc, p):
    return U.upipe_workspace_size(C, U.make_shape(S_l, D, Hq, Hkv, d, Uc), p)


print(f"{'shape':16s} {'C':>2s} {'U':>3s} | {'schedule':10s} | {'UPipe fwd':>9s} {'bwd':>8s} {'chunk':>8s} | "
      f"{'Ulysses fwd':>11s} {'bwd':>8s} {'chunk':>8s} | {'reduction':>9s} {'1-U/H':>6s}   (GiB per rank)")
for name, S, Hq, Hkv, d, D, C, Uc in SHAPES:
    S_l = S // C
    for sched, (pf, pb) in (("overlap", (0, 1)), ("sequential", (2, 3)), ("direct", (4, 5))):
        if C == 1 and sched != "sequential":
            continue
        # pre-allocated gradient buffer (DESIGN A30) or, where that would be larger, the fp32 dX accumulator:
        # U-independent either way
        g = S_l * min((Hq + 2 * Hkv) * d * 2, D * 4)
        up = [ws(C, S_l, Hq, Hkv, d, D, Uc, p) for p in (pf, pb)]
        ul = [ws(C, S_l, Hq, Hkv, d, D, Hq, p) for p in (pf, pb)]
        up_chunk = max(up[0], up[1] - (g if Hq // Uc > 1 else 0))
        ul_chunk = max(ul[0], ul[1])                # one stage: no gradient buffer
        print(f"{name:16s} {C:2d} {Uc:3d} | {sched:10s} | {up[0] / GiB:9.2f} {up[1] / GiB:8.2f} {up_chunk / GiB:8.2f} | "
              f"{ul[0] / GiB:11.2f} {ul[1] / GiB:8.2f} {ul_chunk / GiB:8.2f} | {1 - up_chunk / ul_chunk:9.3f} "
              f"{1 - Uc / Hq:6.3f}")
