#!/usr/bin/env python
"""Per-role cycle breakdown of the attention-backward kernel (CTA (0,0), the longest one):
runs upipe_attn_core_bwd once with UPIPE_BWD_TIMELINE=1 (the library prints the
clock64 accumulators to stderr) and times the launch with CUDA events.

    python profiles/bwd_timeline.py [S] [nq] [nkv] [d]
"""
import os
import sys

os.environ.setdefault("UPIPE_BWD_TIMELINE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_21196_b200 import upipe  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 8
nkv = int(sys.argv[3]) if len(sys.argv) > 3 else 2
d = int(sys.argv[4]) if len(sys.argv) > 4 else 128
dev = torch.device("cuda", 0)


def fill(shape, tid, e):
    t = torch.empty(shape, dtype=torch.bfloat16, device=dev)
    upipe.upipe_synth_fill_bf16(t, t.numel(), 0, tid, e)
    return t


q, k, v, do = fill((S, nq, d), 11, 0), fill((S, nkv, d), 12, 0), fill((S, nkv, d), 13, 0), fill((S, nq, d), 14, 0)
o = torch.empty((S, nq, d), dtype=torch.bfloat16, device=dev)
lse = torch.empty((nq, S), dtype=torch.float32, device=dev)
upipe.upipe_attn_core_fwd(q, k, v, o, lse, S, nq, nkv, d, 1, nq * d, nkv * d, nq * d, S)
delta = torch.empty((S, nq), dtype=torch.float32, device=dev)
upipe.upipe_rowdot(do, nq * d, o, nq * d, delta, nq, S, nq, d)
dq = torch.zeros((S, nq, d), dtype=torch.float32, device=dev)
dk = torch.empty((S, nkv, d), dtype=torch.float32, device=dev)
dv = torch.empty((S, nkv, d), dtype=torch.float32, device=dev)
args = (q, k, v, do, lse, delta, dq, dk, dv, S, nq, nkv, d, 1, nq * d, nkv * d, nq * d, S, nq)
upipe.upipe_attn_core_bwd(*args)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
upipe.upipe_attn_core_bwd(*args)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
pairs = S * (S + 1) // 2
print(f"S={S} nq={nq} nkv={nkv} d={d}: {ms:.3f} ms, {10 * d * pairs * nq / ms / 1e9:.1f} TFLOP/s")
