#!/usr/bin/env python
"""Times the attention core kernels alone (CUDA events, median of N launches) through the C ABI:

    python profiles/attn_time.py [S] [nq] [nkv] [d] [reps]

Prints fwd / bwd milliseconds and TFLOP/s (4*d resp. 10*d flops per causal (query, key) pair
per head). Inputs come from the seeded device generator (synth stream ids 11..14)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_21196_b200 import upipe  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 8
nkv = int(sys.argv[3]) if len(sys.argv) > 3 else 2
d = int(sys.argv[4]) if len(sys.argv) > 4 else 128
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
dev = torch.device("cuda", 0)


def fill(shape, tid):
    t = torch.empty(shape, dtype=torch.bfloat16, device=dev)
    upipe.upipe_synth_fill_bf16(t, t.numel(), 0, tid, 0)
    return t


q, k, v, do = fill((S, nq, d), 11), fill((S, nkv, d), 12), fill((S, nkv, d), 13), fill((S, nq, d), 14)
o = torch.empty((S, nq, d), dtype=torch.bfloat16, device=dev)
lse = torch.empty((nq, S), dtype=torch.float32, device=dev)
delta = torch.empty((S, nq), dtype=torch.float32, device=dev)
dq = torch.zeros((S, nq, d), dtype=torch.float32, device=dev)
dk = torch.empty((S, nkv, d), dtype=torch.float32, device=dev)
dv = torch.empty((S, nkv, d), dtype=torch.float32, device=dev)


def fwd():
    upipe.upipe_attn_core_fwd(q, k, v, o, lse, S, nq, nkv, d, 1, nq * d, nkv * d, nq * d, S)


def bwd():
    upipe.upipe_attn_core_bwd(q, k, v, do, lse, delta, dq, dk, dv, S, nq, nkv, d, 1, nq * d, nkv * d, nq * d, S, nq)


def timed(f):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


fwd()
upipe.upipe_rowdot(do, nq * d, o, nq * d, delta, nq, S, nq, d)
pairs = S * (S + 1) // 2
tf, tb = timed(fwd), timed(bwd)
print(f"S={S} nq={nq} nkv={nkv} d={d}: fwd {tf:.3f} ms {4 * d * pairs * nq / tf / 1e9:.1f} TFLOP/s | "
      f"bwd {tb:.3f} ms {10 * d * pairs * nq / tb / 1e9:.1f} TFLOP/s")
