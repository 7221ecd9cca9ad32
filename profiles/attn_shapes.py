#!/usr/bin/env python
"""Times the attention kernels at the per-rank launch shapes of the BASELINE configs, one GPU,
through the C ABI (CUDA events on the launch stream, median of `reps` launches after a warm-up):

    python profiles/attn_shapes.py [--det] [--reps N] [S:nq:nkv ...]

Default shapes (d = 128, causal; the layer's kernel configuration: the 64-query backward with the
dim-major dQ accumulator):
  131072:8:2   CP 1, U 8 (the N = 1 bench launch)        131072:1:1  CP 8, U 8  (qpd 1, kv_res 1)
  131072:2:1   CP 8, U 16                                131072:4:1  CP 8, U 32 (Ulysses)
  1048576:1:1 / 2:1 / 4:1  the same at S = 1M (BASELINE configs[2], CP 8)
One JSON line per shape: fwd / bwd ms and TFLOP/s (4 d resp. 10 d flops per causal pair and head)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_21196_b200 import upipe  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("shapes", nargs="*", default=["131072:8:2", "131072:1:1", "131072:2:1", "131072:4:1",
                                              "1048576:1:1", "1048576:2:1", "1048576:4:1"])
ap.add_argument("--det", action="store_true", help="deterministic dQ order (UPIPE_CORE_DETERMINISTIC)")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--d", type=int, default=128)
args = ap.parse_args()
dev = torch.device("cuda", 0)
d = args.d


def fill(shape, tid):
    t = torch.empty(shape, dtype=torch.bfloat16, device=dev)
    upipe.upipe_synth_fill_bf16(t, t.numel(), 0, tid, 0)
    return t


def timed(f, reps):
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


for spec in args.shapes:
    S, nq, nkv = (int(v) for v in spec.split(":"))
    q, k, v, do = fill((S, nq, d), 11), fill((S, nkv, d), 12), fill((S, nkv, d), 13), fill((S, nq, d), 14)
    o = torch.empty((S, nq, d), dtype=torch.bfloat16, device=dev)
    lse = torch.empty((nq, S), dtype=torch.float32, device=dev)
    delta = torch.empty((S, nq), dtype=torch.float32, device=dev)
    dm = d == 128
    dq = torch.zeros((nq * d, S) if dm else (S, nq, d), dtype=torch.float32, device=dev)
    dk = torch.empty((S, nkv, d), dtype=torch.float32, device=dev)
    dv = torch.empty((S, nkv, d), dtype=torch.float32, device=dev)
    sem = torch.zeros(upipe.upipe_core_bwd_sem_count(S, nq), dtype=torch.int32, device=dev) if args.det else None

    def fwd():
        upipe.upipe_attn_core_fwd(q, k, v, o, lse, S, nq, nkv, d, 1, nq * d, nkv * d, nq * d, S)

    def bwd():
        if sem is not None:
            sem.zero_()
        upipe.upipe_attn_core_bwd(q, k, v, do, lse, delta, dq, dk, dv, S, nq, nkv, d, 1, nq * d, nkv * d, nq * d,
                                  S, nq, dq_dim_major=dm, dq_sem=sem)

    fwd()
    upipe.upipe_rowdot(do, nq * d, o, nq * d, delta, nq, S, nq, d)
    pairs = S * (S + 1) // 2
    tf, tb = timed(fwd, args.reps), timed(bwd, args.reps)
    print(json.dumps({"S": S, "nq": nq, "nkv": nkv, "d": d, "det": args.det,
                      "fwd_ms": tf, "fwd_tflops": 4 * d * pairs * nq / tf / 1e9,
                      "bwd_ms": tb, "bwd_tflops": 10 * d * pairs * nq / tb / 1e9}), flush=True)
    del q, k, v, do, o, lse, delta, dq, dk, dv, sem
    torch.cuda.empty_cache()
