#!/usr/bin/env python
"""One GPU, C ranks of the single-process fabric (one host thread + stream per rank, all on cuda:0):
runs the layer at a CP-C per-rank shape, so the kernels launch exactly as on rank r of a C-GPU box
(the per-rank GEMM M = S/C, attention over qpd = U/C heads, the unpack of the out all-to-all) -- the
ranks share one GPU, so the step time is NOT a multi-GPU number; use it for ncu captures of the
per-rank launch shapes (e.g. `ncu -k regex:unpack ...`).

    python profiles/fabric_cp8.py [--seq 131072] [--cp 8] [--chunk 8] [--steps 1] [--model llama3-8b|32b]
Inputs are drawn on the device with the library's generator (synth ids)."""
import argparse
import json
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2602_21196_b200 import UPipeAttention, upipe  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=131072)
ap.add_argument("--cp", type=int, default=8)
ap.add_argument("--chunk", type=int, default=8)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--model", default="llama3-8b")
ap.add_argument("--sync", action="store_true")
args = ap.parse_args()
Hq, Hkv, d, D = (32, 8, 128, 4096) if args.model == "llama3-8b" else (64, 8, 128, 5120)
S, C, U = args.seq, args.cp, args.chunk
S_l = S // C
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
e = synth.layer_exponents(D, Hq, d, S, "benign")


def fill(shape, name, start=0):
    t = torch.empty(shape, dtype=torch.bfloat16, device=dev)
    upipe.upipe_synth_fill_bf16(t, t.numel(), 0, synth.TID[name], e[name], start)
    return t


W = [fill((Hq * d, D), "wq"), fill((Hkv * d, D), "wk"), fill((Hkv * d, D), "wv"), fill((D, Hq * d), "wo")]
xs = [fill((S_l, D), "x", r * S_l * D) for r in range(C)]
dys = [fill((S_l, D), "dy", r * S_l * D) for r in range(C)]
torch.cuda.synchronize()
fabric = upipe.upipe_fabric_create(C)
times = [None] * C
errors = []


def rank_main(r):
    try:
        torch.cuda.set_device(0)
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            attn = UPipeAttention(Hq, Hkv, d, D, U, True, fabric=fabric, cp_rank=r, cp_size=C, sync_comm=args.sync)
            ts = []
            for _ in range(args.steps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                y, saved = attn.forward(xs[r], *W)
                attn.backward(xs[r], *W, dys[r], saved)
                e1.record(stream)
                stream.synchronize()
                ts.append(e0.elapsed_time(e1))
            times[r] = ts
            attn.close()
    except Exception as ex:  # surfaced below
        errors.append((r, repr(ex)))


th = [threading.Thread(target=rank_main, args=(r,)) for r in range(C)]
for t in th:
    t.start()
for t in th:
    t.join()
if errors:
    raise SystemExit(f"rank errors: {errors}")
print(json.dumps({"S": S, "C": C, "U": U, "model": args.model, "step_ms_per_rank": times,
                  "note": "C ranks share one GPU: not a multi-GPU timing"}))
