#!/usr/bin/env python
"""Small layer runs for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python profiles/sanitize_layer.py [--cp 2]

BASELINE configs[0] (S = 512, 8 Q / 2 KV heads, d = 64, D = 512, U = 2) fwd + bwd at C = 1, or through the
single-process fabric at C = 2 (two host threads, two streams: the stage-buffer reuse across streams of the
overlapped schedule), plus one d = 128 layer (the 64-query backward kernel, dim-major dQ)."""
import argparse
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2602_21196_b200 import UPipeAttention, upipe  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cp", type=int, default=1)
args = ap.parse_args()
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
C = args.cp
for S, D, Hq, Hkv, d, U in ((512, 512, 8, 2, 64, 2), (512, 512, 8, 2, 128, 4)):
    inp = synth.layer_inputs(0, S, D, Hq, Hkv, d)
    t = {k: torch.from_numpy(np.asarray(v, dtype=np.float32)).to(torch.bfloat16).to(dev)
         for k, v in inp.items() if k != "exponents"}
    S_l = S // C
    fabric = upipe.upipe_fabric_create(C) if C > 1 else None
    errors = []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                kw = dict(fabric=fabric, cp_rank=r, cp_size=C) if C > 1 else {}
                attn = UPipeAttention(Hq, Hkv, d, D, U, True, **kw)
                x = t["x"][r * S_l:(r + 1) * S_l].contiguous()
                dy = t["dy"][r * S_l:(r + 1) * S_l].contiguous()
                y, saved = attn.forward(x, t["wq"], t["wk"], t["wv"], t["wo"])
                attn.backward(x, t["wq"], t["wk"], t["wv"], t["wo"], dy, saved)
                stream.synchronize()
                attn.close()
        except Exception as e:  # surfaced below
            errors.append((r, repr(e)))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(C)]
    for h in th:
        h.start()
    for h in th:
        h.join()
    if errors:
        raise SystemExit(f"errors: {errors}")
    print(f"ok S={S} d={d} C={C}", flush=True)
