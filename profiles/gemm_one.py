#!/usr/bin/env python
"""One GEMM shape through upipe_gemm_xwT (y = x W^T, bf16), CUDA-event median of 5 launches; with
UPIPE_GEMM_TIMELINE=1|2|3 the library prints CTA 0's wait/issue cycle totals (2: MMA only, 3: TMA only).

    python profiles/gemm_one.py M N K"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_21196_b200 import upipe  # noqa: E402

M, N, K = (int(v) for v in sys.argv[1:4])
dev = torch.device("cuda", 0)
x = torch.randn(M, K, device=dev).to(torch.bfloat16)
w = torch.randn(N, K, device=dev).to(torch.bfloat16)
y = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
upipe.upipe_gemm_xwT(x, w, y, M, N, K)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    upipe.upipe_gemm_xwT(x, w, y, M, N, K)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
t = sorted(ts)[2]
print(f"M={M} N={N} K={K}: {t:.3f} ms {2 * M * N * K / t / 1e9:.0f} TF/s")
