#!/usr/bin/env python
"""Our tcgen05 GEMM (upipe_gemm_xwT, y = x W^T, bf16 out) against torch.matmul (cuBLAS) on the
layer's projection shapes; CUDA-event median of 5 launches each.

    python profiles/gemm_time.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_21196_b200 import upipe  # noqa: E402

dev = torch.device("cuda", 0)


def timed(f, reps=5):
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


for M, N, K in ((131072, 1024, 4096), (131072, 4096, 4096), (131072, 4096, 1024), (131072, 256, 4096)):
    x = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
    w = torch.randn(N, K, device=dev, dtype=torch.bfloat16)
    y = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    t_ours = timed(lambda: upipe.upipe_gemm_xwT(x, w, y, M, N, K, 0))
    t_cub = timed(lambda: torch.matmul(x, w.t(), out=y))
    fl = 2.0 * M * N * K
    print(f"M={M} N={N} K={K}: ours {t_ours:.3f} ms {fl / t_ours / 1e9:.0f} TF/s | cuBLAS {t_cub:.3f} ms {fl / t_cub / 1e9:.0f} TF/s")
