#!/usr/bin/env python
"""Our GEMM and cuBLAS (torch.matmul) once each on one projection shape, for an ncu capture:

    ncu --set full -k regex:"gemm|nvjet" python profiles/gemm_ncu_run.py [M N K]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_21196_b200 import upipe  # noqa: E402

M, N, K = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (131072, 4096, 4096)
dev = torch.device("cuda", 0)
x = torch.randn(M, K, device=dev).to(torch.bfloat16)
w = torch.randn(N, K, device=dev).to(torch.bfloat16)
y = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
upipe.upipe_gemm_xwT(x, w, y, M, N, K)
z = x @ w.t()
torch.cuda.synchronize()
