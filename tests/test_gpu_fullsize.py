"""Parity at BASELINE.json's full size, in the launch configuration bench.py times at N=1:
Llama3-8B attention layer (32 Q / 8 KV heads, d=128, hidden 4096), S = 131072 tokens,
C = 1, U = 8, inputs drawn on the device by the same seeded generator. The fp64 oracle
cannot run the whole layer at this size, so it computes sampled outputs one by one
(oracle.layer_fwd_rows: y / O / lse of chosen query rows, spread over tiles and the
ends of the sequence; oracle.layer_bwd_tail: dX of the last w tokens, which a causal
layer determines from the tail rows alone). Bar: the north_star tolerance."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import assert_close, dev, to_np

pytestmark = pytest.mark.gpu

S, D, Hq, Hkv, d, U = 131072, 4096, 32, 8, 128, 8
ROWS = np.array([0, 1, 127, 128, 129, 4095, 65535, 65536, 100003, 131071])
TAIL = 24
REL, ABS = 5e-3, 2e-2


@pytest.mark.parametrize("rope_base", [0.0, 500000.0])
def test_fullsize_bench_workload_sampled_rows(rope_base):
    # rope_base 500000 (Llama3): rotary angles at positions up to 131071 (DESIGN A26)
    from paper_2602_21196_b200 import UPipeAttention, upipe
    e = synth.layer_exponents(D, Hq, d, S)

    def fill(shape, name):
        t = torch.empty(shape, dtype=torch.bfloat16, device=dev())
        upipe.upipe_synth_fill_bf16(t, t.numel(), 0, synth.TID[name], e[name], 0)
        return t

    x, dy = fill((S, D), "x"), fill((S, D), "dy")
    W = [fill((Hq * d, D), "wq"), fill((Hkv * d, D), "wk"), fill((Hkv * d, D), "wv"), fill((D, Hq * d), "wo")]
    attn = UPipeAttention(Hq, Hkv, d, D, U, rope_base=rope_base)
    y, saved = attn.forward(x, *W)
    dx, *_ = attn.backward(x, *W, dy, saved)
    torch.cuda.synchronize()
    y_s = to_np(y[ROWS.tolist()])
    o_s = to_np(saved[0][ROWS.tolist()])
    lse_s = to_np(saved[1][:, ROWS.tolist()])
    dx_t = to_np(dx[S - TAIL:])
    attn.close()
    del x, dy, y, saved, dx, W
    torch.cuda.empty_cache()

    # ---- oracle, fp64 on the host, from the same generator
    wq = synth.draw(0, synth.TID["wq"], (Hq * d, D), e["wq"])
    wk = synth.draw(0, synth.TID["wk"], (Hkv * d, D), e["wk"])
    wv = synth.draw(0, synth.TID["wv"], (Hkv * d, D), e["wv"])
    wo = synth.draw(0, synth.TID["wo"], (D, Hq * d), e["wo"])
    K = np.empty((S, Hkv * d))
    V = np.empty((S, Hkv * d))
    chunk = 8192
    for t0 in range(0, S, chunk):
        xc = synth.draw(0, synth.TID["x"], (chunk, D), e["x"], start=t0 * D)
        K[t0:t0 + chunk] = oracle.project(xc, wk)
        V[t0:t0 + chunk] = oracle.project(xc, wv)
    K = K.reshape(S, Hkv, d)
    V = V.reshape(S, Hkv, d)
    rb = rope_base or None
    if rb:
        K = oracle.rope(K, np.arange(S), rb)
    x_rows = synth.draw_rows(0, synth.TID["x"], D, ROWS, e["x"])
    Y, Oo, L = oracle.layer_fwd_rows(x_rows, ROWS, K, V, wq, wo, Hq, Hkv, d, rope_base=rb)
    assert_close("y rows", y_s, Y, REL, ABS)
    assert_close("o_saved rows", o_s, Oo, REL, ABS)
    # C = 1, U = 8: lse slot s*8 + j holds head 8 s + j, i.e. slot == head (upipe.h, DESIGN A8)
    sh = upipe.make_shape(S, D, Hq, Hkv, d, U)
    order = [upipe.upipe_plan_stage(1, sh, s, 0).q0 + j for s in range(Hq // U) for j in range(U)]
    assert_close("lse rows", lse_s, L[order], REL, ABS)
    x_tail = synth.draw(0, synth.TID["x"], (TAIL, D), e["x"], start=(S - TAIL) * D)
    dy_tail = synth.draw(0, synth.TID["dy"], (TAIL, D), e["dy"], start=(S - TAIL) * D)
    dX = oracle.layer_bwd_tail(x_tail, dy_tail, K, V, wq, wk, wv, wo, Hq, Hkv, d, rope_base=rb)
    assert_close("dx tail rows", dx_t, dX, REL, ABS)


@pytest.mark.timeout(3600)
@pytest.mark.parametrize("nq,nkv", [(8, 2), (1, 1)])
def test_attn_core_32k_full_tensor(nq, nkv):
    # Full-tensor elementwise attention parity at S = 32K (the oracle's BLAS-backed blocks finish in
    # minutes): the bench's per-stage launch shape at CP 1 (8 Q / 2 KV heads of the stage, d 128) and the
    # CP 8 per-rank shape (1 / 1), forward and the 64-query backward with the dim-major dQ accumulator
    # (the layer's configuration), every element of O, LSE, dQ, dK, dV against the fp64 oracle.
    from paper_2602_21196_b200 import upipe
    S, d = 32768, 128
    c = synth.core_inputs(0, S, nq, nkv, d, 1.0)
    from gpu_util import to_bf16
    q, k, v, do = (to_bf16(c[n]) for n in ("q", "k", "v", "do"))
    o = torch.empty((S, nq, d), dtype=torch.bfloat16, device=dev())
    lse = torch.empty((nq, S), dtype=torch.float32, device=dev())
    upipe.upipe_attn_core_fwd(q, k, v, o, lse, S, nq, nkv, d, 1, nq * d, nkv * d, nq * d, S)
    delta = torch.empty((S, nq), dtype=torch.float32, device=dev())
    upipe.upipe_rowdot(do, nq * d, o, nq * d, delta, nq, S, nq, d)
    dq = torch.zeros((nq * d, S), dtype=torch.float32, device=dev())
    dk = torch.empty((S, nkv, d), dtype=torch.float32, device=dev())
    dv = torch.empty((S, nkv, d), dtype=torch.float32, device=dev())
    upipe.upipe_attn_core_bwd(q, k, v, do, lse, delta, dq, dk, dv, S, nq, nkv, d, 1, nq * d, nkv * d, nq * d, S, nq,
                              dq_dim_major=True)
    torch.cuda.synchronize()
    o_np, lse_np = to_np(o), to_np(lse)
    dq_np = to_np(dq.reshape(nq, d, S).permute(2, 0, 1))
    dk_np, dv_np = to_np(dk), to_np(dv)
    del q, k, v, do, o, lse, delta, dq, dk, dv
    torch.cuda.empty_cache()
    O, L = oracle.attn_fwd(c["q"], c["k"], c["v"], causal=True)
    assert_close("O 32K", o_np, O, 3e-3, ABS)
    assert_close("lse 32K", lse_np, L, 1e-4, 2e-4)
    dQ, dK, dV = oracle.attn_bwd(c["q"], c["k"], c["v"], c["do"], causal=True)
    assert_close("dV 32K", dv_np, dV, 3e-3, ABS)
    assert_close("dQ 32K", dq_np, dQ, 4e-3, ABS)
    assert_close("dK 32K", dk_np, dK, 4e-3, ABS)
