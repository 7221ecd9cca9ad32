"""Pins for the fp64 oracle (-m "not gpu"). Each test pins the oracle to something
other than itself: a worked example from the paper/SPEC (tests/golden), a closed
form, an invariant, an independent library routine (torch fp64 SDPA/autograd),
or finite differences."""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle as O
import synth

RNG = np.random.default_rng(1234)


def rand(*shape, scale=1.0):
    return RNG.standard_normal(shape) * scale


# ---------------------------------------------------------------- projection (DESIGN A4)

def test_project_brute_force_sum():
    # plain definition of nn.Linear without bias: y[i, j] = sum_k x[i, k] W[j, k], summed exactly (fsum)
    X, W = rand(5, 7), rand(3, 7)
    Y = O.project(X, W)
    assert Y.shape == (5, 3)
    for i in range(5):
        for j in range(3):
            assert abs(Y[i, j] - math.fsum(X[i, k] * W[j, k] for k in range(7))) <= 1e-13


def test_project_one_hot_rows_gather_columns_bitwise():
    # W row j = e_{c_j}: output column j is exactly input column c_j (catches a transposed operand
    # or a row/column mix-up; this is also how the GPU layout probes build exact payloads)
    S, D = 6, 9
    cols = [4, 0, 8, 4, 2]
    X = rand(S, D)
    W = np.zeros((len(cols), D))
    W[np.arange(len(cols)), cols] = 1.0
    assert np.array_equal(O.project(X, W), X[:, cols])


def test_project_matches_torch_linear():
    X, W = rand(33, 48), rand(20, 48)
    ref = F.linear(torch.from_numpy(X), torch.from_numpy(W)).numpy()
    np.testing.assert_allclose(O.project(X, W), ref, rtol=0, atol=1e-12)


def test_layer_uses_projection_per_head_rows():
    # head h of Q is X Wq[h d:(h+1) d]^T (DESIGN A4): the layer's O for head h only changes when
    # rows of head h (or its kv head) change
    S, D, Hq, Hkv, d = 16, 12, 4, 2, 3
    X, Wq, Wk, Wv, Wo = rand(S, D), rand(Hq * d, D), rand(Hkv * d, D), rand(Hkv * d, D), rand(D, Hq * d)
    _, O1, _ = O.layer_fwd(X, Wq, Wk, Wv, Wo, Hq, Hkv, d)
    Wq2 = Wq.copy()
    Wq2[2 * d:3 * d] += 1.0                       # rows of q head 2
    _, O2, _ = O.layer_fwd(X, Wq2, Wk, Wv, Wo, Hq, Hkv, d)
    changed = [not np.array_equal(O1[:, h * d:(h + 1) * d], O2[:, h * d:(h + 1) * d]) for h in range(Hq)]
    assert changed == [False, False, True, False]


# ---------------------------------------------------------------- attention fwd

def test_spec_s2_example(golden):
    g = golden("spec_attention_examples.json")["s2_example"]
    Q = np.array(g["Q"])[:, None, :]
    K = np.array(g["K"])[:, None, :]
    V = np.array(g["V"])[:, None, :]
    out, _ = O.attn_fwd(Q, K, V, causal=True)
    np.testing.assert_allclose(out[:, 0, :], np.array(g["out"]), rtol=0, atol=1e-15)


def test_zero_keys_gives_prefix_mean():
    # K all zeros, causal -> out[i] = mean(V[0..i])
    S, H, d = 9, 2, 3
    Q = rand(S, H, d)
    K = np.zeros((S, H, d))
    V = rand(S, H, d)
    out, lse = O.attn_fwd(Q, K, V, causal=True)
    pref = np.cumsum(V, axis=0) / np.arange(1, S + 1)[:, None, None]
    np.testing.assert_allclose(out, pref, atol=1e-14)
    # lse of i+1 equal zero scores = ln(i+1)
    np.testing.assert_allclose(lse, np.log(np.arange(1, S + 1))[None, :].repeat(H, 0), atol=1e-14)


def test_constant_v_yields_v():
    S, Hq, Hkv, d = 17, 4, 2, 5
    Q, K = rand(S, Hq, d, scale=2), rand(S, Hkv, d, scale=2)
    row = rand(1, Hkv, d)
    V = np.repeat(row, S, axis=0)
    out, _ = O.attn_fwd(Q, K, V, causal=True)
    np.testing.assert_allclose(out, np.repeat(V[:, [0, 0, 1, 1], :], 1, 0), atol=1e-13)


@pytest.mark.parametrize("S,Hq,Hkv,d,causal", [(8, 4, 2, 4, True), (37, 8, 2, 16, True),
                                               (64, 4, 4, 8, False), (130, 6, 3, 32, True)])
def test_fwd_matches_torch_sdpa(S, Hq, Hkv, d, causal):
    Q, K, V = rand(S, Hq, d), rand(S, Hkv, d), rand(S, Hkv, d)
    out, lse = O.attn_fwd(Q, K, V, causal=causal)
    tq = torch.from_numpy(Q).permute(1, 0, 2)[None]
    tk = torch.from_numpy(K).permute(1, 0, 2)[None]
    tv = torch.from_numpy(V).permute(1, 0, 2)[None]
    ref = F.scaled_dot_product_attention(tq, tk, tv, is_causal=causal, enable_gqa=True)
    np.testing.assert_allclose(out, ref[0].permute(1, 0, 2).numpy(), atol=1e-12)
    # lse against torch.logsumexp of the masked scores (library routine)
    R = Hq // Hkv
    kk = torch.from_numpy(K).repeat_interleave(R, dim=1)
    s = torch.einsum("ihd,jhd->hij", torch.from_numpy(Q), kk) / math.sqrt(d)
    if causal:
        s = s.masked_fill(torch.triu(torch.ones(S, S, dtype=torch.bool), 1), float("-inf"))
    np.testing.assert_allclose(lse, torch.logsumexp(s, -1).numpy(), atol=1e-12)


def test_softmax_rows_sum_to_one_via_lse():
    S, H, d = 40, 3, 6
    Q, K, V = rand(S, H, d), rand(S, H, d), rand(S, H, d)
    _, lse = O.attn_fwd(Q, K, V, causal=True)
    for h in range(H):
        s = Q[:, h] @ K[:, h].T / math.sqrt(d)
        P = np.exp(s - lse[h][:, None]) * np.tril(np.ones((S, S)))
        np.testing.assert_allclose(P.sum(1), 1.0, atol=1e-12)


def test_gqa_equals_mha_with_repeated_kv():
    S, Hq, Hkv, d = 33, 8, 2, 4
    Q, K, V = rand(S, Hq, d), rand(S, Hkv, d), rand(S, Hkv, d)
    a, la = O.attn_fwd(Q, K, V)
    b, lb = O.attn_fwd(Q, np.repeat(K, 4, axis=1), np.repeat(V, 4, axis=1))
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(la, lb)


def test_causal_perturbation_leaves_earlier_rows_bitwise():
    S, Hq, Hkv, d, t = 50, 4, 2, 8, 31
    Q, K, V = rand(S, Hq, d), rand(S, Hkv, d), rand(S, Hkv, d)
    a, la = O.attn_fwd(Q, K, V)
    K2, V2, Q2 = K.copy(), V.copy(), Q.copy()
    K2[t:] += 5.0
    V2[t:] -= 3.0
    Q2[t:] *= 2.0
    b, lb = O.attn_fwd(Q2, K2, V2)
    np.testing.assert_array_equal(a[:t], b[:t])
    np.testing.assert_array_equal(la[:, :t], lb[:, :t])
    assert np.abs(a[t:] - b[t:]).max() > 1e-3


def test_row_sampled_mode_matches_full():
    S, Hq, Hkv, d = 300, 4, 2, 8
    Q, K, V = rand(S, Hq, d), rand(S, Hkv, d), rand(S, Hkv, d)
    a, la = O.attn_fwd(Q, K, V)
    rows = np.array([0, 5, 127, 128, 299])
    b, lb = O.attn_fwd(Q[rows], K, V, rows=rows)
    np.testing.assert_allclose(b, a[rows], atol=1e-14)
    np.testing.assert_allclose(lb, la[:, rows], atol=1e-14)


def test_head_permutation_equivariance():
    # permuting query heads (with the gqa map) permutes the outputs identically
    S, Hq, Hkv, d = 20, 4, 2, 4
    Q, K, V = rand(S, Hq, d), rand(S, Hkv, d), rand(S, Hkv, d)
    a, _ = O.attn_fwd(Q, K, V)
    perm = [2, 0, 3, 1]
    b, _ = O.attn_fwd(Q[:, perm], K, V, kv_of_head=[p // 2 for p in perm])
    np.testing.assert_allclose(b, a[:, perm], atol=1e-15)


# ---------------------------------------------------------------- attention bwd

def test_spec_s1_backward(golden):
    g = golden("spec_attention_examples.json")["s1_backward"]
    arr = {k: np.array(g[k])[:, None, :] for k in ("Q", "K", "V", "dO")}
    dq, dk, dv = O.attn_bwd(arr["Q"], arr["K"], arr["V"], arr["dO"])
    np.testing.assert_array_equal(dq[:, 0], np.array(g["dQ"]))
    np.testing.assert_array_equal(dk[:, 0], np.array(g["dK"]))
    np.testing.assert_array_equal(dv[:, 0], np.array(g["dV"]))


def test_zero_cotangent_zero_grads():
    S, Hq, Hkv, d = 12, 4, 2, 3
    dq, dk, dv = O.attn_bwd(rand(S, Hq, d), rand(S, Hkv, d), rand(S, Hkv, d), np.zeros((S, Hq, d)))
    assert not dq.any() and not dk.any() and not dv.any()


@pytest.mark.parametrize("S,Hq,Hkv,d,causal", [(6, 2, 1, 3, True), (8, 4, 2, 4, True), (5, 2, 2, 2, False)])
def test_bwd_finite_differences(S, Hq, Hkv, d, causal):
    # central differences, step 1e-5, relative error <= 1e-6
    Q, K, V, G = rand(S, Hq, d), rand(S, Hkv, d), rand(S, Hkv, d), rand(S, Hq, d)
    dq, dk, dv = O.attn_bwd(Q, K, V, G, causal)

    def loss(Q_, K_, V_):
        return float(np.sum(O.attn_fwd(Q_, K_, V_, causal)[0] * G))
    h = 1e-5
    for T, dT, idx in ((Q, dq, 0), (K, dk, 1), (V, dv, 2)):
        num = np.zeros_like(T)
        for i in np.ndindex(T.shape):
            args_p = [Q.copy(), K.copy(), V.copy()]
            args_m = [Q.copy(), K.copy(), V.copy()]
            args_p[idx][i] += h
            args_m[idx][i] -= h
            num[i] = (loss(*args_p) - loss(*args_m)) / (2 * h)
        assert np.linalg.norm(num - dT) <= 1e-6 * max(1e-30, np.linalg.norm(dT))


@pytest.mark.parametrize("S,Hq,Hkv,d", [(50, 4, 2, 8), (129, 8, 2, 16)])
def test_bwd_matches_torch_autograd(S, Hq, Hkv, d):
    Q, K, V, G = rand(S, Hq, d), rand(S, Hkv, d), rand(S, Hkv, d), rand(S, Hq, d)
    dq, dk, dv = O.attn_bwd(Q, K, V, G)
    tq, tk, tv = (torch.from_numpy(a.transpose(1, 0, 2).copy())[None].requires_grad_() for a in (Q, K, V))
    out = F.scaled_dot_product_attention(tq, tk, tv, is_causal=True, enable_gqa=True)
    out.backward(torch.from_numpy(G.transpose(1, 0, 2).copy())[None])
    for mine, t in ((dq, tq), (dk, tk), (dv, tv)):
        np.testing.assert_allclose(mine, t.grad[0].permute(1, 0, 2).numpy(), atol=1e-10)


# ---------------------------------------------------------------- layer

def _torch_layer(X, Wq, Wk, Wv, Wo, Hq, Hkv, d):
    S = X.shape[0]
    q = (X @ Wq.T).view(S, Hq, d).transpose(0, 1)[None]
    k = (X @ Wk.T).view(S, Hkv, d).transpose(0, 1)[None]
    v = (X @ Wv.T).view(S, Hkv, d).transpose(0, 1)[None]
    o = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
    return o[0].transpose(0, 1).reshape(S, Hq * d) @ Wo.T


def test_layer_matches_torch_autograd():
    S, D, Hq, Hkv, d = 70, 24, 4, 2, 6
    X, Wq, Wk, Wv = rand(S, D), rand(Hq * d, D, scale=.3), rand(Hkv * d, D, scale=.3), rand(Hkv * d, D, scale=.3)
    Wo, dY = rand(D, Hq * d, scale=.3), rand(S, D)
    Y, _, _ = O.layer_fwd(X, Wq, Wk, Wv, Wo, Hq, Hkv, d)
    grads = O.layer_bwd(X, Wq, Wk, Wv, Wo, dY, Hq, Hkv, d)
    ts = [torch.from_numpy(a).requires_grad_() for a in (X, Wq, Wk, Wv, Wo)]
    ty = _torch_layer(*ts, Hq, Hkv, d)
    np.testing.assert_allclose(Y, ty.detach().numpy(), atol=1e-11)
    ty.backward(torch.from_numpy(dY))
    for mine, t in zip(grads, ts):
        np.testing.assert_allclose(mine, t.grad.numpy(), atol=1e-10)


def test_layer_finite_differences():
    # closed-form check of every gradient: S=6, Hq=2, Hkv=1, d=3, D=5
    S, D, Hq, Hkv, d = 6, 5, 2, 1, 3
    X, Wq, Wk, Wv, Wo, dY = (rand(S, D), rand(Hq * d, D), rand(Hkv * d, D), rand(Hkv * d, D),
                             rand(D, Hq * d), rand(S, D))
    grads = O.layer_bwd(X, Wq, Wk, Wv, Wo, dY, Hq, Hkv, d)
    args = [X, Wq, Wk, Wv, Wo]
    h = 1e-5

    def loss(a):
        return float(np.sum(O.layer_fwd(*a, Hq, Hkv, d)[0] * dY))
    for idx, g in enumerate(grads):
        num = np.zeros_like(args[idx])
        for i in np.ndindex(num.shape):
            ap = [a.copy() for a in args]
            am = [a.copy() for a in args]
            ap[idx][i] += h
            am[idx][i] -= h
            num[i] = (loss(ap) - loss(am)) / (2 * h)
        assert np.linalg.norm(num - g) <= 1e-6 * np.linalg.norm(g)


# ---------------------------------------------------------------- RoPE (DESIGN A26)

def test_rope_is_complex_rotation():
    # each pair (2i, 2i+1) is the complex number a + ib multiplied by exp(1j * p * base**(-2i/d))
    S, H, d, base = 7, 3, 8, 10000.0
    T = rand(S, H, d)
    pos = np.array([0, 1, 2, 5, 100, 4096, 131071])
    got = O.rope(T, pos, base)
    z = T[..., 0::2] + 1j * T[..., 1::2]
    theta = np.array([base ** (-2.0 * i / d) for i in range(d // 2)])
    w = z * np.exp(1j * pos[:, None, None] * theta[None, None, :])
    np.testing.assert_allclose(got[..., 0::2], w.real, atol=1e-12)
    np.testing.assert_allclose(got[..., 1::2], w.imag, atol=1e-12)


def test_rope_relative_position_norm_identity_inverse():
    d, base = 16, 500000.0
    q, k = rand(1, 1, d), rand(1, 1, d)
    def dot(m, n):
        return float(np.sum(O.rope(q, [m], base) * O.rope(k, [n], base)))
    # q_m . k_n depends on m - n only
    for m, n, t in ((5, 2, 7), (100, 100, 1000), (1 << 20, 3, 12345)):
        assert abs(dot(m, n) - dot(m + t, n + t)) < 1e-9
    T = rand(9, 2, d)
    pos = np.arange(9) * 1000
    R = O.rope(T, pos, base)
    np.testing.assert_allclose(np.linalg.norm(R, axis=-1), np.linalg.norm(T, axis=-1), rtol=1e-12)
    np.testing.assert_allclose(O.rope(T, np.zeros(9), base), T, atol=0)
    np.testing.assert_allclose(O.rope(R, pos, base, inverse=True), T, atol=1e-12)


def test_rope_layer_finite_differences():
    S, D, Hq, Hkv, d, base = 6, 5, 2, 1, 4, 100.0
    X, Wq, Wk, Wv, Wo, dY = (rand(S, D), rand(Hq * d, D), rand(Hkv * d, D), rand(Hkv * d, D),
                             rand(D, Hq * d), rand(S, D))
    grads = O.layer_bwd(X, Wq, Wk, Wv, Wo, dY, Hq, Hkv, d, rope_base=base)
    args = [X, Wq, Wk, Wv, Wo]
    h = 1e-5

    def loss(a):
        return float(np.sum(O.layer_fwd(*a, Hq, Hkv, d, rope_base=base)[0] * dY))
    for idx, g in enumerate(grads):
        num = np.zeros_like(args[idx])
        for i in np.ndindex(num.shape):
            ap = [a.copy() for a in args]
            am = [a.copy() for a in args]
            ap[idx][i] += h
            am[idx][i] -= h
            num[i] = (loss(ap) - loss(am)) / (2 * h)
        assert np.linalg.norm(num - g) <= 1e-6 * np.linalg.norm(g)
    # and RoPE changes the layer (the rotation is not silently skipped)
    assert not np.allclose(O.layer_fwd(X, Wq, Wk, Wv, Wo, Hq, Hkv, d)[0], O.layer_fwd(*args, Hq, Hkv, d, rope_base=base)[0])


def test_output_projection_stage_decomposition():
    # sum over stages of O_s Wo_s^T equals O Wo^T (the accumulated output projection)
    S, D, Hq, d, U = 30, 16, 8, 4, 2
    Oo, Wo = rand(S, Hq * d), rand(D, Hq * d)
    acc = np.zeros((S, D))
    for s in range(Hq // U):
        cols = slice(s * U * d, (s + 1) * U * d)
        acc += Oo[:, cols] @ Wo[:, cols].T
    np.testing.assert_allclose(acc, Oo @ Wo.T, atol=1e-12)


# ---------------------------------------------------------------- schedule / volume

def test_fig4_schedule(golden):
    g = golden("gqa_schedule.json")["fig4_16_4_4"]
    st = O.gqa_schedule(g["Hq"], g["Hkv"], g["C"], g["U"])
    assert st[0].heads == g["stage0_q"]
    assert sorted(k for ks in st[0].kv_sent for k in ks) == g["stage0_kv_sent"]
    assert st[1].heads == g["stage1_q"]
    assert [k for ks in st[1].kv_sent for k in ks] == g["stage1_kv_sent"]


@pytest.mark.parametrize("name", ["llama3_8b", "qwen3_32b"])
def test_model_stage_counts(golden, name):
    g = golden("gqa_schedule.json")[name]
    st = O.gqa_schedule(g["Hq"], g["Hkv"], g["C"], g["U"])
    assert len(st) == g["n_stages"]
    if "kv_sent_stages" in g:
        assert [i for i, s in enumerate(st) if any(s.kv_sent)] == g["kv_sent_stages"]


def test_fig3_layouts(golden):
    g = golden("fig3_ulysses_layout.json")
    u = g["ulysses"]
    st = O.gqa_schedule(u["H"], u["H"], u["C"], u["U"])
    assert len(st) == 1 and st[0].q_heads == u["heads_of_device"]
    p = g["upipe"]
    st = O.gqa_schedule(p["H"], p["H"], p["C"], p["U"])
    assert len(st) == p["n_stages"]
    assert [s.heads for s in st] == p["stage_heads"]
    assert st[0].q_heads[0] == p["device0_stage0"]


def test_comm_volume_formulas(golden):
    for c in golden("gqa_schedule.json")["comm_volume"]["cases"]:
        Hq, Hkv, C = c["Hq"], c["Hkv"], c["C"]
        assert O.comm_volume_formula(Hq, Hkv, C, False) == c["naive"]
        assert O.comm_volume_formula(Hq, Hkv, C, True) == c["scheduled"]
        assert O.comm_volume(O.gqa_schedule(Hq, Hkv, C, C), C) == c["scheduled"]
        assert O.comm_volume(O.naive_schedule(Hq, Hkv, C, C), C) == c["naive"]


GRID = [(Hq, Hkv, C, U) for Hq, Hkv in ((8, 2), (16, 4), (8, 8), (32, 8), (12, 4))
        for C in (1, 2, 4) for U in range(C, Hq + 1, C)
        if Hkv % C == 0 and Hq % U == 0 and ((U // C) % (Hq // Hkv) == 0 or (Hq // Hkv) % (U // C) == 0)]


@pytest.mark.parametrize("Hq,Hkv,C,U", GRID)
def test_schedule_invariants(Hq, Hkv, C, U):
    st = O.gqa_schedule(Hq, Hkv, C, U)
    R = Hq // Hkv
    seen = [h for s in st for h in s.heads]
    assert sorted(seen) == list(range(Hq))                  # each q head exactly once
    assert all(len(s.heads) == U for s in st)
    for s in st:
        for p in range(C):
            assert len(s.q_heads[p]) == U // C
            assert {h // R for h in s.q_heads[p]} <= set(s.kv_heads[p])   # KV resident
    # every kv head transferred exactly once per device set (no re-sends)
    sent = [g for s in st for ks in s.kv_sent for g in ks]
    assert sorted(sent) == list(range(Hkv))
    if R > 1 and C > 1:
        assert O.comm_volume(st, C) < O.comm_volume(O.naive_schedule(Hq, Hkv, C, U), C)


# ---------------------------------------------------------------- a2a maps

def test_a2a_round_trip_and_identity():
    C, Sl, d = 4, 3, 2
    heads = [[0, 1], [2, 3], [4, 5], [6, 7]]
    shards = [{h: rand(Sl, d) for h in range(8)} for _ in range(C)]
    full = O.a2a_seq_to_head(shards, heads)
    assert full[1].shape == (C * Sl, 2, d)
    np.testing.assert_array_equal(full[1][Sl:2 * Sl, 0], shards[1][2])   # rank 1's block, head 2
    back = O.a2a_head_to_seq(full, heads, C)
    for r in range(C):
        for h in range(8):
            np.testing.assert_array_equal(back[r][h], shards[r][h])
    one = O.a2a_seq_to_head([shards[0]], [list(range(8))])
    for h in range(8):
        np.testing.assert_array_equal(one[0][:, h], shards[0][h])


# ---------------------------------------------------------------- sharded sim

SIM = [(Hq, Hkv, C, U) for (Hq, Hkv, C, U) in GRID if Hq <= 16]


@pytest.mark.parametrize("Hq,Hkv,C,U", SIM)
def test_upipe_sim_equals_unsharded(Hq, Hkv, C, U):
    S, D, d = 16, 12, 4
    X, Wq, Wk, Wv = rand(S, D), rand(Hq * d, D, scale=.4), rand(Hkv * d, D, scale=.4), rand(Hkv * d, D, scale=.4)
    Wo, dY = rand(D, Hq * d, scale=.4), rand(S, D)
    Y, Ob, lse = O.layer_fwd(X, Wq, Wk, Wv, Wo, Hq, Hkv, d)
    Y2, Ob2, lse2 = O.upipe_forward(X, Wq, Wk, Wv, Wo, Hq, Hkv, d, C, U)
    np.testing.assert_allclose(Y2, Y, atol=1e-12)
    np.testing.assert_allclose(Ob2, Ob, atol=1e-12)
    np.testing.assert_allclose(lse2, lse, atol=1e-12)
    g1 = O.layer_bwd(X, Wq, Wk, Wv, Wo, dY, Hq, Hkv, d)
    g2 = O.upipe_backward(X, Wq, Wk, Wv, Wo, dY, Hq, Hkv, d, C, U)
    for a, b in zip(g2, g1):
        np.testing.assert_allclose(a, b, atol=1e-11)


# ---------------------------------------------------------------- memory

def test_memory_savings_paper_numbers(golden):
    g = golden("memory_savings.json")["qwen3_32b"]
    S, dh = 1 << 20, 128
    u = O.memory_ulysses_mha(S, g["C"], g["H"], dh)
    p = O.memory_upipe_mha(S, g["C"], g["U"], dh)
    assert u == g["ulysses_coeff_S_dhead"] * S * dh
    assert p == g["upipe_coeff_S_dhead"] * S * dh
    assert 1 - p / u == pytest.approx(g["reduction"])


def test_memory_mha_ratio_and_gqa_closed_form():
    # MHA: UPipe/Ulysses intermediate ratio is exactly U/H
    S, d = 1 << 20, 128
    for H, C, U in ((32, 8, 8), (32, 4, 8), (64, 8, 16)):
        assert O.intermediate_elems_gqa(S, C, H, H, d, U) / O.intermediate_elems_gqa(S, C, H, H, d, H) == U / H
    # GQA (DESIGN A22): Llama3-8B CP8 U8 -> total 0.5, Q-path 0.25; 32B CP8 U8 -> 0.3
    assert O.intermediate_elems_gqa(S, 8, 32, 8, d, 8) / O.intermediate_elems_gqa(S, 8, 32, 8, d, 32) == 0.5
    assert O.intermediate_elems_gqa(S, 8, 64, 8, d, 8) / O.intermediate_elems_gqa(S, 8, 64, 8, d, 64) == pytest.approx(0.3)


# ---------------------------------------------------------------- synth generator

def test_synth_values_exact_bf16_and_deterministic():
    v = synth.draw(0, synth.TID["x"], (1000,), 1)
    bits = synth.to_bf16_bits(v)                      # raises if not exactly representable
    np.testing.assert_array_equal(synth.from_bf16_bits(bits), v)
    w = synth.draw(0, synth.TID["x"], (500,), 1, start=500)
    np.testing.assert_array_equal(v[500:], w)         # global indexing: shards agree
    assert abs(v.mean()) < 0.15 and 0.9 < v.std() / (2 / math.sqrt(3)) < 1.1
    assert set(np.unique(synth.draw_codes(3, 2, 0, 100000))) == set(range(256))


def test_row_sampled_layer_matches_full():
    # the row-sampled / tail modes used at full size equal the full oracle on a small case
    S, D, Hq, Hkv, d = 150, 24, 4, 2, 8
    X, Wq, Wk, Wv = rand(S, D), rand(Hq * d, D, scale=.3), rand(Hkv * d, D, scale=.3), rand(Hkv * d, D, scale=.3)
    Wo, dY = rand(D, Hq * d, scale=.3), rand(S, D)
    Y, Oo, L = O.layer_fwd(X, Wq, Wk, Wv, Wo, Hq, Hkv, d)
    K = (X @ Wk.T).reshape(S, Hkv, d)
    V = (X @ Wv.T).reshape(S, Hkv, d)
    rows = np.array([0, 1, 63, 64, 100, 149])
    y, o, lse = O.layer_fwd_rows(X[rows], rows, K, V, Wq, Wo, Hq, Hkv, d)
    np.testing.assert_allclose(y, Y[rows], atol=1e-12)
    np.testing.assert_allclose(lse, L[:, rows], atol=1e-12)
    dX = O.layer_bwd(X, Wq, Wk, Wv, Wo, dY, Hq, Hkv, d)[0]
    w = 17
    np.testing.assert_allclose(O.layer_bwd_tail(X[-w:], dY[-w:], K, V, Wq, Wk, Wv, Wo, Hq, Hkv, d), dX[-w:],
                               atol=1e-11)


def test_row_sampled_layer_matches_full_with_rope():
    S, D, Hq, Hkv, d, base = 150, 24, 4, 2, 8, 50.0
    X, Wq, Wk, Wv = rand(S, D), rand(Hq * d, D, scale=.3), rand(Hkv * d, D, scale=.3), rand(Hkv * d, D, scale=.3)
    Wo, dY = rand(D, Hq * d, scale=.3), rand(S, D)
    Y, Oo, L = O.layer_fwd(X, Wq, Wk, Wv, Wo, Hq, Hkv, d, rope_base=base)
    K = O.rope((X @ Wk.T).reshape(S, Hkv, d), np.arange(S), base)
    V = (X @ Wv.T).reshape(S, Hkv, d)
    rows = np.array([0, 1, 63, 64, 100, 149])
    y, o, lse = O.layer_fwd_rows(X[rows], rows, K, V, Wq, Wo, Hq, Hkv, d, rope_base=base)
    np.testing.assert_allclose(y, Y[rows], atol=1e-12)
    np.testing.assert_allclose(lse, L[:, rows], atol=1e-12)
    dX = O.layer_bwd(X, Wq, Wk, Wv, Wo, dY, Hq, Hkv, d, rope_base=base)[0]
    w = 17
    np.testing.assert_allclose(O.layer_bwd_tail(X[-w:], dY[-w:], K, V, Wq, Wk, Wv, Wo, Hq, Hkv, d, rope_base=base),
                               dX[-w:], atol=1e-11)


# ---------------------------------------------------------------- ring blocks and the hybrid (N4)

def _partial(rng_rows, H=2, d=3):
    return rand(rng_rows, H, d), rand(H, rng_rows)


def test_merge_empty_partial_is_identity():
    # merge(p, empty-sentinel) = p (both argument orders)
    Op, lp = _partial(5)
    empty_O, empty_l = np.zeros_like(Op), np.full_like(lp, -np.inf)
    for a, b in (((Op, lp), (empty_O, empty_l)), ((empty_O, empty_l), (Op, lp))):
        Om, lm = O.merge_partials(*a, *b)
        np.testing.assert_array_equal(lm, lp)
        np.testing.assert_allclose(Om, Op, rtol=0, atol=0)
    Om, lm = O.merge_partials(empty_O, empty_l, empty_O, empty_l)
    assert np.all(np.isneginf(lm)) and np.all(Om == 0)


def test_merge_equal_halves():
    # merge(p, p) has lse' = lse + ln 2 and out' = out
    Op, lp = _partial(7)
    Om, lm = O.merge_partials(Op, lp, Op, lp)
    np.testing.assert_allclose(lm, lp + math.log(2.0), rtol=0, atol=1e-14)
    np.testing.assert_allclose(Om, Op, rtol=0, atol=1e-14)


def test_merge_two_single_key_partials_is_two_key_softmax():
    # partials of one key each == softmax attention over both keys (brute force)
    d = 4
    q, k0, k1, v0, v1 = (rand(d) for _ in range(5))
    s0, s1 = q @ k0 / math.sqrt(d), q @ k1 / math.sqrt(d)
    # a single-key partial: O = v, lse = s (softmax over one key)
    Om, lm = O.merge_partials(v0[None, None], np.array([[s0]]), v1[None, None], np.array([[s1]]))
    w0, w1 = math.exp(s0), math.exp(s1)
    np.testing.assert_allclose(Om[0, 0], (w0 * v0 + w1 * v1) / (w0 + w1), rtol=0, atol=1e-12)
    np.testing.assert_allclose(lm[0, 0], math.log(w0 + w1), rtol=0, atol=1e-12)


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("cuts", [(0, 6, 13, 20), (0, 10, 20), (0, 3, 4, 17, 20)])
def test_blocks_merge_to_full_attention(causal, cuts):
    # merging the per-key-block partials in ring order (own block first) reproduces attn_fwd over
    # all keys (the method exactness of ring attention); blocks after the query block are
    # fully masked under causality and merge as the identity
    S, Hq, Hkv, d = 20, 4, 2, 3
    Q, K, V = rand(S, Hq, d), rand(S, Hkv, d), rand(S, Hkv, d)
    Of, lf = O.attn_fwd(Q, K, V, causal)
    nb = len(cuts) - 1
    for i in range(nb):
        q0, q1 = cuts[i], cuts[i + 1]
        Oacc = lacc = None
        for t in range(nb):
            j = (i - t) % nb
            k0, k1 = cuts[j], cuts[j + 1]
            Op, lp = O.attn_fwd_block(Q[q0:q1], K[k0:k1], V[k0:k1], q0, k0, causal)
            Oacc, lacc = (Op, lp) if t == 0 else O.merge_partials(Oacc, lacc, Op, lp)
        np.testing.assert_allclose(Oacc, Of[q0:q1], rtol=0, atol=1e-12)
        np.testing.assert_allclose(lacc, lf[:, q0:q1], rtol=0, atol=1e-12)


@pytest.mark.parametrize("causal", [True, False])
def test_block_gradients_sum_to_attn_bwd(causal):
    # the ring backward: per (query block, key block) contributions with the FINAL lse and D sum
    # to attn_bwd (itself pinned by finite differences and torch autograd)
    S, Hq, Hkv, d = 18, 4, 2, 3
    Q, K, V, dO = rand(S, Hq, d), rand(S, Hkv, d), rand(S, Hkv, d), rand(S, Hq, d)
    gq, gk, gv = O.attn_bwd(Q, K, V, dO, causal)
    Of, lf = O.attn_fwd(Q, K, V, causal)
    Dv = O.rowdot(dO, Of)
    cuts = (0, 5, 12, 18)
    dQ, dK, dV = np.zeros_like(Q), np.zeros_like(K), np.zeros_like(V)
    for i in range(3):
        q0, q1 = cuts[i], cuts[i + 1]
        for j in range(3):
            k0, k1 = cuts[j], cuts[j + 1]
            bq, bk, bv = O.attn_bwd_block(Q[q0:q1], K[k0:k1], V[k0:k1], dO[q0:q1], lf[:, q0:q1], Dv[q0:q1],
                                          q0, k0, causal)
            dQ[q0:q1] += bq
            dK[k0:k1] += bk
            dV[k0:k1] += bv
    np.testing.assert_allclose(dQ, gq, rtol=0, atol=1e-12)
    np.testing.assert_allclose(dK, gk, rtol=0, atol=1e-12)
    np.testing.assert_allclose(dV, gv, rtol=0, atol=1e-12)


HYB = [(8, 2, 1, 2, 2), (8, 2, 2, 2, 2), (8, 2, 2, 2, 4), (8, 4, 1, 4, 4), (8, 4, 2, 2, 2),
       (16, 4, 2, 2, 8), (8, 8, 4, 1, 4), (8, 2, 2, 1, 2)]


@pytest.mark.parametrize("Hq,Hkv,a,r,U", HYB)
def test_hybrid_sim_equals_unsharded(Hq, Hkv, a, r, U):
    # UPipe x Ring (a Ulysses ranks per group, r ring groups) is exact: equal to the
    # un-sharded layer for every split, forward and backward
    S, D, d = 16, 12, 4
    X, Wq, Wk, Wv = rand(S, D), rand(Hq * d, D, scale=.4), rand(Hkv * d, D, scale=.4), rand(Hkv * d, D, scale=.4)
    Wo, dY = rand(D, Hq * d, scale=.4), rand(S, D)
    Y, Ob, lse = O.layer_fwd(X, Wq, Wk, Wv, Wo, Hq, Hkv, d)
    Y2, Ob2, lse2 = O.hybrid_forward(X, Wq, Wk, Wv, Wo, Hq, Hkv, d, a, r, U)
    np.testing.assert_allclose(Y2, Y, atol=1e-12)
    np.testing.assert_allclose(Ob2, Ob, atol=1e-12)
    np.testing.assert_allclose(lse2, lse, atol=1e-12)
    g1 = O.layer_bwd(X, Wq, Wk, Wv, Wo, dY, Hq, Hkv, d)
    g2 = O.hybrid_backward(X, Wq, Wk, Wv, Wo, dY, Hq, Hkv, d, a, r, U)
    for x2, x1 in zip(g2, g1):
        np.testing.assert_allclose(x2, x1, atol=1e-11)


def test_hybrid_degenerate_compositions():
    # a = C, r = 1 is UPipe/Ulysses itself (bitwise: same operations in the same order);
    # a = 1, r = C is pure ring attention (equal to the oracle)
    Hq, Hkv, d, S, D = 8, 2, 4, 16, 12
    X, Wq, Wk, Wv = rand(S, D), rand(Hq * d, D, scale=.4), rand(Hkv * d, D, scale=.4), rand(Hkv * d, D, scale=.4)
    Wo = rand(D, Hq * d, scale=.4)
    for U in (2, 4, 8):
        a = O.hybrid_forward(X, Wq, Wk, Wv, Wo, Hq, Hkv, d, 2, 1, U)
        b = O.upipe_forward(X, Wq, Wk, Wv, Wo, Hq, Hkv, d, 2, U)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)
    ring = O.hybrid_forward(X, Wq, Wk, Wv, Wo, Hq, Hkv, d, 1, 4, 8)
    ref = O.layer_fwd(X, Wq, Wk, Wv, Wo, Hq, Hkv, d)
    for x, y in zip(ring, ref):
        np.testing.assert_allclose(x, y, atol=1e-12)


# ---------------------------------------------------------------- Qwen3 per-head q/k RMSNorm

def test_rms_norm_heads_hand_values_and_invariants():
    # textbook RMSNorm on a hand example: T = (3, 4): mean square 12.5, gamma = (1, 2)
    y, rstd = O.rms_norm_heads(np.array([[[3.0, 4.0]]]), np.array([1.0, 2.0]), 0.0)
    np.testing.assert_allclose(y[0, 0], [0.8485281374238570, 2.262741699796952], rtol=0, atol=1e-15)
    np.testing.assert_allclose(rstd, [[1 / math.sqrt(12.5)]], rtol=1e-15)
    T = rand(5, 3, 8)
    y1, _ = O.rms_norm_heads(T, np.ones(8), 0.0)
    np.testing.assert_allclose(np.mean(y1 ** 2, axis=-1), 1.0, rtol=1e-13)        # unit RMS for gamma = 1
    np.testing.assert_allclose(O.rms_norm_heads(7.5 * T, np.ones(8), 0.0)[0], y1, rtol=1e-13)   # scale invariant
    g = rand(8)
    np.testing.assert_allclose(O.rms_norm_heads(T, g, 0.0)[0], y1 * g, rtol=1e-13)  # gamma is a per-dim scale
    # eps enters under the root: rstd = 1/sqrt(ms + eps)
    _, r2 = O.rms_norm_heads(T, g, 0.25)
    np.testing.assert_allclose(r2, 1 / np.sqrt(np.mean(T ** 2, -1) + 0.25), rtol=1e-15)


def test_rms_norm_heads_bwd_matches_torch_rms_norm_autograd():
    T, G, g = rand(6, 3, 8), rand(6, 3, 8), rand(8)
    dT, dg = O.rms_norm_heads_bwd(T, g, 1e-6, G)
    tT, tg = torch.from_numpy(T).requires_grad_(), torch.from_numpy(g).requires_grad_()
    ty = F.rms_norm(tT, (8,), weight=tg, eps=1e-6)            # library routine, independent of the oracle
    np.testing.assert_allclose(O.rms_norm_heads(T, g, 1e-6)[0], ty.detach().numpy(), atol=1e-13)
    ty.backward(torch.from_numpy(G))
    np.testing.assert_allclose(dT, tT.grad.numpy(), atol=1e-12)
    np.testing.assert_allclose(dg, tg.grad.numpy(), atol=1e-12)


def _torch_layer_qknorm(X, Wq, Wk, Wv, Wo, gq, gk, Hq, Hkv, d, eps):
    S = X.shape[0]
    q = F.rms_norm((X @ Wq.T).view(S, Hq, d), (d,), weight=gq, eps=eps).transpose(0, 1)[None]
    k = F.rms_norm((X @ Wk.T).view(S, Hkv, d), (d,), weight=gk, eps=eps).transpose(0, 1)[None]
    v = (X @ Wv.T).view(S, Hkv, d).transpose(0, 1)[None]
    o = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
    return o[0].transpose(0, 1).reshape(S, Hq * d) @ Wo.T


def test_qk_norm_layer_matches_torch_autograd():
    S, D, Hq, Hkv, d, eps = 40, 24, 4, 2, 8, 1e-6
    X, Wq, Wk, Wv = rand(S, D), rand(Hq * d, D, scale=.3), rand(Hkv * d, D, scale=.3), rand(Hkv * d, D, scale=.3)
    Wo, dY, gq, gk = rand(D, Hq * d, scale=.3), rand(S, D), 1 + 0.3 * rand(d), 1 + 0.3 * rand(d)
    Y, _, _ = O.layer_fwd(X, Wq, Wk, Wv, Wo, Hq, Hkv, d, qk_norm=(gq, gk, eps))
    grads = O.layer_bwd(X, Wq, Wk, Wv, Wo, dY, Hq, Hkv, d, qk_norm=(gq, gk, eps))
    assert len(grads) == 7
    ts = [torch.from_numpy(a).requires_grad_() for a in (X, Wq, Wk, Wv, Wo, gq, gk)]
    ty = _torch_layer_qknorm(*ts, Hq, Hkv, d, eps)
    np.testing.assert_allclose(Y, ty.detach().numpy(), atol=1e-11)
    ty.backward(torch.from_numpy(dY))
    for mine, t in zip(grads, ts):
        np.testing.assert_allclose(mine, t.grad.numpy(), atol=1e-10)


def test_qk_norm_rope_layer_finite_differences():
    # norm, then RoPE (Qwen3 order): every gradient incl. d(gamma_q), d(gamma_k) by central differences
    S, D, Hq, Hkv, d, base, eps = 5, 5, 2, 1, 4, 100.0, 1e-6
    X, Wq, Wk, Wv, Wo, dY = (rand(S, D), rand(Hq * d, D), rand(Hkv * d, D), rand(Hkv * d, D),
                             rand(D, Hq * d), rand(S, D))
    gq, gk = 1 + 0.3 * rand(d), 1 + 0.3 * rand(d)
    args = [X, Wq, Wk, Wv, Wo, gq, gk]
    grads = O.layer_bwd(X, Wq, Wk, Wv, Wo, dY, Hq, Hkv, d, rope_base=base, qk_norm=(gq, gk, eps))
    h = 1e-5

    def loss(a):
        return float(np.sum(O.layer_fwd(*a[:5], Hq, Hkv, d, rope_base=base, qk_norm=(a[5], a[6], eps))[0] * dY))
    for idx, g in enumerate(grads):
        num = np.zeros_like(args[idx])
        for i in np.ndindex(num.shape):
            ap = [a.copy() for a in args]
            am = [a.copy() for a in args]
            ap[idx][i] += h
            am[idx][i] -= h
            num[i] = (loss(ap) - loss(am)) / (2 * h)
        assert np.linalg.norm(num - g) <= 1e-6 * np.linalg.norm(g), idx
    # the norm changes the layer (not silently skipped)
    assert not np.allclose(O.layer_fwd(X, Wq, Wk, Wv, Wo, Hq, Hkv, d, rope_base=base)[0],
                           O.layer_fwd(X, Wq, Wk, Wv, Wo, Hq, Hkv, d, rope_base=base, qk_norm=(gq, gk, eps))[0])
