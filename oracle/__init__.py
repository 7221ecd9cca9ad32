"""fp64 CPU oracle for UPipe's headwise-chunked Ulysses attention layer.

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may import
this package. The product path (``paper_2602_21196_b200``) never imports it and
shares no code with it; the only shared module is ``synth`` (input generation,
no arithmetic of the method).

Citations: ``P:n`` = /root/reference/PAPER.md line n, ``S:n`` = SPEC.md line n.
Readings of silent/ambiguous points are DESIGN.md §"Readings" (A1..A25, same
numbering as SURVEY.md §8c).

Everything is float64 numpy. Library primitives used as single steps: matmul
(``@``), ``exp``, ``log``, ``max``, ``sum``. Rows of the attention are
independent by definition, so they are processed in blocks of rows only to bound
memory; each row is computed with the plain (non-online) softmax definition.

Functions and their pins (tests/test_oracle_*.py):

* ``attn_fwd``      -- pinned: SPEC worked examples, torch fp64 SDPA,
                       closed forms (constant V, zero K), rows sum to 1, GQA==MHA
                       with repeated K/V, causal perturbation.
* ``attn_bwd``      -- pinned: central finite differences, torch fp64 autograd,
                       dO=0, S=1 closed form.
* ``layer_fwd/bwd`` -- pinned: finite differences on all of dX, dW*, torch fp64
                       autograd of the composed layer, stage decomposition.
* ``gqa_schedule``, ``comm_volume`` -- pinned: Fig. 4 / §4.1 example,
                       §4.1 volume formulas with the paper's numbers,
                       SPEC S:279-281.
* ``a2a_seq_to_head``/``a2a_head_to_seq`` -- pinned: §3.1 example,
                       round trip identity, C=1 identity.
* ``upipe_forward/backward`` (sharded simulation) -- pinned: equal to the
                       un-sharded oracle for every (C, U) (method exactness).
* ``memory_*``      -- pinned: §3.4 numbers (96 -> 12 S d_head, 87.5 %).
* ``merge_partials`` -- pinned: SPEC S:64-66 (empty partial is the identity,
                       merge(p, p) = (p.out, p.lse + ln 2), two one-key partials = the
                       brute-force two-key softmax).
* ``attn_fwd_block``/``attn_bwd_block`` -- pinned: merged in ring order / summed over
                       key blocks they reproduce ``attn_fwd`` / ``attn_bwd`` (themselves
                       pinned above), causal and not, with fully masked blocks.
* ``hybrid_forward/backward`` (UPipe x Ring) -- pinned: equal to the
                       un-sharded layer for every (a, r, U) of a grid; a = C, r = 1 is
                       bitwise ``upipe_forward``; a = 1 is pure ring attention.
* ``rms_norm_heads``/``rms_norm_heads_bwd`` (Qwen3 per-head q/k RMSNorm)
                    -- pinned: the textbook RMSNorm definition on hand values, unit-RMS
                       output for gamma = 1, scale invariance (x -> c x leaves the output
                       unchanged up to eps), torch fp64 autograd of the composed layer and
                       central finite differences on dX, dW and d(gamma_q), d(gamma_k).
* ``rope``          -- pinned: complex-exponential form (each pair times e^{i p theta_i}),
                       relative-position invariance of q.k, norm preservation, position 0 =
                       identity, inverse o forward = identity; the RoPE layer's gradients by
                       central finite differences.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------
# Attention core  (Table 1 stage 2; DESIGN A1-A3, A17)
# ----------------------------------------------------------------------------

_ROW_BLOCK = 512


def _kv_map(Hq: int, Hkv: int, kv_of_head=None):
    """GQA map: query head h reads kv head floor(h / R), R = Hq/Hkv (DESIGN A3)."""
    if kv_of_head is not None:
        return list(kv_of_head)
    if Hq % Hkv:
        raise ValueError("Hq % Hkv != 0 (S:37)")
    R = Hq // Hkv
    return [h // R for h in range(Hq)]


def attn_fwd(Q, K, V, causal=True, kv_of_head=None, rows=None):
    """Causal GQA softmax attention, scale 1/sqrt(d) (DESIGN A1, A2).

    Q: [S, Hq, d], K/V: [Skv, Hkv, d] (float64). Key j is visible to query i iff
    j <= i (global token index). Returns O [S, Hq, d] and the natural-log
    log-sum-exp lse [Hq, S] with lse_i = m_i + ln(sum_j exp(s_ij - m_i)).

    ``rows``: optional array of query rows to compute (row-sampled mode); the
    returned O/lse then have len(rows) rows, in that order, and Q must be the full
    [S, Hq, d] tensor or only those rows (``Q.shape[0] == len(rows)``).
    """
    Sq, Hq, d = Q.shape
    Skv, Hkv, _ = K.shape
    kvh = _kv_map(Hq, Hkv, kv_of_head)
    scale = 1.0 / math.sqrt(d)
    if rows is None:
        qrows = np.arange(Sq)
        Qr = Q
    else:
        qrows = np.asarray(rows, dtype=np.int64)
        Qr = Q if Q.shape[0] == len(qrows) else Q[qrows]
    n = len(qrows)
    O = np.zeros((n, Hq, d))
    lse = np.zeros((Hq, n))
    keys = np.arange(Skv)
    for h in range(Hq):
        g = kvh[h]
        for b0 in range(0, n, _ROW_BLOCK):
            b1 = min(n, b0 + _ROW_BLOCK)
            qi = qrows[b0:b1]
            s = (Qr[b0:b1, h, :] @ K[:, g, :].T) * scale          # s_ij = <q_i,k_j>/sqrt(d)
            if causal:
                s = np.where(keys[None, :] <= qi[:, None], s, -np.inf)
            m = np.max(s, axis=1, keepdims=True)                    # m_i
            l = np.sum(np.exp(s - m), axis=1, keepdims=True)        # l_i
            lse_b = m + np.log(l)                                   # lse_i
            P = np.exp(s - lse_b)                                   # P_ij
            O[b0:b1, h, :] = P @ V[:, g, :]                         # O_i = sum_j P_ij V_j
            lse[h, b0:b1] = lse_b[:, 0]
    return O, lse


def attn_bwd(Q, K, V, dO, causal=True, kv_of_head=None):
    """Gradients of O = attn_fwd(Q,K,V) for cotangent dO.

    D_i = <dO_i, O_i>; dV_j += sum_i P_ij dO_i; dP_ij = <dO_i, V_j>;
    dS_ij = P_ij (dP_ij - D_i); dQ_i = (1/sqrt d) sum_j dS_ij K_j;
    dK_j += (1/sqrt d) sum_i dS_ij Q_i, kv gradients summed over the group's heads.
    P is recomputed from its definition (no saved state is trusted).
    """
    S, Hq, d = Q.shape
    Skv, Hkv, _ = K.shape
    kvh = _kv_map(Hq, Hkv, kv_of_head)
    scale = 1.0 / math.sqrt(d)
    dQ = np.zeros_like(Q)
    dK = np.zeros_like(K)
    dV = np.zeros_like(V)
    keys = np.arange(Skv)
    for h in range(Hq):
        g = kvh[h]
        for b0 in range(0, S, _ROW_BLOCK):
            b1 = min(S, b0 + _ROW_BLOCK)
            qi = np.arange(b0, b1)
            s = (Q[b0:b1, h, :] @ K[:, g, :].T) * scale
            if causal:
                s = np.where(keys[None, :] <= qi[:, None], s, -np.inf)
            m = np.max(s, axis=1, keepdims=True)
            P = np.exp(s - m)
            P /= np.sum(P, axis=1, keepdims=True)
            Ob = P @ V[:, g, :]
            dOb = dO[b0:b1, h, :]
            Dv = np.sum(dOb * Ob, axis=1, keepdims=True)            # D_i
            dV[:, g, :] += P.T @ dOb
            dP = dOb @ V[:, g, :].T
            dS = P * (dP - Dv)
            dQ[b0:b1, h, :] = (dS @ K[:, g, :]) * scale
            dK[:, g, :] += (dS.T @ Q[b0:b1, h, :]) * scale
    return dQ, dK, dV


def rowdot(dO, O):
    """D_i = <dO_i, O_i> per (row, head) (the D term of attn_bwd). [S,H,d] -> [S,H]."""
    return np.sum(dO * O, axis=-1)


def project(X, W):
    """Projection of the input into heads, X W^T with nn.Linear W [out, in] (DESIGN A4)."""
    return X @ W.T


# ----------------------------------------------------------------------------
# Layer = projections + attention + output projection (§3.1)
# Weights are nn.Linear [out, in]; head h <-> rows [h d, (h+1) d) (DESIGN A4).
# ----------------------------------------------------------------------------


def rope(T, positions, base, inverse=False):
    """Rotary position embedding (the paper's RoPE) in the original
    interleaved-pair form (RoFormer; Llama's reference ``apply_rotary_emb``): head-dim pairs
    (2i, 2i+1), i < d/2, of the token at position p are rotated by the angle
    p * base**(-2i/d):  (a, b) -> (a cos - b sin, a sin + b cos).  ``inverse`` rotates by the
    negative angle (the transpose), which maps gradients w.r.t. rotated Q/K back (DESIGN A26).
    T: [S, H, d]; positions: [S] (global token index)."""
    d = T.shape[-1]
    i = np.arange(d // 2, dtype=np.float64)
    ang = np.asarray(positions, dtype=np.float64)[:, None] * base ** (-2.0 * i / d)   # [S, d/2]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    if inverse:
        s = -s
    a, b = T[..., 0::2], T[..., 1::2]
    out = np.empty_like(T, dtype=np.float64)
    out[..., 0::2] = a * c - b * s
    out[..., 1::2] = a * s + b * c
    return out


def rms_norm_heads(T, gamma, eps):
    """Per-head RMSNorm over the head dimension (Qwen3's q_norm / k_norm, applied to each head of
    the projected Q and K before RoPE; the paper's second model family, whose attention
    module the paper overrides as a whole):  y = T / sqrt(mean_e T_e^2 + eps) * gamma.
    T: [S, H, d], gamma: [d].  Returns (y, rstd [S, H])."""
    rstd = 1.0 / np.sqrt(np.mean(T * T, axis=-1) + eps)
    return T * rstd[..., None] * gamma, rstd


def rms_norm_heads_bwd(T, gamma, eps, G):
    """Chain rule of ``rms_norm_heads`` for the cotangent G of its output:
    T_hat = T * rstd,  dT_hat = G * gamma,  dT = rstd * (dT_hat - T_hat * mean_e(dT_hat * T_hat)),
    dgamma = sum over tokens and heads of G * T_hat.  Returns (dT, dgamma)."""
    rstd = 1.0 / np.sqrt(np.mean(T * T, axis=-1) + eps)
    T_hat = T * rstd[..., None]
    dT_hat = G * gamma
    dT = rstd[..., None] * (dT_hat - T_hat * np.mean(dT_hat * T_hat, axis=-1, keepdims=True))
    dgamma = np.sum(G * T_hat, axis=(0, 1))
    return dT, dgamma


def _qkv(X, Wq, Wk, Wv, Hq, Hkv, d, rope_base, pos0=0, qk_norm=None):
    S = X.shape[0]
    Q = project(X, Wq).reshape(S, Hq, d)
    K = project(X, Wk).reshape(S, Hkv, d)
    V = project(X, Wv).reshape(S, Hkv, d)
    if qk_norm is not None:              # (gamma_q, gamma_k, eps): Qwen3 order, norm then RoPE
        gq, gk, eps = qk_norm
        Q, K = rms_norm_heads(Q, gq, eps)[0], rms_norm_heads(K, gk, eps)[0]
    if rope_base:
        pos = np.arange(pos0, pos0 + S)
        Q, K = rope(Q, pos, rope_base), rope(K, pos, rope_base)
    return Q, K, V


def layer_fwd(X, Wq, Wk, Wv, Wo, Hq, Hkv, d, causal=True, rope_base=None, qk_norm=None):
    """Y = O Wo^T with O = attn(X Wq^T, X Wk^T, X Wv^T) (Q and K rotated by ``rope`` at their
    token positions when ``rope_base`` is given; per-head RMSNorm of Q and K first when
    ``qk_norm`` = (gamma_q, gamma_k, eps) is given).  Returns (Y, O [S,Hq*d], lse [Hq,S])."""
    S = X.shape[0]
    Q, K, V = _qkv(X, Wq, Wk, Wv, Hq, Hkv, d, rope_base, qk_norm=qk_norm)
    O, lse = attn_fwd(Q, K, V, causal)
    O2 = O.reshape(S, Hq * d)
    return project(O2, Wo), O2, lse


def layer_bwd(X, Wq, Wk, Wv, Wo, dY, Hq, Hkv, d, causal=True, rope_base=None, qk_norm=None):
    """(dX, dWq, dWk, dWv, dWo) of the layer for cotangent dY; with RoPE the
    gradients w.r.t. the rotated Q/K are rotated back (chain rule through an orthogonal map); with
    ``qk_norm`` they then pass through ``rms_norm_heads_bwd`` and (dgamma_q, dgamma_k) are appended."""
    S = X.shape[0]
    Q, K, V = _qkv(X, Wq, Wk, Wv, Hq, Hkv, d, rope_base, qk_norm=qk_norm)
    O, _ = attn_fwd(Q, K, V, causal)
    O2 = O.reshape(S, Hq * d)
    dWo = dY.T @ O2
    dO = (dY @ Wo).reshape(S, Hq, d)
    dQ, dK, dV = attn_bwd(Q, K, V, dO, causal)
    if rope_base:
        pos = np.arange(S)
        dQ, dK = rope(dQ, pos, rope_base, inverse=True), rope(dK, pos, rope_base, inverse=True)
    extra = ()
    if qk_norm is not None:
        gq, gk, eps = qk_norm
        dQ, dgq = rms_norm_heads_bwd(project(X, Wq).reshape(S, Hq, d), gq, eps, dQ)
        dK, dgk = rms_norm_heads_bwd(project(X, Wk).reshape(S, Hkv, d), gk, eps, dK)
        extra = (dgq, dgk)
    dQ2, dK2, dV2 = dQ.reshape(S, -1), dK.reshape(S, -1), dV.reshape(S, -1)
    dWq = dQ2.T @ X
    dWk = dK2.T @ X
    dWv = dV2.T @ X
    dX = dQ2 @ Wq + dK2 @ Wk + dV2 @ Wv
    return (dX, dWq, dWk, dWv, dWo) + extra


def layer_fwd_rows(X_rows, rows, K, V, Wq, Wo, Hq, Hkv, d, causal=True, rope_base=None):
    """Row-sampled forward: y, O, lse of the given query rows only.

    ``X_rows`` are those rows of X; ``K``, ``V`` = X Wk^T, X Wv^T for all tokens ([S, Hkv, d]).
    Each row is computed exactly as in ``layer_fwd`` (rows of attention are independent).
    """
    Qr = project(X_rows, Wq).reshape(len(rows), Hq, d)
    if rope_base:                        # K is passed already rotated (rope(X Wk^T, arange(S)))
        Qr = rope(Qr, rows, rope_base)
    O, lse = attn_fwd(Qr, K, V, causal, rows=rows)
    O2 = O.reshape(len(rows), Hq * d)
    return project(O2, Wo), O2, lse


def layer_bwd_tail(X_tail, dY_tail, K, V, Wq, Wk, Wv, Wo, Hq, Hkv, d, rope_base=None):
    """dX of the last w tokens of a causal layer (w = len(X_tail)), following the same
    formulas as ``attn_bwd``/``layer_bwd``: with a causal mask, dK_j and dV_j of a key j in
    the tail only receive contributions from queries i >= j, which are all in the tail;
    dQ_i needs row i against all keys. So the tail's dX is exact from the tail rows alone."""
    S = K.shape[0]
    w = X_tail.shape[0]
    t0 = S - w
    R = Hq // Hkv
    scale = 1.0 / math.sqrt(d)
    Qt = project(X_tail, Wq).reshape(w, Hq, d)
    if rope_base:                        # K is passed already rotated; Q of the tail rotated here
        Qt = rope(Qt, np.arange(t0, S), rope_base)
    dOt = (dY_tail @ Wo).reshape(w, Hq, d)
    dQ = np.zeros((w, Hq, d))
    dK = np.zeros((w, Hkv, d))
    dV = np.zeros((w, Hkv, d))
    qi = np.arange(t0, S)
    keys = np.arange(S)
    for h in range(Hq):
        g = h // R
        s = (Qt[:, h, :] @ K[:, g, :].T) * scale
        s = np.where(keys[None, :] <= qi[:, None], s, -np.inf)
        m = np.max(s, axis=1, keepdims=True)
        P = np.exp(s - m)
        P /= np.sum(P, axis=1, keepdims=True)
        Ot = P @ V[:, g, :]
        Dv = np.sum(dOt[:, h, :] * Ot, axis=1, keepdims=True)
        dP = dOt[:, h, :] @ V[:, g, :].T
        dS = P * (dP - Dv)
        dQ[:, h, :] = (dS @ K[:, g, :]) * scale
        dK[:, g, :] += (dS[:, t0:].T @ Qt[:, h, :]) * scale
        dV[:, g, :] += P[:, t0:].T @ dOt[:, h, :]
    if rope_base:
        dQ = rope(dQ, np.arange(t0, S), rope_base, inverse=True)
        dK = rope(dK, np.arange(t0, S), rope_base, inverse=True)
    return dQ.reshape(w, -1) @ Wq + dK.reshape(w, -1) @ Wk + dV.reshape(w, -1) @ Wv


# ----------------------------------------------------------------------------
# GQA schedule  (§4.1, Fig. 4 caption P:306; DESIGN A8)
# ----------------------------------------------------------------------------


@dataclass
class Stage:
    q_heads: list                       # per device p: list of global q heads (qpd of them)
    kv_heads: list                      # per device p: kv heads resident for this stage
    kv_sent: list                       # per device p: kv heads newly sent in this stage
    heads: list = field(default_factory=list)   # all U q heads of the stage, device-major


def gqa_schedule(Hq, Hkv, C, U):
    """Head -> (stage, device) assignment and KV transfers (§4.1, Fig. 4).

    Written as the paper describes it: stages are grouped into super-stages. The
    first stage of a super-stage "communicate[s] as many unique key/value heads as
    possible along with the corresponding queries"; the following stages "only
    communicate the next queries of the corresponding groups, reusing the key/value
    tensors". With R = Hq/Hkv (the paper's G, DESIGN A3):

    * super-stage b gives device p the KV heads (b C + p) kv_res + i, i < kv_res
      (round robin over devices), kv_res = max(1, qpd/R);
    * stage r of the super-stage gives device p the next qpd = U/C queries of
      those groups: g R + r qpd + j (qpd <= R), or all R queries of its kv_res
      groups (qpd >= R, one stage per super-stage).

    Reproduces Fig. 3b (MHA: stage 0 = H0, H1), Fig. 4 (16/4/4: stage 0
    Q0,Q4,Q8,Q12 with K0..K3) and Ulysses at U = Hq.
    Reading for U > C and Hkv > C: DESIGN A8. Hkv % C != 0 or qpd, R not dividing
    one another: unsupported (DESIGN A9).
    """
    if U % C:
        raise ValueError("U must be divisible by C (P:317)")
    if Hq % U:
        raise ValueError("Hq % U != 0")
    if Hq % Hkv:
        raise ValueError("Hq % Hkv != 0")
    if Hkv % C:
        raise ValueError("Hkv % C != 0: unsupported GQA shape (DESIGN A9)")
    R = Hq // Hkv
    qpd = U // C
    if R % qpd and qpd % R:
        raise ValueError("qpd and R must divide one another (DESIGN A9)")
    kv_res = max(1, qpd // R)
    sigma = max(1, R // qpd)
    stages = []
    for b in range(Hkv // (C * kv_res)):
        kv_of_dev = [[(b * C + p) * kv_res + i for i in range(kv_res)] for p in range(C)]
        for r in range(sigma):
            q_of_dev = []
            for p in range(C):
                if qpd <= R:
                    q_of_dev.append([g * R + r * qpd + j for g in kv_of_dev[p] for j in range(qpd)])
                else:
                    q_of_dev.append([g * R + j for g in kv_of_dev[p] for j in range(R)])
            stages.append(Stage(q_heads=q_of_dev, kv_heads=[list(k) for k in kv_of_dev],
                                kv_sent=[list(k) for k in kv_of_dev] if r == 0 else [[] for _ in range(C)],
                                heads=[h for q in q_of_dev for h in q]))
    return stages


def naive_schedule(Hq, Hkv, C, U):
    """Naive processing: stage s takes heads [sU, (s+1)U), device p the
    p-th block of U/C, and K/V for every q head are re-sent each stage."""
    R = Hq // Hkv
    qpd = U // C
    stages = []
    for s in range(Hq // U):
        qh = [list(range(s * U + p * qpd, s * U + (p + 1) * qpd)) for p in range(C)]
        kv = [[h // R for h in q] for q in qh]       # one K/V per q head, duplicates sent
        stages.append(Stage(q_heads=qh, kv_heads=kv, kv_sent=kv,
                            heads=[h for q in qh for h in q]))
    return stages


def comm_volume(stages, C):
    """Head-slices (one head x S/C tokens) each device sends in the forward inp_all_to_all:
    for every stage and every other device q: its q heads, plus K and V for kv_sent."""
    vol = 0
    for st in stages:
        for q in range(1, C):
            vol += len(st.q_heads[q]) + 2 * len(st.kv_sent[q])
    return vol


def comm_volume_formula(Hq, Hkv, C, scheduled):
    """P:373 naive 3 (H/C)(C-1); P:380 scheduled (3+G-1) H/(C G) (C-1), G = R = Hq/Hkv."""
    G = Hq // Hkv
    if not scheduled:
        return 3 * (Hq // C) * (C - 1)
    return (3 + G - 1) * Hq * (C - 1) // (C * G)


# ----------------------------------------------------------------------------
# All-to-all resharding (§3.1) on explicit per-device arrays
# ----------------------------------------------------------------------------


def a2a_seq_to_head(shards, heads_of_device):
    """inp_all_to_all: device r holds [S/C, Hx, d] for the stage's heads (device-major:
    the heads of device p are columns heads_of_device offsets). Returns per device p
    [S, n_p, d] covering all tokens (rank r's block at rows r S/C ...) for its heads.

    ``shards[r]``: dict head -> [S/C, d] array.  ``heads_of_device[p]``: list of heads.
    """
    C = len(shards)
    out = []
    for p in range(C):
        cols = [np.concatenate([shards[r][h] for r in range(C)], axis=0) for h in heads_of_device[p]]
        out.append(np.stack(cols, axis=1))
    return out


def a2a_head_to_seq(full, heads_of_device, C):
    """out_all_to_all: device p holds [S, n_p, d] for its heads; returns per device r a
    dict head -> [S/C, d] (rank r's token block)."""
    S = full[0].shape[0]
    Sl = S // C
    res = [dict() for _ in range(C)]
    for p in range(C):
        for j, h in enumerate(heads_of_device[p]):
            for r in range(C):
                res[r][h] = full[p][r * Sl:(r + 1) * Sl, j, :]
    return res


# ----------------------------------------------------------------------------
# Sharded UPipe simulation (§3.3, §4.1) in fp64
# ----------------------------------------------------------------------------


def upipe_forward(X, Wq, Wk, Wv, Wo, Hq, Hkv, d, C, U, causal=True, schedule=None):
    """Stage loop of §3.3 on C simulated devices. Returns (Y [S,D], O [S,Hq d], lse [Hq,S]).

    Per stage: every device projects its sequence shard for the stage's U heads
    (P:316), inp_all_to_all Q then K then V, attention on its U/C
    heads over the full sequence, out_all_to_all, the output is
    written into a pre-allocated buffer and the output projection is
    accumulated (BASELINE north_star).
    """
    S, D = X.shape
    if S % C:
        raise ValueError("S % C != 0")
    Sl = S // C
    stages = schedule or gqa_schedule(Hq, Hkv, C, U)
    Xs = [X[r * Sl:(r + 1) * Sl] for r in range(C)]
    O_buf = [np.zeros((Sl, Hq * d)) for _ in range(C)]     # pre-allocated output
    Y_acc = [np.zeros((Sl, D)) for _ in range(C)]
    lse_all = np.zeros((Hq, S))
    kv_res = [None] * C                                      # resident K/V per device
    for st in stages:
        qsh = [{h: project(Xs[r], Wq[h * d:(h + 1) * d]) for h in st.heads} for r in range(C)]
        Qh = a2a_seq_to_head(qsh, st.q_heads)
        if any(st.kv_sent[p] for p in range(C)):
            kv_heads = [st.kv_heads[p] for p in range(C)]
            all_kv = sorted({g for p in range(C) for g in kv_heads[p]})
            ksh = [{g: project(Xs[r], Wk[g * d:(g + 1) * d]) for g in all_kv} for r in range(C)]
            vsh = [{g: project(Xs[r], Wv[g * d:(g + 1) * d]) for g in all_kv} for r in range(C)]
            Kh = a2a_seq_to_head(ksh, kv_heads)
            Vh = a2a_seq_to_head(vsh, kv_heads)
            kv_res = [(kv_heads[p], Kh[p], Vh[p]) for p in range(C)]
        Oh = []
        for p in range(C):
            kvlist, Kp, Vp = kv_res[p]
            kmap = [kvlist.index(h // (Hq // Hkv)) for h in st.q_heads[p]]
            Op, lp = attn_fwd(Qh[p], Kp, Vp, causal, kv_of_head=kmap)
            Oh.append(Op)
            for j, h in enumerate(st.q_heads[p]):
                lse_all[h] = lp[j]
        Os = a2a_head_to_seq(Oh, st.q_heads, C)
        for r in range(C):
            for h in st.heads:
                O_buf[r][:, h * d:(h + 1) * d] = Os[r][h]
                Y_acc[r] += project(Os[r][h], Wo[:, h * d:(h + 1) * d])
    return np.concatenate(Y_acc, 0), np.concatenate(O_buf, 0), lse_all


def upipe_backward(X, Wq, Wk, Wv, Wo, dY, Hq, Hkv, d, C, U, causal=True, schedule=None):
    """Backward stage loop (Table 4 order: out_all_to_all of dO, attention
    backward, inp_all_to_all of dQ/dK/dV), recomputing the stage's projections
    (full AC). KV gradients are accumulated over the stages that share the
    resident K/V and sent back when the K/V buffer is retired. dW is summed over
    devices at the end (the FSDP reduction). Returns (dX, dWq, dWk, dWv, dWo).
    """
    S, D = X.shape
    Sl = S // C
    R = Hq // Hkv
    stages = schedule or gqa_schedule(Hq, Hkv, C, U)
    _, O_full, _ = upipe_forward(X, Wq, Wk, Wv, Wo, Hq, Hkv, d, C, U, causal, stages)
    Xs = [X[r * Sl:(r + 1) * Sl] for r in range(C)]
    dYs = [dY[r * Sl:(r + 1) * Sl] for r in range(C)]
    Os = [O_full[r * Sl:(r + 1) * Sl] for r in range(C)]
    dX = [np.zeros((Sl, D)) for _ in range(C)]
    dW = [dict(q=np.zeros_like(Wq), k=np.zeros_like(Wk), v=np.zeros_like(Wv),
               o=np.zeros_like(Wo)) for _ in range(C)]
    kv_state = [None] * C

    def retire(p_state_list):
        # send accumulated dK/dV of every device back to sequence layout
        heads_of = [st_[0] for st_ in p_state_list]
        dKs = a2a_head_to_seq([st_[3] for st_ in p_state_list], heads_of, C)
        dVs = a2a_head_to_seq([st_[4] for st_ in p_state_list], heads_of, C)
        for r in range(C):
            for g in sorted({g for h in heads_of for g in h}):
                dX[r] += dKs[r][g] @ Wk[g * d:(g + 1) * d] + dVs[r][g] @ Wv[g * d:(g + 1) * d]
                dW[r]["k"][g * d:(g + 1) * d] += dKs[r][g].T @ Xs[r]
                dW[r]["v"][g * d:(g + 1) * d] += dVs[r][g].T @ Xs[r]

    for st in stages:
        if any(st.kv_sent[p] for p in range(C)):
            if kv_state[0] is not None:
                retire(kv_state)
            kv_heads = [st.kv_heads[p] for p in range(C)]
            all_kv = sorted({g for p in range(C) for g in kv_heads[p]})
            ksh = [{g: project(Xs[r], Wk[g * d:(g + 1) * d]) for g in all_kv} for r in range(C)]
            vsh = [{g: project(Xs[r], Wv[g * d:(g + 1) * d]) for g in all_kv} for r in range(C)]
            Kh = a2a_seq_to_head(ksh, kv_heads)
            Vh = a2a_seq_to_head(vsh, kv_heads)
            kv_state = [(kv_heads[p], Kh[p], Vh[p], np.zeros_like(Kh[p]), np.zeros_like(Vh[p]))
                        for p in range(C)]
        qsh = [{h: project(Xs[r], Wq[h * d:(h + 1) * d]) for h in st.heads} for r in range(C)]
        dosh = [{h: dYs[r] @ Wo[:, h * d:(h + 1) * d] for h in st.heads} for r in range(C)]
        Qh = a2a_seq_to_head(qsh, st.q_heads)
        dOh = a2a_seq_to_head(dosh, st.q_heads)
        dQh = []
        for p in range(C):
            kvlist, Kp, Vp, dKp, dVp = kv_state[p]
            kmap = [kvlist.index(h // R) for h in st.q_heads[p]]
            dq, dk, dv = attn_bwd(Qh[p], Kp, Vp, dOh[p], causal, kv_of_head=kmap)
            dKp += dk
            dVp += dv
            dQh.append(dq)
        dQs = a2a_head_to_seq(dQh, st.q_heads, C)
        for r in range(C):
            for h in st.heads:
                dX[r] += dQs[r][h] @ Wq[h * d:(h + 1) * d]
                dW[r]["q"][h * d:(h + 1) * d] += dQs[r][h].T @ Xs[r]
                dW[r]["o"][:, h * d:(h + 1) * d] += dYs[r].T @ Os[r][:, h * d:(h + 1) * d]
    retire(kv_state)
    tot = {k: sum(dW[r][k] for r in range(C)) for k in ("q", "k", "v", "o")}
    return np.concatenate(dX, 0), tot["q"], tot["k"], tot["v"], tot["o"]


# ----------------------------------------------------------------------------
# Ring attention blocks and the UPipe x Ring hybrid (§2.1,
# P:172 "extends to hybrid schemes such as USP")
# ----------------------------------------------------------------------------


def attn_fwd_block(Q, K, V, q_pos0, k_pos0, causal=True, kv_of_head=None):
    """Partial attention of one ring step: query rows at global positions q_pos0 + i
    over the key block at k_pos0 + j ("a local attention ... then exchanges the
    K, V shards among the devices in a ring fashion"). Plain softmax over the block's
    visible keys. Rows that see no key of the block return O = 0 and lse = -inf (the
    empty partial). Returns O [Sq, Hq, d], lse [Hq, Sq]."""
    Sq, Hq, d = Q.shape
    Skv, Hkv, _ = K.shape
    kvh = _kv_map(Hq, Hkv, kv_of_head)
    scale = 1.0 / math.sqrt(d)
    qpos = q_pos0 + np.arange(Sq)
    kpos = k_pos0 + np.arange(Skv)
    vis = (kpos[None, :] <= qpos[:, None]) if causal else np.ones((Sq, Skv), dtype=bool)
    O = np.zeros((Sq, Hq, d))
    lse = np.full((Hq, Sq), -np.inf)
    rows = np.nonzero(vis.any(axis=1))[0]
    if len(rows) == 0:
        return O, lse
    for h in range(Hq):
        g = kvh[h]
        s = (Q[rows, h, :] @ K[:, g, :].T) * scale
        s = np.where(vis[rows], s, -np.inf)
        m = np.max(s, axis=1, keepdims=True)
        l = np.sum(np.exp(s - m), axis=1, keepdims=True)
        lse_b = m + np.log(l)
        O[rows, h, :] = np.exp(s - lse_b) @ V[:, g, :]
        lse[h, rows] = lse_b[:, 0]
    return O, lse


def merge_partials(Oa, lse_a, Ob, lse_b):
    """Ring-step combine ("online softmax compatible version" of §2.1):
    lse' = log(exp(lse_a) + exp(lse_b)) computed with max subtraction;
    O' = exp(lse_a - lse') O_a + exp(lse_b - lse') O_b. O: [S, H, d], lse: [H, S].
    An empty partial (lse = -inf) is the identity."""
    m = np.maximum(lse_a, lse_b)
    m_safe = np.where(np.isfinite(m), m, 0.0)
    wa = np.exp(lse_a - m_safe)                 # exp(-inf) = 0 for an empty side
    wb = np.exp(lse_b - m_safe)
    tot = wa + wb
    lse = np.where(tot > 0, m_safe + np.log(np.where(tot > 0, tot, 1.0)), -np.inf)
    ca = np.where(tot > 0, wa / np.where(tot > 0, tot, 1.0), 0.0)
    cb = np.where(tot > 0, wb / np.where(tot > 0, tot, 1.0), 0.0)
    O = ca.T[:, :, None] * Oa + cb.T[:, :, None] * Ob
    return O, lse


def attn_bwd_block(Q, K, V, dO, lse, Dv, q_pos0, k_pos0, causal=True, kv_of_head=None):
    """Gradient contributions of one ring step (the ring-attention backward): with the
    final (merged) lse of the query rows and D_i = <dO_i, O_i> of the final O,
    P_ij = exp(s_ij - lse_i) on the block's visible pairs, dV_j = sum_i P_ij dO_i,
    dP_ij = <dO_i, V_j>, dS_ij = P_ij (dP_ij - D_i), dQ_i = (1/sqrt d) sum_j dS_ij K_j,
    dK_j = (1/sqrt d) sum_i dS_ij Q_i (S:51-55 restricted to the block's keys; the sums
    over blocks are the un-sharded gradients). lse: [Hq, Sq], Dv: [Sq, Hq].
    Returns (dQ [Sq,Hq,d], dK [Skv,Hkv,d], dV [Skv,Hkv,d])."""
    Sq, Hq, d = Q.shape
    Skv, Hkv, _ = K.shape
    kvh = _kv_map(Hq, Hkv, kv_of_head)
    scale = 1.0 / math.sqrt(d)
    qpos = q_pos0 + np.arange(Sq)
    kpos = k_pos0 + np.arange(Skv)
    vis = (kpos[None, :] <= qpos[:, None]) if causal else np.ones((Sq, Skv), dtype=bool)
    dQ = np.zeros_like(Q)
    dK = np.zeros_like(K)
    dV = np.zeros_like(V)
    for h in range(Hq):
        g = kvh[h]
        s = (Q[:, h, :] @ K[:, g, :].T) * scale
        P = np.where(vis, np.exp(np.where(vis, s, 0.0) - lse[h][:, None]), 0.0)
        dV[:, g, :] += P.T @ dO[:, h, :]
        dP = dO[:, h, :] @ V[:, g, :].T
        dS = P * (dP - Dv[:, h][:, None])
        dQ[:, h, :] = (dS @ K[:, g, :]) * scale
        dK[:, g, :] += (dS.T @ Q[:, h, :]) * scale
    return dQ, dK, dV


def _hybrid_groups(S, a, r):
    """Rank g = i a + u (ring index i, Ulysses index u) holds tokens [g S_l, (g+1) S_l);
    Ulysses group i = ranks i a .. i a + a - 1 holds the contiguous ring block
    [i S_b, (i+1) S_b), S_b = S / r (DESIGN A27)."""
    C = a * r
    if S % C:
        raise ValueError("S % (a r) != 0")
    return S // C, S // r


def hybrid_forward(X, Wq, Wk, Wv, Wo, Hq, Hkv, d, a, r, U, causal=True):
    """UPipe inside each Ulysses group of a ranks, Ring Attention across the r groups
    (USP layout). Per stage (the GQA schedule of the group, C -> a):
    the group's ranks project their shards, inp_all_to_all inside the group gives rank
    (i, u) its heads over ring block i; the ring then visits the K/V blocks
    j = i, i-1, ... (mod r) and merges the partials (merge_partials); blocks j > i are
    invisible under the causal mask. out_all_to_all inside the group; O into the
    pre-allocated output, Y accumulated. Returns (Y [S,D], O [S,Hq d], lse [Hq,S])."""
    S, D = X.shape
    Sl, Sb = _hybrid_groups(S, a, r)
    stages = gqa_schedule(Hq, Hkv, a, U)
    R = Hq // Hkv
    Xs = [X[g * Sl:(g + 1) * Sl] for g in range(a * r)]
    O_buf = [np.zeros((Sl, Hq * d)) for _ in range(a * r)]
    Y_acc = [np.zeros((Sl, D)) for _ in range(a * r)]
    lse_all = np.zeros((Hq, S))
    kv_res = [[None] * a for _ in range(r)]
    for st in stages:
        Qh, Oh = [], []
        for i in range(r):
            grp = [Xs[i * a + u] for u in range(a)]
            qsh = [{h: grp[u] @ Wq[h * d:(h + 1) * d].T for h in st.heads} for u in range(a)]
            Qh.append(a2a_seq_to_head(qsh, st.q_heads))
            if any(st.kv_sent[u] for u in range(a)):
                kv_heads = [st.kv_heads[u] for u in range(a)]
                all_kv = sorted({g for u in range(a) for g in kv_heads[u]})
                ksh = [{g: grp[u] @ Wk[g * d:(g + 1) * d].T for g in all_kv} for u in range(a)]
                vsh = [{g: grp[u] @ Wv[g * d:(g + 1) * d].T for g in all_kv} for u in range(a)]
                Kh, Vh = a2a_seq_to_head(ksh, kv_heads), a2a_seq_to_head(vsh, kv_heads)
                kv_res[i] = [(kv_heads[u], Kh[u], Vh[u]) for u in range(a)]
        for i in range(r):
            Oi = []
            for u in range(a):
                kvlist = kv_res[i][u][0]
                kmap = [kvlist.index(h // R) for h in st.q_heads[u]]
                Oacc, lacc = None, None
                for t in range(r):                       # ring step t: block j = i - t (mod r)
                    j = (i - t) % r
                    _, Kj, Vj = kv_res[j][u]
                    Op, lp = attn_fwd_block(Qh[i][u], Kj, Vj, i * Sb, j * Sb, causal, kmap)
                    Oacc, lacc = (Op, lp) if t == 0 else merge_partials(Oacc, lacc, Op, lp)
                Oi.append(Oacc)
                for jj, h in enumerate(st.q_heads[u]):
                    lse_all[h, i * Sb:(i + 1) * Sb] = lacc[jj]
            Oh.append(Oi)
        for i in range(r):
            Os = a2a_head_to_seq(Oh[i], st.q_heads, a)
            for u in range(a):
                g = i * a + u
                for h in st.heads:
                    O_buf[g][:, h * d:(h + 1) * d] = Os[u][h]
                    Y_acc[g] += Os[u][h] @ Wo[:, h * d:(h + 1) * d].T
    return np.concatenate(Y_acc, 0), np.concatenate(O_buf, 0), lse_all


def hybrid_backward(X, Wq, Wk, Wv, Wo, dY, Hq, Hkv, d, a, r, U, causal=True):
    """Backward of hybrid_forward: per stage the group recomputes Q/K/V and sends
    dO seq->head inside the group; D_i = <dO_i, O_i> from the final O; the ring visits
    the K/V blocks again and each step adds its attn_bwd_block contributions to dQ of the
    local rows and to dK/dV of the visiting block (which travel back to their owner);
    dQ/dK/dV head->seq inside the group; dX, dW as in upipe_backward; dW summed over all
    a r ranks. Returns (dX, dWq, dWk, dWv, dWo)."""
    S, D = X.shape
    Sl, Sb = _hybrid_groups(S, a, r)
    C = a * r
    R = Hq // Hkv
    stages = gqa_schedule(Hq, Hkv, a, U)
    _, O_full, lse_full = hybrid_forward(X, Wq, Wk, Wv, Wo, Hq, Hkv, d, a, r, U, causal)
    Xs = [X[g * Sl:(g + 1) * Sl] for g in range(C)]
    dYs = [dY[g * Sl:(g + 1) * Sl] for g in range(C)]
    Os = [O_full[g * Sl:(g + 1) * Sl] for g in range(C)]
    dX = [np.zeros((Sl, D)) for _ in range(C)]
    dW = dict(q=np.zeros_like(Wq), k=np.zeros_like(Wk), v=np.zeros_like(Wv), o=np.zeros_like(Wo))
    kv_state = [None] * r

    def retire(i):
        heads_of = [s_[0] for s_ in kv_state[i]]
        dKs = a2a_head_to_seq([s_[3] for s_ in kv_state[i]], heads_of, a)
        dVs = a2a_head_to_seq([s_[4] for s_ in kv_state[i]], heads_of, a)
        for u in range(a):
            g = i * a + u
            for kvh in sorted({k for hs in heads_of for k in hs}):
                dX[g] += dKs[u][kvh] @ Wk[kvh * d:(kvh + 1) * d] + dVs[u][kvh] @ Wv[kvh * d:(kvh + 1) * d]
                dW["k"][kvh * d:(kvh + 1) * d] += dKs[u][kvh].T @ Xs[g]
                dW["v"][kvh * d:(kvh + 1) * d] += dVs[u][kvh].T @ Xs[g]

    for st in stages:
        if any(st.kv_sent[u] for u in range(a)):
            for i in range(r):
                if kv_state[i] is not None:
                    retire(i)
                grp = [Xs[i * a + u] for u in range(a)]
                kv_heads = [st.kv_heads[u] for u in range(a)]
                all_kv = sorted({g for u in range(a) for g in kv_heads[u]})
                ksh = [{g: grp[u] @ Wk[g * d:(g + 1) * d].T for g in all_kv} for u in range(a)]
                vsh = [{g: grp[u] @ Wv[g * d:(g + 1) * d].T for g in all_kv} for u in range(a)]
                Kh, Vh = a2a_seq_to_head(ksh, kv_heads), a2a_seq_to_head(vsh, kv_heads)
                kv_state[i] = [(kv_heads[u], Kh[u], Vh[u], np.zeros_like(Kh[u]), np.zeros_like(Vh[u]))
                               for u in range(a)]
        Qh, dOh, Dh = [], [], []
        for i in range(r):
            grp = [i * a + u for u in range(a)]
            qsh = [{h: Xs[g] @ Wq[h * d:(h + 1) * d].T for h in st.heads} for g in grp]
            dosh = [{h: dYs[g] @ Wo[:, h * d:(h + 1) * d] for h in st.heads} for g in grp]
            osh = [{h: Os[g][:, h * d:(h + 1) * d] for h in st.heads} for g in grp]
            Qh.append(a2a_seq_to_head(qsh, st.q_heads))
            dOh.append(a2a_seq_to_head(dosh, st.q_heads))
            Oh = a2a_seq_to_head(osh, st.q_heads)
            Dh.append([rowdot(dOh[i][u], Oh[u]) for u in range(a)])
        dQh = [[None] * a for _ in range(r)]
        for i in range(r):
            for u in range(a):
                kvlist = kv_state[i][u][0]
                kmap = [kvlist.index(h // R) for h in st.q_heads[u]]
                lse_i = np.stack([lse_full[h, i * Sb:(i + 1) * Sb] for h in st.q_heads[u]])
                dq = np.zeros_like(Qh[i][u])
                for t in range(r):
                    j = (i - t) % r
                    _, Kj, Vj, dKj, dVj = kv_state[j][u]
                    bq, bk, bv = attn_bwd_block(Qh[i][u], Kj, Vj, dOh[i][u], lse_i, Dh[i][u],
                                                i * Sb, j * Sb, causal, kmap)
                    dq += bq
                    dKj += bk
                    dVj += bv
                dQh[i][u] = dq
        for i in range(r):
            dQs = a2a_head_to_seq(dQh[i], st.q_heads, a)
            for u in range(a):
                g = i * a + u
                for h in st.heads:
                    dX[g] += dQs[u][h] @ Wq[h * d:(h + 1) * d]
                    dW["q"][h * d:(h + 1) * d] += dQs[u][h].T @ Xs[g]
                    dW["o"][:, h * d:(h + 1) * d] += dYs[g].T @ Os[g][:, h * d:(h + 1) * d]
    for i in range(r):
        retire(i)
    return np.concatenate(dX, 0), dW["q"], dW["k"], dW["v"], dW["o"]


# ----------------------------------------------------------------------------
# Memory accounting (§3.4; DESIGN A21-A22)
# ----------------------------------------------------------------------------


def memory_ulysses_mha(S, C, H, d_head):
    """6 (S/C) H d_head bytes of QKV + the same for a2a buffers = 12 (S/C) H d_head."""
    return 12 * (S // C) * H * d_head


def memory_upipe_mha(S, C, U, d_head):
    """H replaced by U: 12 (S/C) U d_head bytes."""
    return 12 * (S // C) * U * d_head


def intermediate_elems_gqa(S, C, Hq, Hkv, d, U):
    """Per-device forward intermediates (elements, all held): Q/K/V after projection plus
    their a2a receive buffers (DESIGN A22). UPipe holds U q heads and C*kv_res kv heads
    per stage (send side) and the same on the receive side."""
    qpd = U // C
    R = Hq // Hkv
    kv_res = 1 if qpd <= R else qpd // R
    Sl = S // C
    return 2 * Sl * d * (U + 2 * C * kv_res)
