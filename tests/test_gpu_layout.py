"""Bit-exact layout parity of the integer steps of the hot path, through the REAL layer code.

Steps covered: F1's send layout (the projection epilogue) and F2's inp all-to-all
(Q, K, V), F4's out all-to-all and F5's unpack into o_saved, B1/B3's recomputed Q/K/V and dO + delta
all-to-alls, B5's dQ/dK/dV all-to-alls back. upipe_attn_fwd / upipe_attn_bwd run with the test-only
probe of include/upipe.h (receive buffers copied out; head-layout O / dQ / dK / dV injected in place
of the attention kernels), on the single-process fabric at C = 2/4/8, plain UPipe and the ring
hybrid's Ulysses groups, overlapped and sequential schedules.

Expected values come from the oracle only: the projections with one-hot weight rows
(oracle.project, pinned by tests/test_oracle.py::test_project_one_hot_rows_gather_columns_bitwise)
and the oracle's all-to-all maps (oracle.a2a_seq_to_head / a2a_head_to_seq, §3.1) applied
to the head assignment of oracle.gqa_schedule. Payloads are hashed bf16 bit patterns
(synth.payload_bits). Bar: bitwise equality (north_star: "sharding and all-to-all index
permutations bit-exact").
"""
import threading

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import dev

pytestmark = pytest.mark.gpu

ONE = 0x3F80          # bf16 bits of 1.0


def bits_tensor(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16).copy()).view(torch.bfloat16).to(dev())


def tensor_bits(t):
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def vals(bits):
    return synth.from_bf16_bits(bits)


def one_hot_rows(cols, n_cols):
    """W[j, cols[j]] = 1 (nn.Linear [out, in]): X W^T copies input column cols[j] to output column j."""
    W = np.zeros((len(cols), n_cols), dtype=np.uint16)
    W[np.arange(len(cols)), cols] = ONE
    return W


def run_probe(C, ring, S_l, D, Hq, Hkv, d, U, sync, seed=0):
    a = C // ring
    S = C * S_l
    S_b = a * S_l
    qpd = U // a
    rng = np.random.default_rng(seed)
    perm = rng.permutation(D)
    colq = perm[np.arange(Hq * d) % D]
    colk = perm[(Hq * d + np.arange(Hkv * d)) % D]
    colv = perm[(Hq * d + Hkv * d + np.arange(Hkv * d)) % D]
    colo = rng.permutation(D)[np.arange(Hq * d) % D]
    Wq, Wk, Wv = one_hot_rows(colq, D), one_hot_rows(colk, D), one_hot_rows(colv, D)
    Wo = np.ascontiguousarray(one_hot_rows(colo, D).T)            # [D, Hq d]: dO = dY Wo copies columns
    xb = synth.payload_bits(seed, 41, (S, D))
    dyb = synth.payload_bits(seed, 42, (S, D))
    sched = oracle.gqa_schedule(Hq, Hkv, a, U)
    nu = len(sched)
    kv_res = len(sched[0].kv_heads[0])

    from paper_2602_21196_b200 import UPipeAttention, upipe
    fabric = upipe.upipe_fabric_create(C)
    W_t = [bits_tensor(w) for w in (Wq, Wk, Wv, Wo)]
    out = [[None] * nu for _ in range(C)]
    inj = {}
    for g in range(C):
        for s in range(nu):
            inj[g, s] = {"o_head": synth.payload_bits(seed, 1000 + 16 * g + s, (S_b, qpd * d)),
                         "dq_head": synth.payload_bits(seed, 2000 + 16 * g + s, (S_b, qpd * d)),
                         "dk_head": synth.payload_bits(seed, 3000 + 16 * g + s, (S_b, kv_res * d)),
                         "dv_head": synth.payload_bits(seed, 4000 + 16 * g + s, (S_b, kv_res * d))}
    # backward inputs: o_saved with a single 1 per head row (delta = rowsum(dO * O) = dO[t, h d], exact
    # in fp32), lse large so that the un-probed stages' real attention backward sees P = 0
    o_bwd = np.zeros((S_l, Hq * d), dtype=np.uint16)
    o_bwd[:, ::d] = ONE
    errors = []

    def rank_main(g):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                attn = UPipeAttention(Hq, Hkv, d, D, U, True, fabric=fabric, cp_rank=g, cp_size=C, sync_comm=sync,
                                      ring_degree=ring)
                x = bits_tensor(xb[g * S_l:(g + 1) * S_l])
                dy = bits_tensor(dyb[g * S_l:(g + 1) * S_l])
                ob = bits_tensor(o_bwd)
                lse = torch.full((Hq // a, S_b), 30.0, dtype=torch.float32, device=dev())
                for s in range(nu):
                    bf = lambda n: torch.zeros((S_b, n), dtype=torch.bfloat16, device=dev())   # noqa: E731
                    f = {"q_recv": bf(qpd * d), "k_recv": bf(kv_res * d), "v_recv": bf(kv_res * d)}
                    ij = {k: bits_tensor(v) for k, v in inj[g, s].items()}
                    upipe.upipe_test_set_probe(attn.ctx, s, o_head=ij["o_head"], **f)
                    _, saved = attn.forward(x, *W_t)
                    b = {"q_recv": bf(qpd * d), "k_recv": bf(kv_res * d), "v_recv": bf(kv_res * d),
                         "do_recv": bf(qpd * d), "delta_recv": torch.zeros((S_b, qpd), dtype=torch.float32, device=dev()),
                         "dq_recv": bf(qpd * d), "dk_recv": bf(kv_res * d), "dv_recv": bf(kv_res * d)}
                    upipe.upipe_test_set_probe(attn.ctx, s, dq_head=ij["dq_head"], dk_head=ij["dk_head"],
                                               dv_head=ij["dv_head"], **b)
                    attn.backward(x, *W_t, dy, (ob, lse))
                    upipe.upipe_test_set_probe(attn.ctx, -1)
                    stream.synchronize()
                    out[g][s] = {"fwd": {k: tensor_bits(v) for k, v in f.items()}, "o_saved": tensor_bits(saved[0]),
                                 "bwd": {k: (v.cpu().numpy() if v.dtype == torch.float32 else tensor_bits(v))
                                         for k, v in b.items()}}
                attn.close()
        except Exception as e:                          # surfaced below
            errors.append((g, e))

    th = [threading.Thread(target=rank_main, args=(g,)) for g in range(C)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    upipe.upipe_fabric_destroy(fabric)
    if errors:
        raise errors[0][1]

    # ---------------------------------------------------------------- expected, from the oracle
    X, DY = vals(xb), vals(dyb)
    Q = synth.to_bf16_bits(oracle.project(X, vals(Wq)))
    K = synth.to_bf16_bits(oracle.project(X, vals(Wk)))
    V = synth.to_bf16_bits(oracle.project(X, vals(Wv)))
    dO_v = oracle.project(DY, vals(Wo).T)                                 # dY Wo
    dO = synth.to_bf16_bits(dO_v)
    O_b = np.tile(vals(o_bwd), (C, 1))
    delta = oracle.rowdot(dO_v.reshape(S, Hq, d), O_b.reshape(S, Hq, d)).astype(np.float32)   # exact: one product
    checked = 0

    def shards(T, grp, heads, width):
        return [{h: T[r * S_l:(r + 1) * S_l, h * width:(h + 1) * width] for h in heads} for r in grp]

    for i in range(ring):
        grp = [i * a + u for u in range(a)]
        tok = slice(i * S_b, (i + 1) * S_b)
        for s in range(nu):
            st = sched[s]
            heads = st.heads
            kv_sent = any(len(k) for k in st.kv_sent)
            kv_last = s == nu - 1 or any(len(k) for k in sched[s + 1].kv_sent)
            all_kv = sorted({g for k in st.kv_heads for g in k})
            q_full = oracle.a2a_seq_to_head(shards(Q, grp, heads, d), st.q_heads)
            do_full = oracle.a2a_seq_to_head(shards(dO, grp, heads, d), st.q_heads)
            k_full = oracle.a2a_seq_to_head(shards(K, grp, all_kv, d), st.kv_heads)
            v_full = oracle.a2a_seq_to_head(shards(V, grp, all_kv, d), st.kv_heads)
            o_back = oracle.a2a_head_to_seq([inj[g, s]["o_head"].reshape(S_b, qpd, d) for g in grp], st.q_heads, a)
            dq_back = oracle.a2a_head_to_seq([inj[g, s]["dq_head"].reshape(S_b, qpd, d) for g in grp], st.q_heads, a)
            dk_back = oracle.a2a_head_to_seq([inj[g, s]["dk_head"].reshape(S_b, kv_res, d) for g in grp], st.kv_heads, a)
            dv_back = oracle.a2a_head_to_seq([inj[g, s]["dv_head"].reshape(S_b, kv_res, d) for g in grp], st.kv_heads, a)
            for u, g in enumerate(grp):
                got = out[g][s]
                for pas in ("fwd", "bwd"):
                    np.testing.assert_array_equal(got[pas]["q_recv"], q_full[u].reshape(S_b, -1),
                                                  err_msg=f"{pas} Q recv rank {g} stage {s}")
                    if kv_sent:
                        np.testing.assert_array_equal(got[pas]["k_recv"], k_full[u].reshape(S_b, -1),
                                                      err_msg=f"{pas} K recv rank {g} stage {s}")
                        np.testing.assert_array_equal(got[pas]["v_recv"], v_full[u].reshape(S_b, -1),
                                                      err_msg=f"{pas} V recv rank {g} stage {s}")
                np.testing.assert_array_equal(got["bwd"]["do_recv"], do_full[u].reshape(S_b, -1),
                                              err_msg=f"dO recv rank {g} stage {s}")
                np.testing.assert_array_equal(got["bwd"]["delta_recv"], delta[tok][:, st.q_heads[u]],
                                              err_msg=f"delta recv rank {g} stage {s}")
                for h in heads:                       # F4 + F5: this stage's columns of o_saved on rank g
                    np.testing.assert_array_equal(got["o_saved"][:, h * d:(h + 1) * d], o_back[u][h],
                                                  err_msg=f"o_saved rank {g} stage {s} head {h}")
                # B5: block p of the receive buffer = device p's heads, this rank's tokens
                dq_want = np.concatenate([np.concatenate([dq_back[u][h] for h in st.q_heads[p]], 1) for p in range(a)], 0)
                np.testing.assert_array_equal(got["bwd"]["dq_recv"], dq_want, err_msg=f"dQ recv rank {g} stage {s}")
                if kv_last:
                    for name, back in (("dk_recv", dk_back), ("dv_recv", dv_back)):
                        want = np.concatenate([np.concatenate([back[u][h] for h in st.kv_heads[p]], 1)
                                               for p in range(a)], 0)
                        np.testing.assert_array_equal(got["bwd"][name], want, err_msg=f"{name} rank {g} stage {s}")
                checked += 1
    assert checked == C * nu


@pytest.mark.parametrize("C,ring,S_l,D,Hq,Hkv,d,U,sync", [
    (2, 1, 256, 512, 8, 2, 64, 2, False),        # BASELINE configs[0] schedule (CP 2, U 2), overlapped
    (2, 1, 256, 512, 8, 2, 64, 2, True),         # ... sequential (the paper's one buffer set)
    (2, 1, 200, 512, 8, 2, 64, 8, False),        # ragged S_l, Ulysses (U = Hq)
    (4, 1, 128, 2048, 32, 8, 64, 8, False),      # qpd = 2 < R = 4 (sigma = 2)
    (8, 1, 128, 4096, 32, 8, 128, 8, False),     # Llama3-8B at CP 8, U 8 (BASELINE configs[1]/[2] schedule)
    (8, 1, 128, 4096, 32, 8, 128, 16, True),     # ... U 16
    (8, 1, 128, 4096, 32, 8, 128, 32, False),    # ... U 32 (Ulysses), qpd = R
    (8, 1, 128, 5120, 64, 8, 128, 8, False),     # 32B-class (64Q / 8KV, D 5120): BASELINE configs[4] schedule
    (8, 1, 128, 2048, 32, 32, 64, 8, False),     # MHA control (R = 1)
    (4, 1, 128, 1024, 16, 4, 64, 16, False),     # qpd = R = 4: kv_res = 1, sigma = 1
    (4, 1, 128, 1024, 16, 4, 64, 8, True),       # qpd = 2 < R = 4 (sigma = 2), sequential
    (4, 2, 128, 512, 8, 2, 64, 2, True),         # ring hybrid: Ulysses groups of 2 inside a ring of 2
    (8, 2, 128, 1024, 16, 4, 64, 4, True),       # 4 x 2 hybrid
])
def test_layout_bit_exact(C, ring, S_l, D, Hq, Hkv, d, U, sync):
    run_probe(C, ring, S_l, D, Hq, Hkv, d, U, sync)


def test_layout_kv_res_two():
    # qpd = 8 > R = 4: two KV heads resident per device (kv_res = 2), one stage per super-stage
    run_probe(2, 1, 128, 2048, 32, 8, 64, 16, False)
