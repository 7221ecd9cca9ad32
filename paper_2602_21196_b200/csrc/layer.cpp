// UPipe stage loops (SURVEY §8a F0-F7 forward, B1-B8 backward).
// P:310-330 §3.3 (stage loop, buffer reuse, pre-allocated output), P:355 (Q, K, V
// all-to-alls issued one after the other), §4.1 (KV sent once per
// super-stage), Table 4 P:686 (backward order: dO seq->head, attention backward,
// dQ/dK/dV head->seq), P:439 (projections recomputed in backward).
#include <cstdio>

#include "kernels.h"
#include "upipe_internal.h"

namespace upipe {

namespace {

using bf16p = const upipe_bf16*;

struct Err {
  upipe_ctx_s* ctx;
  upipe_status_t fail(upipe_status_t st, const std::string& msg) {
    ctx->last_error = msg;
    return st;
  }
};

#define UP_CUDA(expr)                                                             \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess)                                                        \
      return E.fail(UPIPE_ERR_CUDA, std::string(#expr ": ") + (errbuf[0] ? errbuf : cudaGetErrorString(_e))); \
  } while (0)

// Brackets one step with trace events on the call's stream (no-op when tracing is off).
struct Step {
  upipe_ctx_s* ctx;
  cudaStream_t st;
  int cat;
  cudaEvent_t a = nullptr;
  Step(upipe_ctx_s* c, cudaStream_t s, int k) : ctx(c), st(s), cat(k) {
    if (ctx->tracer.on) {
      a = ctx->tracer.get();
      cudaEventRecord(a, st);
    }
  }
  ~Step() {
    if (a) {
      cudaEvent_t b = ctx->tracer.get();
      cudaEventRecord(b, st);
      ctx->tracer.recs.push_back({cat, a, b});
    }
  }
};

#define UP_T(cat, macro, expr)            \
  do {                                    \
    Step _step(ctx, st, UPIPE_TRACE_##cat); \
    macro(expr);                          \
  } while (0)

#define UP_COMM(expr)                                  \
  do {                                                 \
    std::string _m;                                    \
    upipe_status_t _s = (expr);                        \
    if (_s != UPIPE_OK) return E.fail(_s, _m.empty() ? std::string(#expr) : _m); \
  } while (0)

// Projection of this rank's shard for the stage's heads, written straight into the
// all-to-all send layout [C][S_l][seg] (pack fused into the GEMM epilogue).
//   W rows of device p's heads start at row0 + p * row_step; seg = heads_per_device * d.
GemmProblem proj_to_send(const Plan& P, const void* x, const void* W, int64_t W_rows, int64_t row0,
                         int64_t row_step, int64_t seg, void* send) {
  GemmProblem g;
  g.M = P.S_l;
  g.N = (int64_t)P.C * seg;
  g.K = P.D;
  g.a = OperandMap{x, P.D, P.S_l, P.D, false};
  g.b = OperandMap{W, P.D, W_rows, P.D, false};
  g.b.o_base = row0;
  g.b.o_len = seg;
  g.b.o_istride = row_step;
  g.c.out_bf16 = send;
  g.c.ld_bf16 = seg;
  g.c.n_len = seg;
  g.c.r_nstride = P.S_l;
  g.c.epi = Epi::kStoreBF16;
  return g;
}

}  // namespace

upipe_status_t layer_fwd(upipe_ctx_s* ctx, const Plan& P, bf16p x, bf16p wq, bf16p wk, bf16p wv, bf16p wo,
                         upipe_bf16* y, upipe_bf16* o_saved, float* lse_saved, char* ws, cudaStream_t st) {
  Err E{ctx};
  char errbuf[512] = {0};
  Transport& T = *ctx->transport;
  const FwdWs W = fwd_workspace(P);
  const int C = P.C, me = ctx->rank, d = P.d;
  const int64_t qseg = (int64_t)P.qpd * d, kseg = (int64_t)P.kv_res * d;
  const int64_t HqD = (int64_t)P.Hq * d;
  const size_t qbytes = (size_t)P.S_l * qseg * 2, kbytes = (size_t)P.S_l * kseg * 2;
  for (int s = 0; s < P.nstages; ++s) {
    const int64_t q0 = P.q0(s, 0), kv0 = P.kv0(s, 0);
    const int64_t qstep = (int64_t)P.q_dev_stride() * d;
    // F1: Q_s = x Wq[rows(s)]^T -> send layout
    UP_T(GEMM, UP_CUDA, gemm_run(proj_to_send(P, x, wq, HqD, q0 * d, qstep, qseg, ws + W.qsend), st, errbuf, sizeof errbuf));
    // F2: inp_all_to_all, Q first, then K and V when this stage starts a super-stage
    UP_T(COMM, UP_COMM, T.alltoall(ws + W.qsend, ws + W.qrecv, qbytes, st, _m));
    if (P.kv_sent(s)) {
      const int64_t kvrows = (int64_t)P.Hkv * d;
      UP_T(GEMM, UP_CUDA, gemm_run(proj_to_send(P, x, wk, kvrows, kv0 * d, kseg, kseg, ws + W.ksend), st, errbuf, sizeof errbuf));
      UP_T(COMM, UP_COMM, T.alltoall(ws + W.ksend, ws + W.krecv, kbytes, st, _m));
      UP_T(GEMM, UP_CUDA, gemm_run(proj_to_send(P, x, wv, kvrows, kv0 * d, kseg, kseg, ws + W.vsend), st, errbuf, sizeof errbuf));
      UP_T(COMM, UP_COMM, T.alltoall(ws + W.vsend, ws + W.vrecv, kbytes, st, _m));
    }
    // F3: attention over the full sequence for this device's qpd heads
    AttnFwdProblem a{};
    a.q = ws + W.qrecv;
    a.k = ws + W.krecv;
    a.v = ws + W.vrecv;
    const int64_t my_q0 = P.q0(s, me);
    if (C == 1) {
      a.o = o_saved + my_q0 * d;  // no out all-to-all: write straight into the pre-allocated output
      a.ldo = HqD;
    } else {
      a.o = ws + W.osend;
      a.ldo = qseg;
    }
    a.lse = lse_saved + (int64_t)s * P.qpd * P.S;
    a.S = P.S;
    a.nq = P.qpd;
    a.nkv = P.kv_res;
    a.d = d;
    a.causal = P.sh.causal;
    a.ldq = qseg;
    a.ldkv = kseg;
    a.ld_lse = P.S;
    UP_T(ATTN_FWD, UP_CUDA, attn_fwd_run(a, st, errbuf, sizeof errbuf));
    if (C > 1) {
      // F4: out_all_to_all, F5: fill the pre-allocated output o_saved
      UP_T(COMM, UP_COMM, T.alltoall(ws + W.osend, ws + W.orecv, qbytes, st, _m));
      UP_T(AUX, UP_CUDA, unpack_cols_run(ws + W.orecv, P.S_l, C, (int)qseg, o_saved, HqD, q0 * d, qstep, st));
    }
    // F6: y (+)= O_s Wo[:, cols(s)]^T ; fp32 accumulator across stages, bf16 on the last stage (F7 fused)
    GemmProblem g;
    g.M = P.S_l;
    g.N = P.D;
    g.K = (int64_t)P.U * d;
    g.a = OperandMap{o_saved, HqD, P.S_l, HqD, false};
    g.b = OperandMap{wo, HqD, P.D, HqD, false};
    for (OperandMap* m : {&g.a, &g.b}) {
      m->k_base = q0 * d;
      m->k_len = qseg;
      m->k_kstride = qstep;
    }
    g.c.out_f32 = ws + W.yacc;
    g.c.ld_f32 = P.D;
    g.c.out_bf16 = y;
    g.c.ld_bf16 = P.D;
    if (P.nstages == 1) g.c.epi = Epi::kStoreBF16;
    else if (s == 0) g.c.epi = Epi::kStoreF32;
    else if (s == P.nstages - 1) g.c.epi = Epi::kAccF32ToBF16;
    else g.c.epi = Epi::kAccF32;
    UP_T(GEMM, UP_CUDA, gemm_run(g, st, errbuf, sizeof errbuf));
  }
  return UPIPE_OK;
}

upipe_status_t layer_bwd(upipe_ctx_s* ctx, const Plan& P, bf16p x, bf16p wq, bf16p wk, bf16p wv, bf16p wo,
                         bf16p dy, bf16p o_saved, const float* lse_saved, upipe_bf16* dx, float* dwq, float* dwk,
                         float* dwv, float* dwo, int reduce_dw, char* ws, cudaStream_t st) {
  Err E{ctx};
  char errbuf[512] = {0};
  Transport& T = *ctx->transport;
  const BwdWs W = bwd_workspace(P);
  const int C = P.C, d = P.d;
  const int64_t qseg = (int64_t)P.qpd * d, kseg = (int64_t)P.kv_res * d;
  const int64_t HqD = (int64_t)P.Hq * d, HkvD = (int64_t)P.Hkv * d;
  const size_t qbytes = (size_t)P.S_l * qseg * 2, kbytes = (size_t)P.S_l * kseg * 2;
  const int64_t qstep = (int64_t)P.q_dev_stride() * d;

  // dWo = dY^T O over this rank's tokens (all stages at once: o_saved holds every head)
  {
    GemmProblem g;
    g.M = P.D;
    g.N = HqD;
    g.K = P.S_l;
    g.a = OperandMap{dy, P.D, P.S_l, P.D, true};
    g.b = OperandMap{o_saved, HqD, P.S_l, HqD, true};
    g.c.out_f32 = dwo;
    g.c.ld_f32 = HqD;
    g.c.epi = Epi::kStoreF32;
    UP_T(GEMM, UP_CUDA, gemm_run(g, st, errbuf, sizeof errbuf));
  }
  const int n_dx_terms = P.nstages + 2 * (P.nstages / P.sigma);
  int dx_term = 0;
  auto dx_epi = [&](GemmProblem& g) {
    g.c.out_f32 = ws + W.dxacc;
    g.c.ld_f32 = P.D;
    g.c.out_bf16 = dx;
    g.c.ld_bf16 = P.D;
    g.c.epi = dx_term == 0 ? Epi::kStoreF32 : (dx_term == n_dx_terms - 1 ? Epi::kAccF32ToBF16 : Epi::kAccF32);
    ++dx_term;
  };
  // dX += dG_s W_s (G = Q, K or V): A = received gradient [C][S_l][seg], B = W rows (MN-major)
  auto dx_gemm = [&](const void* grecv, int64_t seg, const void* Wt, int64_t W_rows, int64_t row0, int64_t row_step) {
    GemmProblem g;
    g.M = P.S_l;
    g.N = P.D;
    g.K = (int64_t)C * seg;
    g.a = OperandMap{grecv, seg, (int64_t)C * P.S_l, seg, false};
    g.a.k_len = seg;
    g.a.k_kstride = 0;
    g.a.o_kstride = P.S_l;
    g.b = OperandMap{Wt, P.D, W_rows, P.D, true};
    g.b.k_base = row0;
    g.b.k_len = seg;
    g.b.k_kstride = row_step;
    dx_epi(g);
    return g;
  };
  // dW rows of the stage's heads: dW[row0 + p*row_step + j][:] = sum_t grecv[p][t][j] x[t][:]
  auto dw_gemm = [&](const void* grecv, int64_t seg, float* dW, int64_t row0, int64_t row_step) {
    GemmProblem g;
    g.M = (int64_t)C * seg;
    g.N = P.D;
    g.K = P.S_l;
    g.a = OperandMap{grecv, seg, (int64_t)C * P.S_l, seg, true};
    g.a.o_len = seg;
    g.a.o_istride = 0;
    g.a.k_istride = P.S_l;
    g.b = OperandMap{x, P.D, P.S_l, P.D, true};
    g.c.out_f32 = dW;
    g.c.ld_f32 = P.D;
    g.c.r_base = row0;
    g.c.m_len = seg;
    g.c.r_mstride = row_step;
    g.c.epi = Epi::kStoreF32;
    return g;
  };

  for (int s = 0; s < P.nstages; ++s) {
    const int64_t q0 = P.q0(s, 0), kv0 = P.kv0(s, 0);
    // B1: recompute the stage's projections and inp_all_to_all
    UP_T(GEMM, UP_CUDA, gemm_run(proj_to_send(P, x, wq, HqD, q0 * d, qstep, qseg, ws + W.qsend), st, errbuf, sizeof errbuf));
    UP_T(COMM, UP_COMM, T.alltoall(ws + W.qsend, ws + W.qrecv, qbytes, st, _m));
    if (P.kv_sent(s)) {
      UP_T(GEMM, UP_CUDA, gemm_run(proj_to_send(P, x, wk, HkvD, kv0 * d, kseg, kseg, ws + W.ksend), st, errbuf, sizeof errbuf));
      UP_T(COMM, UP_COMM, T.alltoall(ws + W.ksend, ws + W.krecv, kbytes, st, _m));
      UP_T(GEMM, UP_CUDA, gemm_run(proj_to_send(P, x, wv, HkvD, kv0 * d, kseg, kseg, ws + W.vsend), st, errbuf, sizeof errbuf));
      UP_T(COMM, UP_COMM, T.alltoall(ws + W.vsend, ws + W.vrecv, kbytes, st, _m));
    }
    // B2: dO_s = dY Wo[:, cols(s)] straight into the send layout; delta = rowsum(dO*O) (A13)
    {
      GemmProblem g;
      g.M = P.S_l;
      g.N = (int64_t)C * qseg;
      g.K = P.D;
      g.a = OperandMap{dy, P.D, P.S_l, P.D, false};
      g.b = OperandMap{wo, HqD, P.D, HqD, true};
      g.b.o_base = q0 * d;
      g.b.o_len = qseg;
      g.b.o_istride = qstep;
      g.c.out_bf16 = ws + W.dosend;
      g.c.ld_bf16 = qseg;
      g.c.n_len = qseg;
      g.c.r_nstride = P.S_l;
      g.c.epi = Epi::kStoreBF16;
      UP_T(GEMM, UP_CUDA, gemm_run(g, st, errbuf, sizeof errbuf));
      for (int p = 0; p < C; ++p)
        UP_T(AUX, UP_CUDA, rowdot_run((const upipe_bf16*)(ws + W.dosend) + (int64_t)p * P.S_l * qseg, qseg,
                           o_saved + (int64_t)P.q0(s, p) * d, HqD, (float*)(ws + W.dsend) + (int64_t)p * P.S_l * P.qpd,
                           P.qpd, P.S_l, P.qpd, d, st));
    }
    // B3: dO and delta seq->head ("during out_all_to_all", Table 4)
    UP_T(COMM, UP_COMM, T.alltoall(ws + W.dosend, ws + W.dorecv, qbytes, st, _m));
    UP_T(COMM, UP_COMM, T.alltoall(ws + W.dsend, ws + W.drecv, (size_t)P.S_l * P.qpd * 4, st, _m));
    // B4: attention backward; dK/dV accumulate over the sigma stages sharing the resident K/V
    UP_T(AUX, UP_CUDA, cudaMemsetAsync(ws + W.dqacc, 0, (size_t)P.S * qseg * 4, st));
    const int r = s % P.sigma;
    const bool last = P.kv_last(s);
    AttnBwdProblem b{};
    b.q = ws + W.qrecv;
    b.k = ws + W.krecv;
    b.v = ws + W.vrecv;
    b.dout = ws + W.dorecv;
    b.lse = lse_saved + (int64_t)s * P.qpd * P.S;
    b.delta = (const float*)(ws + W.drecv);
    b.dq_acc = (float*)(ws + W.dqacc);
    b.dk_acc = P.sigma > 1 ? (float*)(ws + W.dkacc) : nullptr;
    b.dv_acc = P.sigma > 1 ? (float*)(ws + W.dvacc) : nullptr;
    b.dk_bf16 = last ? ws + W.dksend : nullptr;
    b.dv_bf16 = last ? ws + W.dvsend : nullptr;
    b.S = P.S;
    b.nq = P.qpd;
    b.nkv = P.kv_res;
    b.d = d;
    b.causal = P.sh.causal;
    b.ldq = qseg;
    b.ldkv = kseg;
    b.ldo_grad = qseg;
    b.ld_lse = P.S;
    b.ld_delta = P.qpd;
    b.ld_kvb = kseg;
    b.kv_accumulate = r > 0;
    b.kv_write_acc = !last;
    UP_T(ATTN_BWD, UP_CUDA, attn_bwd_run(b, st, errbuf, sizeof errbuf));
    // B5: dQ fp32 -> bf16 send layout, head->seq ("during inp_all_to_all")
    UP_T(AUX, UP_CUDA, cvt_f32_bf16_run((const float*)(ws + W.dqacc), qseg, ws + W.dqsend, qseg, P.S, qseg, 1.0f, st));
    UP_T(COMM, UP_COMM, T.alltoall(ws + W.dqsend, ws + W.dqrecv, qbytes, st, _m));
    // B6: dX and dWq for the stage's q heads
    UP_T(GEMM, UP_CUDA, gemm_run(dx_gemm(ws + W.dqrecv, qseg, wq, HqD, q0 * d, qstep), st, errbuf, sizeof errbuf));
    UP_T(GEMM, UP_CUDA, gemm_run(dw_gemm(ws + W.dqrecv, qseg, dwq, q0 * d, qstep), st, errbuf, sizeof errbuf));
    if (last) {
      // retire the super-stage's K/V: dK, dV head->seq, then their dX / dW terms
      UP_T(COMM, UP_COMM, T.alltoall(ws + W.dksend, ws + W.dkrecv, kbytes, st, _m));
      UP_T(COMM, UP_COMM, T.alltoall(ws + W.dvsend, ws + W.dvrecv, kbytes, st, _m));
      UP_T(GEMM, UP_CUDA, gemm_run(dx_gemm(ws + W.dkrecv, kseg, wk, HkvD, kv0 * d, kseg), st, errbuf, sizeof errbuf));
      UP_T(GEMM, UP_CUDA, gemm_run(dx_gemm(ws + W.dvrecv, kseg, wv, HkvD, kv0 * d, kseg), st, errbuf, sizeof errbuf));
      UP_T(GEMM, UP_CUDA, gemm_run(dw_gemm(ws + W.dkrecv, kseg, dwk, kv0 * d, kseg), st, errbuf, sizeof errbuf));
      UP_T(GEMM, UP_CUDA, gemm_run(dw_gemm(ws + W.dvrecv, kseg, dwv, kv0 * d, kseg), st, errbuf, sizeof errbuf));
    }
  }
  // B7: dW summed over the CP group (the FSDP gradient reduction of P:437, A14)
  if (reduce_dw && C > 1) {
    UP_T(COMM, UP_COMM, T.allreduce_sum_f32(dwq, (size_t)HqD * P.D, st, _m));
    UP_T(COMM, UP_COMM, T.allreduce_sum_f32(dwk, (size_t)HkvD * P.D, st, _m));
    UP_T(COMM, UP_COMM, T.allreduce_sum_f32(dwv, (size_t)HkvD * P.D, st, _m));
    UP_T(COMM, UP_COMM, T.allreduce_sum_f32(dwo, (size_t)HqD * P.D, st, _m));
  }
  return UPIPE_OK;
}

}  // namespace upipe
