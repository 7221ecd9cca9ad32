// Shape validation, GQA stage plan and workspace layout (§8b preconditions).
#include <cstdio>

#include "kernels.h"
#include "upipe_internal.h"

namespace upipe {

namespace {
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
}  // namespace

upipe_status_t validate_shape(int C, const upipe_shape_t* sh, std::string& msg) {
  auto bad = [&](upipe_status_t st, const char* what) {
    msg = what;
    return st;
  };
  if (!sh) return bad(UPIPE_ERR_INVALID_ARG, "shape == NULL");
  if (C < 1 || C > 64) return bad(UPIPE_ERR_INVALID_ARG, "cp_size must be in [1, 64]");
  // UPipe x Ring (DESIGN A27): the UPipe constraints below apply to the Ulysses degree a = C / r
  if (sh->ring_degree < 0 || sh->ring_degree > C) return bad(UPIPE_ERR_INVALID_ARG, "ring_degree must be in [0, cp_size]");
  const int ring = sh->ring_degree > 1 ? sh->ring_degree : 1;
  if (C % ring) return bad(UPIPE_ERR_INVALID_ARG, "cp_size % ring_degree != 0 (C = Ulysses degree x ring degree)");
  const int C_total = C;
  C /= ring;
  if (sh->seq_local < 1) return bad(UPIPE_ERR_INVALID_ARG, "seq_local >= 1 required (S = S_l * C, S:239)");
  if (sh->n_q_heads < 1 || sh->n_kv_heads < 1) return bad(UPIPE_ERR_INVALID_ARG, "head counts must be >= 1");
  if (sh->n_q_heads % sh->n_kv_heads) return bad(UPIPE_ERR_INVALID_ARG, "n_q_heads % n_kv_heads != 0 (S:37)");
  if (sh->chunk_heads < 1) return bad(UPIPE_ERR_INVALID_ARG, "chunk_heads >= 1 required");
  if (sh->chunk_heads % C) return bad(UPIPE_ERR_INVALID_ARG, "chunk_heads % cp_size != 0 (P:317: U must be divisible by C)");
  if (sh->n_q_heads % sh->chunk_heads) return bad(UPIPE_ERR_INVALID_ARG, "n_q_heads % chunk_heads != 0 (H/U stages, P:315)");
  if (sh->causal != 0 && sh->causal != 1) return bad(UPIPE_ERR_INVALID_ARG, "causal must be 0 or 1");
  if (!(sh->rope_base == 0.f || (sh->rope_base > 1.f && sh->rope_base < 1e30f)))
    return bad(UPIPE_ERR_INVALID_ARG, "rope_base must be 0 (off) or a finite base > 1 (DESIGN A26)");
  if (!(sh->qk_norm_eps >= 0.f && sh->qk_norm_eps < 1.f))
    return bad(UPIPE_ERR_INVALID_ARG, "qk_norm_eps must be 0 (off) or in (0, 1) (Qwen3: 1e-6; DESIGN A29)");
  if (sh->head_dim != 64 && sh->head_dim != 128) return bad(UPIPE_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  if (sh->hidden < 64 || sh->hidden % 64) return bad(UPIPE_ERR_UNSUPPORTED, "hidden % 64 != 0 (TMA tile granule)");
  if (sh->n_kv_heads % C)
    return bad(UPIPE_ERR_UNSUPPORTED, "n_kv_heads % cp_size != 0 (GQA schedule needs whole kv heads per device, DESIGN A9)");
  const int R = sh->n_q_heads / sh->n_kv_heads;
  const int qpd = sh->chunk_heads / C;
  if (R % qpd && qpd % R)
    return bad(UPIPE_ERR_UNSUPPORTED, "chunk_heads/cp_size and n_q_heads/n_kv_heads must divide one another (DESIGN A8)");
  const int64_t S = sh->seq_local * C_total;
  if (S > (int64_t(1) << 31) - 256) return bad(UPIPE_ERR_UNSUPPORTED, "S >= 2^31 tokens (TMA coordinate range)");
  if ((int64_t)sh->n_q_heads * sh->head_dim > 65536) return bad(UPIPE_ERR_UNSUPPORTED, "n_q_heads*head_dim > 65536");
  msg.clear();
  return UPIPE_OK;
}

Plan make_plan(int C, const upipe_shape_t& sh) {
  Plan p;
  p.ring = sh.ring_degree > 1 ? sh.ring_degree : 1;
  C /= p.ring;                              // the UPipe stage loop runs inside a Ulysses group of a = C / r ranks
  p.C = C;
  p.sh = sh;
  p.S_l = sh.seq_local;
  p.S = sh.seq_local * C;                   // tokens of the group's ring block (all tokens when r = 1)
  p.Hq = sh.n_q_heads;
  p.Hkv = sh.n_kv_heads;
  p.d = sh.head_dim;
  p.D = sh.hidden;
  p.U = sh.chunk_heads;
  p.R = p.Hq / p.Hkv;
  p.qpd = p.U / C;
  p.kv_res = p.qpd > p.R ? p.qpd / p.R : 1;
  p.sigma = p.qpd < p.R ? p.R / p.qpd : 1;
  p.nstages = p.Hq / p.U;
  return p;
}

FwdWs fwd_workspace(const Plan& p, bool overlap, bool direct) {
  // overlap (C > 1): the next stage's inp all-to-all runs while this stage's attention reads its
  // buffers, so the Q/K/V receive, Q send and O send/receive buffers are doubled (DESIGN A23).
  FwdWs w{};
  const size_t qe = (size_t)p.S * p.qpd * p.d * 2;     // one Q-sized chunk, bf16
  const size_t ke = (size_t)p.S * p.kv_res * p.d * 2;  // one K-sized chunk, bf16
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align256(bytes);
    return o;
  };
  // UPIPE_FLAG_DIRECT: producers write the peers' receive buffers, so no send buffer is allocated (the
  // offset 0 placeholders are never used)
  direct = direct && p.C > 1;
  auto take_send = [&](size_t bytes) { return direct ? size_t(0) : take(bytes); };
  const bool comm = p.C > 1;
  const bool dbl = comm && overlap;
  for (int i = 0; i < 2; ++i) {
    const bool fresh = i == 0 || dbl;
    w.qsend[i] = fresh ? take_send(qe) : w.qsend[0];
    w.qrecv[i] = !comm ? w.qsend[i] : (fresh ? take(qe) : w.qrecv[0]);
  }
  w.ksend = take_send(ke);
  w.vsend = take_send(ke);
  for (int i = 0; i < 2; ++i) {
    const bool fresh = i == 0 || dbl;
    w.krecv[i] = !comm ? w.ksend : (fresh ? take(ke) : w.krecv[0]);
    w.vrecv[i] = !comm ? w.vsend : (fresh ? take(ke) : w.vrecv[0]);
    w.osend[i] = !comm ? 0 : (fresh ? take_send(qe) : w.osend[0]);
    w.orecv[i] = !comm ? 0 : (fresh ? take(qe) : w.orecv[0]);
  }
  if (p.ring > 1) {                         // ring hybrid (sequential schedule): visiting K/V blocks, fp32 O
    for (int i = 0; i < 2; ++i) {
      w.kring[i] = take(ke);
      w.vring[i] = take(ke);
    }
    w.oacc = take(qe * 2);
    w.opart = take(qe * 2);
    w.lsepart = take((size_t)p.S * p.qpd * 4);
  }
  w.total = off;
  return w;
}

BwdWs bwd_workspace(const Plan& p, bool overlap, bool direct) {
  BwdWs w{};
  const size_t qe = (size_t)p.S * p.qpd * p.d * 2;
  const size_t ke = (size_t)p.S * p.kv_res * p.d * 2;
  const size_t de = (size_t)p.S * p.qpd * 4;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align256(bytes);
    return o;
  };
  // UPIPE_FLAG_DIRECT: producers write the peers' receive buffers, so no send buffer is allocated (the
  // offset 0 placeholders are never used)
  direct = direct && p.C > 1;
  auto take_send = [&](size_t bytes) { return direct ? size_t(0) : take(bytes); };
  const bool comm = p.C > 1;
  const bool dbl = comm && overlap;
  for (int i = 0; i < 2; ++i) {
    const bool fresh = i == 0 || dbl;
    w.qsend[i] = fresh ? take_send(qe) : w.qsend[0];
    w.qrecv[i] = !comm ? w.qsend[i] : (fresh ? take(qe) : w.qrecv[0]);
    w.dosend[i] = fresh ? take_send(qe) : w.dosend[0];
    w.dorecv[i] = !comm ? w.dosend[i] : (fresh ? take(qe) : w.dorecv[0]);
    w.dsend[i] = fresh ? take_send(de) : w.dsend[0];
    w.drecv[i] = !comm ? w.dsend[i] : (fresh ? take(de) : w.drecv[0]);
    // fp32 dQ accumulator: [S][qpd d], or dim-major [qpd d][S4] (S4 = S rounded up to 4 floats, TMA stride)
    w.dqacc[i] = fresh ? take(((size_t)p.S + 3) / 4 * 4 * p.qpd * p.d * 4) : w.dqacc[0];
    w.dqsend[i] = fresh ? take_send(qe) : w.dqsend[0];
    w.dqrecv[i] = !comm ? w.dqsend[i] : (fresh ? take(qe) : w.dqrecv[0]);
  }
  w.ksend = take_send(ke);
  w.vsend = take_send(ke);
  for (int i = 0; i < 2; ++i) {
    const bool fresh = i == 0 || dbl;
    w.krecv[i] = !comm ? w.ksend : (fresh ? take(ke) : w.krecv[0]);
    w.vrecv[i] = !comm ? w.vsend : (fresh ? take(ke) : w.vrecv[0]);
  }
  w.dkacc = p.sigma > 1 || p.ring > 1 ? take(ke * 2) : 0;
  w.dvacc = p.sigma > 1 || p.ring > 1 ? take(ke * 2) : 0;
  if (p.ring > 1) {                         // visiting K/V blocks and their travelling fp32 dK/dV accumulators
    for (int i = 0; i < 2; ++i) {
      w.kring[i] = take(ke);
      w.vring[i] = take(ke);
      w.dkring[i] = take(ke * 2);
      w.dvring[i] = take(ke * 2);
    }
  }
  w.dksend = take_send(ke);
  w.dvsend = take_send(ke);
  w.dkrecv = comm ? take(ke) : w.dksend;
  w.dvrecv = comm ? take(ke) : w.dvsend;
  // dX: the pre-allocated gradient buffer G [S_l][(Hq + 2 Hkv) d] bf16 (DESIGN A30), or with the naive
  // ablation the fp32 accumulator [S_l][D] (one stage: dX is stored in bf16 directly)
  w.gbuf = p.gbuf() ? take((size_t)p.S_l * (p.Hq + 2 * p.Hkv) * p.d * 2) : 0;
  w.dxacc = !p.gbuf() && p.nstages > 1 ? take((size_t)p.S_l * p.D * 4) : 0;
  if (p.sh.qk_norm_eps > 0.f) {             // Qwen3 q/k norm (DESIGN A29): normalised copies for the attention
    for (int i = 0; i < 2; ++i) {           // (the receive buffers keep the pre-norm heads for the chain rule),
      const bool fresh = i == 0 || dbl;     // fp32 dK for the fused norm backward, d(gamma) scratch
      w.qn[i] = fresh ? take(qe) : w.qn[0];
      w.kn[i] = fresh ? take(ke) : w.kn[0];
    }
    if (!w.dkacc) w.dkacc = take(ke * 2);
    w.dgam = take((size_t)(2 + kNormBwdMaxBlocks) * p.d * 4);   // d(gamma_q), d(gamma_k), det partials
  }
  w.dqsem = take((size_t)attn_bwd_sem_count(p.S, p.qpd) * 4);     // deterministic mode (a few hundred KB)
  w.total = off;
  return w;
}

}  // namespace upipe
