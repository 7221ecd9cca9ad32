// UPipe stage loops (SURVEY §8a F0-F7 forward, B1-B8 backward).
// P:310-330 §3.3 (stage loop, buffer reuse, pre-allocated output), P:355 (Q, K, V
// all-to-alls issued one after the other), §4.1 (KV sent once per
// super-stage), Table 4 P:686 (backward order: dO seq->head, attention backward,
// dQ/dK/dV head->seq), P:439 (projections recomputed in backward).
//
// Two schedules run the same per-stage steps:
//  * sequential (C == 1, or UPIPE_FLAG_SYNC_COMM): one buffer set, everything on the
//    caller's stream: the paper's memory-minimal form;
//  * overlapped (C > 1, default): the next stage's projections are issued before the
//    current stage's attention and its all-to-all runs on the ctx's high-priority comm
//    stream, so it overlaps the attention (north_star: "the next chunk's NCCL
//    all-to-all over NVLink is overlapped on a side stream with the current chunk's
//    attention"); the out all-to-all of stage s overlaps attention s+1. Costs a second
//    buffer set (DESIGN A23). Cross-stream order is carried by CUDA events.
#include <cmath>
#include <cstdio>
#include <vector>
#include <cstdlib>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost nothing unless a profiler injects itself

#include "kernels.h"
#include "upipe_internal.h"

namespace upipe {

namespace {

using bf16p = const upipe_bf16*;

// Brackets one step with trace events on the stream it runs on (no-op when tracing is off) and an NVTX range
// named after the step (host-side enqueue range; nsys / ncu correlate the step's launches with it).
struct Step {
  upipe_ctx_s* ctx;
  cudaStream_t st;
  int cat;
  const char* label;
  cudaEvent_t a = nullptr;
  Step(upipe_ctx_s* c, cudaStream_t s, int k, const char* l = "") : ctx(c), st(s), cat(k), label(l) {
    nvtxRangePushA(label && label[0] ? label : "upipe step");
    if (ctx->tracer.on) {
      a = ctx->tracer.get();
      cudaEventRecord(a, st);
    }
  }
  ~Step() {
    nvtxRangePop();
    if (a) {
      cudaEvent_t b = ctx->tracer.get();
      cudaEventRecord(b, st);
      ctx->tracer.recs.push_back({cat, a, b, label});
    }
  }
};

bool debug_sync() {
  static const bool on = [] {
    const char* e = getenv("UPIPE_DEBUG_SYNC");
    return e && e[0] == '1';
  }();
  return on;
}

// Runs one step, reports failures into ctx->last_error.
struct Runner {
  upipe_ctx_s* ctx;
  upipe_status_t status = UPIPE_OK;
  char errbuf[512] = {0};
  template <class F>
  bool run(int cat, cudaStream_t s, const char* what, F&& f) {
    if (status != UPIPE_OK) return false;
    Step step(ctx, s, cat, what);
    errbuf[0] = 0;
    cudaError_t e = f(errbuf);
    if (debug_sync()) {                  // UPIPE_DEBUG_SYNC=1: synchronise and log every step (hang triage)
      fprintf(stderr, "[upipe step] %s ...", what);
      cudaError_t e2 = cudaStreamSynchronize(s);
      fprintf(stderr, " %s\n", cudaGetErrorString(e2));
      if (e == cudaSuccess) e = e2;
    }
    if (e != cudaSuccess) {
      ctx->last_error = std::string(what) + ": " + (errbuf[0] ? errbuf : cudaGetErrorString(e));
      status = UPIPE_ERR_CUDA;
      return false;
    }
    return true;
  }
  template <class F>
  bool comm(cudaStream_t s, const char* what, F&& f) {
    if (status != UPIPE_OK) return false;
    Step step(ctx, s, UPIPE_TRACE_COMM, what);
    std::string m;
    upipe_status_t st = f(m);
    if (st != UPIPE_OK) {
      ctx->last_error = std::string(what) + ": " + m;
      status = st;
      return false;
    }
    return true;
  }
};

// Projection of this rank's shard for the stage's heads, written straight into the
// all-to-all send layout [C][S_l][seg] (pack fused into the GEMM epilogue).
//   W rows of device p's heads start at row0 + p * row_step; seg = heads_per_device * d.
GemmProblem proj_to_send(const Plan& P, const void* x, const void* W, int64_t W_rows, int64_t row0,
                         int64_t row_step, int64_t seg, void* send, const RopeRef& rope = RopeRef{}) {
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
  g.c.rope = rope;                       // Q/K: rotary embedding at the tokens' global positions
  return g;
}

// RoPE tables for angles p * base^(-2i/d), p < S (DESIGN A26): computed in double on the host once.
upipe_status_t ensure_rope(upipe_ctx_s* ctx, const Plan& P, RopeRef& ref) {
  ref = RopeRef{};
  if (P.sh.rope_base == 0.f) return UPIPE_OK;
  RopeTables& T = ctx->rope;
  const int64_t n_hi = (P.S * P.ring + 1023) / 1024;     // positions of the whole sequence (all ring blocks)
  if (T.base != P.sh.rope_base || T.d != P.d || T.n_hi < n_hi) {
    if (T.hi) cudaFree(T.hi);
    if (T.lo) cudaFree(T.lo);
    T.hi = T.lo = nullptr;
    const int h2 = P.d / 2;
    std::vector<float2> hi((size_t)n_hi * h2), lo((size_t)1024 * h2);
    const double two_pi = 6.283185307179586476925286766559;
    for (int i = 0; i < h2; ++i) {
      const double f = std::pow((double)P.sh.rope_base, -2.0 * i / P.d);
      for (int64_t h = 0; h < n_hi; ++h) {
        const double a = std::fmod((double)h * 1024.0 * f, two_pi);
        hi[(size_t)h * h2 + i] = make_float2((float)std::cos(a), (float)std::sin(a));
      }
      for (int l = 0; l < 1024; ++l) {
        const double a = (double)l * f;
        lo[(size_t)l * h2 + i] = make_float2((float)std::cos(a), (float)std::sin(a));
      }
    }
    if (cudaMalloc(&T.hi, hi.size() * sizeof(float2)) != cudaSuccess ||
        cudaMalloc(&T.lo, lo.size() * sizeof(float2)) != cudaSuccess ||
        cudaMemcpy(T.hi, hi.data(), hi.size() * sizeof(float2), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(T.lo, lo.data(), lo.size() * sizeof(float2), cudaMemcpyHostToDevice) != cudaSuccess) {
      ctx->last_error = "cannot build the RoPE tables";
      return UPIPE_ERR_CUDA;
    }
    T.base = P.sh.rope_base;
    T.d = P.d;
    T.n_hi = n_hi;
  }
  ref.hi = T.hi;
  ref.lo = T.lo;
  ref.d = P.d;
  ref.pos0 = 0;
  return UPIPE_OK;
}

upipe_status_t ensure_pipe(upipe_ctx_s* ctx) {
  Pipe& p = ctx->pipe;
  if (p.ready) return UPIPE_OK;
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (cudaStreamCreateWithPriority(&p.comm, cudaStreamNonBlocking, hi) != cudaSuccess) {
    ctx->last_error = "cannot create the comm stream";
    return UPIPE_ERR_CUDA;
  }
  for (auto& e : p.ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      ctx->last_error = "cannot create pipeline events";
      return UPIPE_ERR_CUDA;
    }
  p.ready = true;
  return UPIPE_OK;
}

// Test-only layout probe copies (upipe_test_set_probe): no-op for a null destination.
cudaError_t probe_copy(void* dst, const void* src, size_t bytes, cudaStream_t q) {
  if (!dst || !src || bytes == 0) return cudaSuccess;
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, q);
}

// UPIPE_FLAG_DIRECT: checks the transport can write peer memory.
upipe_status_t check_direct(upipe_ctx_s* ctx, const Plan& P) {
  if (!direct_enabled(ctx->flags, P)) return UPIPE_OK;
  if (!ctx->transport->peer_capable()) {
    ctx->last_error = "UPIPE_FLAG_DIRECT needs a ctx with peer memory (upipe_ipc_create + upipe_ipc_connect)";
    return UPIPE_ERR_STATE;
  }
  if (P.C > kMaxSeg) {
    ctx->last_error = "UPIPE_FLAG_DIRECT: Ulysses degree > 8 (one box) is not supported";
    return UPIPE_ERR_UNSUPPORTED;
  }
  return UPIPE_OK;
}

// Block `me` of every group peer's copy of the receive buffer `local_recv` (same offset in each rank's
// symmetric region): segment p of a producer's output goes to peer first + p. rows = rows per block.
bool peer_blocks(Transport& T, int first, int C, int me, const char* local_recv, size_t block_bytes, int64_t rows,
                 SegPtrs& out) {
  out = SegPtrs{};
  out.n = C;
  out.rows = rows;
  for (int p = 0; p < C; ++p) {
    char* b = static_cast<char*>(T.peer_ptr(first + p, local_recv));
    if (!b) return false;
    out.p[p] = b + (size_t)me * block_bytes;
  }
  return true;
}

}  // namespace

// ============================================================================ forward
upipe_status_t layer_fwd(upipe_ctx_s* ctx, const Plan& P, bf16p x, bf16p wq, bf16p wk, bf16p wv, bf16p wo,
                         const upipe_qk_norm_t* qkn, upipe_bf16* y, upipe_bf16* o_saved, float* lse_saved, char* ws,
                         cudaStream_t st) {
  const bool ov = overlap_enabled(ctx->flags, P);
  const bool dir = direct_enabled(ctx->flags, P);        // N2: producers write the peers' receive buffers
  if (upipe_status_t s = check_direct(ctx, P)) return s;
  if (ov || P.ring > 1) {                               // the ring hybrid overlaps its transfers on the comm stream
    if (upipe_status_t s = ensure_pipe(ctx)) return s;
  }
  Runner R{ctx};
  Transport& T = *ctx->transport;
  const FwdWs W = fwd_workspace(P, ov, dir);
  RopeRef rope_seq;                        // projections: rows are this rank's tokens rank*S_l + t
  if (upipe_status_t s = ensure_rope(ctx, P, rope_seq)) return s;
  // Qwen3 q/k norm (DESIGN A29): the projections send the pre-norm heads; each head owner normalises (and
  // rotates: RoPE follows the norm) its received rows in place before the attention
  const bool qknorm = P.sh.qk_norm_eps > 0.f;
  RopeRef rope_head = rope_seq;            // head layout: rows are the ring block's tokens (ring_i S ..)
  rope_head.pos0 = (int64_t)(ctx->rank / P.C) * P.S;
  if (qknorm) rope_seq = RopeRef{};
  rope_seq.pos0 = (int64_t)ctx->rank * P.S_l;
  // Ulysses group of the ring hybrid (DESIGN A27): ranks [first, first + C); plain UPipe: first = 0, C = cp_size
  const int C = P.C, me = ctx->rank % P.C, d = P.d;
  const int ring_i = ctx->rank / P.C, first = ring_i * P.C;
  auto a2a = [&](const char* what, const void* snd, void* rcv, size_t bytes, cudaStream_t q) {
    R.comm(q, what, [&](std::string& m) { return T.alltoall_group(snd, rcv, bytes, first, C, q, m); });
  };
  const int64_t qseg = (int64_t)P.qpd * d, kseg = (int64_t)P.kv_res * d;
  const int64_t HqD = (int64_t)P.Hq * d, kvrows = (int64_t)P.Hkv * d;
  const size_t qbytes = (size_t)P.S_l * qseg * 2, kbytes = (size_t)P.S_l * kseg * 2;
  const int64_t qstep = (int64_t)P.q_dev_stride() * d;
  auto kvb = [&](int s) { return ov ? P.kv_group(s) & 1 : 0; };
  // N2: the projection epilogues store block p of their output into block `me` of peer p's receive buffer
  auto direct_to = [&](GemmProblem g, const char* recv, size_t block_bytes, char* e) -> GemmProblem {
    if (!peer_blocks(T, first, C, me, recv, block_bytes, P.S_l, g.c.seg))
      snprintf(e, 512, "receive buffer outside the symmetric region");
    g.c.out_bf16 = nullptr;
    g.c.r_nstride = 0;
    return g;
  };

  // F1: Q_s (and K_s, V_s at a super-stage start) -> send buffer set b (N2: the peers' receive set b)
  auto proj = [&](int s, int b, cudaStream_t q) {
    const int64_t q0 = P.q0(s, 0), kv0 = P.kv0(s, 0);
    R.run(UPIPE_TRACE_GEMM, q, "proj Q", [&](char* e) {
      GemmProblem g = proj_to_send(P, x, wq, HqD, q0 * d, qstep, qseg, ws + W.qsend[b], rope_seq);
      if (dir) g = direct_to(g, ws + W.qrecv[b], qbytes, e);
      return e[0] ? cudaErrorInvalidValue : gemm_run(g, q, e, 512);
    });
    if (P.kv_sent(s)) {                    // K | V in one N-concatenated GEMM (X read once for both)
      const int kb = kvb(s);
      R.run(UPIPE_TRACE_GEMM, q, "proj K|V", [&](char* e) {
        GemmProblem g[2] = {proj_to_send(P, x, wk, kvrows, kv0 * d, kseg, kseg, ws + W.ksend, rope_seq),
                            proj_to_send(P, x, wv, kvrows, kv0 * d, kseg, kseg, ws + W.vsend)};
        if (dir) {
          g[0] = direct_to(g[0], ws + W.krecv[kb], kbytes, e);
          g[1] = direct_to(g[1], ws + W.vrecv[kb], kbytes, e);
        }
        return e[0] ? cudaErrorInvalidValue : gemm_run_group(g, 2, GemmGroup::kNConcat, q, e, 512);
      });
    }
  };
  // N2 handshake around a collective whose producers push into the peers: every group peer's receive
  // buffers are free (ready flags), ... the producers run ..., every peer's pushes have landed here
  auto push_begin = [&](const char* what, cudaStream_t q) {
    uint32_t e = 0;
    R.comm(q, what, [&](std::string& m) { return T.push_begin(first, C, q, &e, m); });
    return e;
  };
  auto push_end = [&](uint32_t e, const char* what, cudaStream_t q) {
    R.comm(q, what, [&](std::string& m) { return T.push_end(e, first, C, q, m); });
  };
  const upipe_probe_t& pr = ctx->probe;   // test-only layout probe (stage -1: off)
  auto probe_in = [&](int s, int b, cudaStream_t q) {
    if (pr.stage != s) return;
    R.run(UPIPE_TRACE_AUX, q, "probe recv", [&](char*) {
      cudaError_t e = probe_copy(pr.q_recv, ws + W.qrecv[b], (size_t)P.S * qseg * 2, q);
      if (e == cudaSuccess && P.kv_sent(s)) e = probe_copy(pr.k_recv, ws + W.krecv[kvb(s)], (size_t)P.S * kseg * 2, q);
      if (e == cudaSuccess && P.kv_sent(s)) e = probe_copy(pr.v_recv, ws + W.vrecv[kvb(s)], (size_t)P.S * kseg * 2, q);
      return e;
    });
  };
  // F2: inp_all_to_all, Q first, then K and V
  auto inp = [&](int s, int b, cudaStream_t q) {
    a2a("a2a Q", ws + W.qsend[b], ws + W.qrecv[b], qbytes, q);
    if (P.kv_sent(s)) {
      const int kb = kvb(s);
      a2a("a2a K", ws + W.ksend, ws + W.krecv[kb], kbytes, q);
      a2a("a2a V", ws + W.vsend, ws + W.vrecv[kb], kbytes, q);
    }
    probe_in(s, b, q);
  };
  // F3: attention over the full sequence for this device's qpd heads
  auto attn = [&](int s, int b, cudaStream_t q) {
    if (pr.stage == s && pr.o_head) {      // test probe: the injected head-layout O replaces the attention
      if (dir) {
        ctx->last_error = "layout probe O injection is not available with UPIPE_FLAG_DIRECT";
        R.status = UPIPE_ERR_INVALID_ARG;
        return;
      }
      R.run(UPIPE_TRACE_AUX, q, "probe inject O", [&](char*) {
        if (C == 1)
          return cudaMemcpy2DAsync(o_saved + (int64_t)P.q0(s, me) * d, HqD * 2, pr.o_head, qseg * 2, qseg * 2, P.S,
                                   cudaMemcpyDeviceToDevice, q);
        return probe_copy(ws + W.osend[b], pr.o_head, (size_t)P.S * qseg * 2, q);
      });
      return;
    }
    if (qknorm) {
      R.run(UPIPE_TRACE_AUX, q, "q norm", [&](char*) {
        return qk_prep_run(ws + W.qrecv[b], ws + W.qrecv[b], P.S, P.qpd, d, qseg, qkn->q_norm_w, P.sh.qk_norm_eps,
                           rope_head, q);
      });
      if (P.kv_sent(s))                    // once per super-stage: the K heads stay resident for sigma stages
        R.run(UPIPE_TRACE_AUX, q, "k norm", [&](char*) {
          return qk_prep_run(ws + W.krecv[kvb(s)], ws + W.krecv[kvb(s)], P.S, P.kv_res, d, kseg, qkn->k_norm_w,
                             P.sh.qk_norm_eps, rope_head, q);
        });
    }
    AttnFwdProblem a{};
    a.q = ws + W.qrecv[b];
    a.k = ws + W.krecv[kvb(s)];
    a.v = ws + W.vrecv[kvb(s)];
    if (C == 1) {
      a.o = o_saved + (int64_t)P.q0(s, me) * d;  // no out all-to-all: straight into the pre-allocated output
      a.ldo = HqD;
    } else if (dir) {                      // N2: rows of rank p's tokens -> block `me` of p's O receive buffer
      a.o = nullptr;
      a.ldo = qseg;
      if (!peer_blocks(T, first, C, me, ws + W.orecv[b], qbytes, P.S_l, a.o_seg)) {
        ctx->last_error = "attn fwd: O receive buffer outside the symmetric region";
        R.status = UPIPE_ERR_STATE;
        return;
      }
    } else {
      a.o = ws + W.osend[b];
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
    if (P.ring == 1) {
      R.run(UPIPE_TRACE_ATTN_FWD, q, "attn fwd", [&](char* e) { return attn_fwd_run(a, q, e, 512); });
      return;
    }
    // Ring hybrid (DESIGN A27): this rank's heads over ring block ring_i. Step t visits K/V
    // block j = ring_i - t (mod r), passed around the ring of the r ranks with the same Ulysses index;
    // each visible block's partial (fp32 O, lse) is merged by its LSE. Own block first (causal).
    void* const o_dst = a.o;
    const int64_t ld_dst = a.ldo;
    const SegPtrs o_seg_dst = a.o_seg;                  // N2: the merged O goes to the owners (below)
    a.o_seg = SegPtrs{};                                // the ring's attention writes fp32 partials
    float* const lse_acc = a.lse;
    a.o32 = (float*)(ws + W.oacc);
    a.ldo32 = qseg;
    const int r = P.ring;
    const int nxt = ((ring_i + 1) % r) * C + me, prv = ((ring_i + r - 1) % r) * C + me;
    const size_t kvbytes = (size_t)P.S * kseg * 2;
    // The ring transfers run on the ctx's comm stream, one step ahead of the attention on q: step t+1's
    // K/V block travels while step t's block is attended (double-buffered ring buffers; the comm stream
    // waits until the attention of step t-1 has read the buffer it receives into). Every collective of
    // the ring is issued on the comm stream, in the same order on every rank.
    cudaStream_t cs = ctx->pipe.comm;
    cudaEvent_t* rev = ctx->pipe.ev + 13;               // [0] own block ready, [1..2] received, [3..4] read
    auto ring_step = [&](int t, const void* ks, const void* vs) {   // receive block of step t into set t & 1
      char* kn = ws + W.kring[t & 1];
      char* vn = ws + W.vring[t & 1];
      if (t >= 3) cudaStreamWaitEvent(cs, rev[3 + (t & 1)], 0);   // attention of step t-2 read this set
      R.comm(cs, "ring K", [&](std::string& m) { return T.sendrecv(ks, nxt, kn, prv, kvbytes, cs, m); });
      R.comm(cs, "ring V", [&](std::string& m) { return T.sendrecv(vs, nxt, vn, prv, kvbytes, cs, m); });
      cudaEventRecord(rev[1 + (t & 1)], cs);
    };
    if (r > 1) {                                        // the first hop overlaps the own-block attention
      cudaEventRecord(rev[0], q);                       // own K/V block (and the stage's a2a) complete
      cudaStreamWaitEvent(cs, rev[0], 0);
      ring_step(1, a.k, a.v);                           // K/V are read-only for the attention below
    }
    R.run(UPIPE_TRACE_ATTN_FWD, q, "attn fwd (ring own block)", [&](char* e) { return attn_fwd_run(a, q, e, 512); });
    for (int t = 1; t < r && R.status == UPIPE_OK; ++t) {
      char* kn = ws + W.kring[t & 1];
      char* vn = ws + W.vring[t & 1];
      if (t + 1 < r) ring_step(t + 1, kn, vn);          // forward block t while it is attended (read-only)
      cudaStreamWaitEvent(q, rev[1 + (t & 1)], 0);
      const int j = (ring_i + r - t) % r;
      if (!(P.sh.causal && j > ring_i)) {                // else the whole block lies after every local query
        AttnFwdProblem b2 = a;
        b2.k = kn;
        b2.v = vn;
        b2.causal = 0;                                    // j < i: every key precedes every local query
        b2.o32 = (float*)(ws + W.opart);
        b2.lse = (float*)(ws + W.lsepart);
        R.run(UPIPE_TRACE_ATTN_FWD, q, "attn fwd (ring block)", [&](char* e) { return attn_fwd_run(b2, q, e, 512); });
        R.run(UPIPE_TRACE_AUX, q, "merge partials", [&](char*) {
          return merge_partials_run((float*)(ws + W.oacc), (const float*)(ws + W.opart), qseg, lse_acc,
                                    (const float*)(ws + W.lsepart), P.S, P.S, P.qpd, d, q);
        });
      }
      cudaEventRecord(rev[3 + (t & 1)], q);             // step t's buffers read
    }
    if (r > 1) {                                        // the comm stream's work is done before the next stage
      cudaEventRecord(rev[0], cs);
      cudaStreamWaitEvent(q, rev[0], 0);
    }
    R.run(UPIPE_TRACE_AUX, q, "O fp32 -> bf16", [&](char*) {
      if (o_seg_dst.n)
        return cvt_f32_bf16_seg_run((const float*)(ws + W.oacc), qseg, o_seg_dst, ld_dst, P.S, qseg, 1.0f, q,
                                    RopeRef{});
      return cvt_f32_bf16_run((const float*)(ws + W.oacc), qseg, o_dst, ld_dst, P.S, qseg, 1.0f, q);
    });
  };
  // F4: out_all_to_all
  auto outa = [&](int s, int b, cudaStream_t q) {
    (void)s;
    a2a("a2a O", ws + W.osend[b], ws + W.orecv[b], qbytes, q);
  };
  // F5: fill o_saved from the stage's out all-to-all (C == 1: attention wrote it directly)
  auto post = [&](int s, int b, cudaStream_t q) {
    const int64_t q0 = P.q0(s, 0);
    if (C > 1)
      R.run(UPIPE_TRACE_AUX, q, "unpack O", [&](char*) {
        return unpack_cols_run(ws + W.orecv[b], P.S_l, C, (int)qseg, o_saved, HqD, q0 * d, qstep, q);
      });
  };
  // F6/F7: y = O Wo^T once every head's O is in the pre-allocated output: one GEMM
  // with K = Hq*d and a bf16 epilogue, no fp32 accumulator across stages (DESIGN A24)
  auto out_proj = [&](cudaStream_t q) {
    GemmProblem g;
    g.M = P.S_l;
    g.N = P.D;
    g.K = HqD;
    g.a = OperandMap{o_saved, HqD, P.S_l, HqD, false};
    g.b = OperandMap{wo, HqD, P.D, HqD, false};
    g.c.out_bf16 = y;
    g.c.ld_bf16 = P.D;
    g.c.epi = Epi::kStoreBF16;
    R.run(UPIPE_TRACE_GEMM, q, "out proj", [&](char* e) { return gemm_run(g, q, e, 512); });
  };

  const int nu = P.nstages;
  if (dir) {
    // N2: one stream, one buffer set; each all-to-all happens inside its producer (projection / attention
    // epilogues writing peer memory), bracketed by the ready/done flag handshake
    for (int s = 0; s < nu && R.status == UPIPE_OK; ++s) {
      const uint32_t e_in = push_begin("direct QKV begin", st);
      proj(s, 0, st);
      push_end(e_in, "direct QKV end", st);
      probe_in(s, 0, st);
      const uint32_t e_o = push_begin("direct O begin", st);
      attn(s, 0, st);
      push_end(e_o, "direct O end", st);
      post(s, 0, st);
    }
    out_proj(st);
    return R.status;
  }
  if (!ov) {
    for (int s = 0; s < nu && R.status == UPIPE_OK; ++s) {
      proj(s, 0, st);
      if (C > 1) inp(s, 0, st);
      else probe_in(s, 0, st);
      attn(s, 0, st);
      if (C > 1) outa(s, 0, st);
      post(s, 0, st);
    }
    out_proj(st);
    return R.status;
  }
  // ---- overlapped schedule
  cudaStream_t cs = ctx->pipe.comm;
  cudaEvent_t* ev = ctx->pipe.ev;
  cudaEvent_t e_begin = ev[0], *e_proj = ev + 1, *e_in = ev + 3, *e_attn = ev + 5, *e_out = ev + 7, *e_post = ev + 9;
  cudaEventRecord(e_begin, st);
  cudaStreamWaitEvent(cs, e_begin, 0);
  proj(0, 0, st);
  cudaEventRecord(e_proj[0], st);
  cudaStreamWaitEvent(cs, e_proj[0], 0);
  inp(0, 0, cs);
  cudaEventRecord(e_in[0], cs);
  for (int s = 0; s < nu && R.status == UPIPE_OK; ++s) {
    const int b = s & 1;
    if (s + 1 < nu) {
      const int b1 = (s + 1) & 1;
      if (s >= 1) cudaStreamWaitEvent(st, e_in[b1], 0);          // a2a(s-1) has read send set b1
      if (P.kv_sent(s + 1)) cudaStreamWaitEvent(st, e_in[b], 0);  // a2a(s) has read the single K/V send buffers
      proj(s + 1, b1, st);
      cudaEventRecord(e_proj[b1], st);
      cudaStreamWaitEvent(cs, e_proj[b1], 0);
      if (s >= 1) cudaStreamWaitEvent(cs, e_attn[b1], 0);         // attention(s-1) has read receive set b1
      inp(s + 1, b1, cs);
      cudaEventRecord(e_in[b1], cs);
    }
    cudaStreamWaitEvent(st, e_in[b], 0);
    attn(s, b, st);
    cudaEventRecord(e_attn[b], st);
    cudaStreamWaitEvent(cs, e_attn[b], 0);
    if (s >= 2) cudaStreamWaitEvent(cs, e_post[b], 0);            // post(s-2) has read O receive set b
    outa(s, b, cs);
    cudaEventRecord(e_out[b], cs);
    if (s >= 1) {
      cudaStreamWaitEvent(st, e_out[(s - 1) & 1], 0);
      post(s - 1, (s - 1) & 1, st);
      cudaEventRecord(e_post[(s - 1) & 1], st);
    }
  }
  cudaStreamWaitEvent(st, e_out[(nu - 1) & 1], 0);
  post(nu - 1, (nu - 1) & 1, st);
  out_proj(st);
  return R.status;
}

// ============================================================================ backward
upipe_status_t layer_bwd(upipe_ctx_s* ctx, const Plan& P, bf16p x, bf16p wq, bf16p wk, bf16p wv, bf16p wo,
                         const upipe_qk_norm_t* qkn, bf16p dy, bf16p o_saved, const float* lse_saved, upipe_bf16* dx,
                         float* dwq, float* dwk, float* dwv, float* dwo, int reduce_dw, char* ws, cudaStream_t st) {
  const bool ov = overlap_enabled(ctx->flags, P);
  const bool dir = direct_enabled(ctx->flags, P);        // N2: producers write the peers' receive buffers
  if (upipe_status_t s = check_direct(ctx, P)) return s;
  if (ov || P.ring > 1) {                               // the ring hybrid overlaps its transfers on the comm stream
    if (upipe_status_t s = ensure_pipe(ctx)) return s;
  }
  Runner R{ctx};
  Transport& T = *ctx->transport;
  const BwdWs W = bwd_workspace(P, ov, dir);
  const int C = P.C, me = ctx->rank % P.C, d = P.d;
  const int ring_i = ctx->rank / P.C, first = ring_i * P.C;   // Ulysses group (DESIGN A27)
  RopeRef rope_seq, rope_head;             // seq layout (projections) / head layout (rows = the group's tokens)
  if (upipe_status_t s = ensure_rope(ctx, P, rope_seq)) return s;
  rope_head = rope_seq;
  rope_head.pos0 = (int64_t)ring_i * P.S;
  const bool qknorm = P.sh.qk_norm_eps > 0.f;   // DESIGN A29: projections send pre-norm heads (no RoPE there)
  if (qknorm) rope_seq = RopeRef{};
  rope_seq.pos0 = (int64_t)ctx->rank * P.S_l;
  auto a2a = [&](const char* what, const void* snd, void* rcv, size_t bytes, cudaStream_t q) {
    R.comm(q, what, [&](std::string& m) { return T.alltoall_group(snd, rcv, bytes, first, C, q, m); });
  };
  const int64_t qseg = (int64_t)P.qpd * d, kseg = (int64_t)P.kv_res * d;
  const int64_t HqD = (int64_t)P.Hq * d, HkvD = (int64_t)P.Hkv * d;
  const size_t qbytes = (size_t)P.S_l * qseg * 2, kbytes = (size_t)P.S_l * kseg * 2;
  const size_t dbytes = (size_t)P.S_l * P.qpd * 4;
  const int64_t qstep = (int64_t)P.q_dev_stride() * d;
  auto kvb = [&](int s) { return ov ? P.kv_group(s) & 1 : 0; };
  auto direct_to = [&](GemmProblem g, const char* recv, size_t block_bytes, char* e) -> GemmProblem {
    if (!peer_blocks(T, first, C, me, recv, block_bytes, P.S_l, g.c.seg))
      snprintf(e, 512, "receive buffer outside the symmetric region");
    g.c.out_bf16 = nullptr;
    g.c.r_nstride = 0;
    return g;
  };
  auto push_begin = [&](const char* what, cudaStream_t q) {
    uint32_t e = 0;
    R.comm(q, what, [&](std::string& m) { return T.push_begin(first, C, q, &e, m); });
    return e;
  };
  auto push_end = [&](uint32_t e, const char* what, cudaStream_t q) {
    R.comm(q, what, [&](std::string& m) { return T.push_end(e, first, C, q, m); });
  };

  if (qknorm)                                           // d(gamma_q), d(gamma_k) accumulate over the stages
    R.run(UPIPE_TRACE_AUX, st, "memset d(gamma)", [&](char*) {
      return cudaMemsetAsync(ws + W.dgam, 0, (size_t)2 * d * 4, st);
    });
  // UPIPE_FLAG_DETERMINISTIC: no split-K either (its partial products are added in arrival order)
  const bool det_order = (ctx->flags & UPIPE_FLAG_DETERMINISTIC) != 0;
  // The weight gradients are zeroed first so their long-K GEMMs (K = S_l, only M x N = 1536 x 4096 output tiles)
  // may split K across all SMs and add their partials (gemm.cu split-K); every dW row is written by one GEMM.
  R.run(UPIPE_TRACE_AUX, st, "zero dW", [&](char*) {
    cudaError_t e = cudaMemsetAsync(dwq, 0, (size_t)HqD * P.D * 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(dwk, 0, (size_t)HkvD * P.D * 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(dwv, 0, (size_t)HkvD * P.D * 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(dwo, 0, (size_t)HqD * P.D * 4, st);
    return e;
  });
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
    g.c.zeroed = !det_order;
    R.run(UPIPE_TRACE_GEMM, st, "dWo", [&](char* e) { return gemm_run(g, st, e, 512); });
  }
  const int n_dx_terms = P.nstages;   // one K-concatenated dX GEMM per stage
  int dx_term = 0;
  auto dx_epi = [&](GemmProblem& g) {
    g.c.out_f32 = ws + W.dxacc;
    g.c.ld_f32 = P.D;
    g.c.out_bf16 = dx;
    g.c.ld_bf16 = P.D;
    if (n_dx_terms == 1) g.c.epi = Epi::kStoreBF16;
    else g.c.epi = dx_term == 0 ? Epi::kStoreF32 : (dx_term == n_dx_terms - 1 ? Epi::kAccF32ToBF16 : Epi::kAccF32);
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
    g.c.zeroed = !det_order;                     // zeroed at the start of the backward: split-K allowed
    return g;
  };

  // B1 + B2: recompute the stage's projections, dO_s = dY Wo[:, cols(s)], delta = rowsum(dO*O) (A13)
  auto pre = [&](int s, int b, cudaStream_t q) {
    const int64_t q0 = P.q0(s, 0), kv0 = P.kv0(s, 0);
    R.run(UPIPE_TRACE_GEMM, q, "proj Q", [&](char* e) {
      GemmProblem g = proj_to_send(P, x, wq, HqD, q0 * d, qstep, qseg, ws + W.qsend[b], rope_seq);
      if (dir) g = direct_to(g, ws + W.qrecv[b], qbytes, e);
      return e[0] ? cudaErrorInvalidValue : gemm_run(g, q, e, 512);
    });
    if (P.kv_sent(s)) {                    // K | V in one N-concatenated GEMM (X read once for both)
      const int kb = kvb(s);
      R.run(UPIPE_TRACE_GEMM, q, "proj K|V", [&](char* e) {
        GemmProblem g[2] = {proj_to_send(P, x, wk, HkvD, kv0 * d, kseg, kseg, ws + W.ksend, rope_seq),
                            proj_to_send(P, x, wv, HkvD, kv0 * d, kseg, kseg, ws + W.vsend)};
        if (dir) {
          g[0] = direct_to(g[0], ws + W.krecv[kb], kbytes, e);
          g[1] = direct_to(g[1], ws + W.vrecv[kb], kbytes, e);
        }
        return e[0] ? cudaErrorInvalidValue : gemm_run_group(g, 2, GemmGroup::kNConcat, q, e, 512);
      });
    }
    GemmProblem g;
    g.M = P.S_l;
    g.N = (int64_t)C * qseg;
    g.K = P.D;
    g.a = OperandMap{dy, P.D, P.S_l, P.D, false};
    g.b = OperandMap{wo, HqD, P.D, HqD, true};
    g.b.o_base = q0 * d;
    g.b.o_len = qseg;
    g.b.o_istride = qstep;
    g.c.out_bf16 = ws + W.dosend[b];
    g.c.ld_bf16 = qseg;
    g.c.n_len = qseg;
    g.c.r_nstride = P.S_l;
    g.c.epi = Epi::kStoreBF16;
    static const bool fuse_env = [] {                // UPIPE_FUSED_ROWDOT=0: separate row-dot kernel (A/B)
      const char* e = getenv("UPIPE_FUSED_ROWDOT");
      return !(e && e[0] == '0');
    }();
    if (!dir && !fuse_env) {
      g.c.out_bf16 = ws + W.dosend[b];
      R.run(UPIPE_TRACE_GEMM, q, "dO", [&](char* e) { return gemm_run(g, q, e, 512); });
      for (int p = 0; p < C; ++p)
        R.run(UPIPE_TRACE_AUX, q, "rowdot", [&](char*) {
          return rowdot_run((const upipe_bf16*)(ws + W.dosend[b]) + (int64_t)p * P.S_l * qseg, qseg,
                            o_saved + (int64_t)P.q0(s, p) * d, HqD, (float*)(ws + W.dsend[b]) + (int64_t)p * P.S_l * P.qpd,
                            P.qpd, P.S_l, P.qpd, d, q);
        });
      return;
    }
    // delta = rowsum(dO * O) fused into the epilogue (A13): dO column (p, nin) <-> o_saved column
    // q0(s, p) d + nin = q0 d + p qstep + nin; delta of (token t, head j) -> block p of the delta send
    // buffer [C][S_l][qpd] (N2: block `me` of peer p's delta receive buffer)
    g.c.dot.o = o_saved;
    g.c.dot.ld_o = HqD;
    g.c.dot.col0 = q0 * d;
    g.c.dot.col_stride = qstep;
    g.c.dot.ld_dst = P.qpd;
    g.c.dot.d = d;
    R.run(UPIPE_TRACE_GEMM, q, "dO + delta", [&](char* e) {
      if (dir) {
        g = direct_to(g, ws + W.dorecv[b], qbytes, e);
        SegPtrs ds;
        if (!e[0] && !peer_blocks(T, first, C, me, ws + W.drecv[b], dbytes, P.S_l, ds))
          snprintf(e, 512, "delta receive buffer outside the symmetric region");
        for (int p = 0; p < C; ++p) g.c.dot.dst[p] = static_cast<float*>(ds.p[p]);
        g.c.dot.dst_stride = 0;
      } else {
        g.c.dot.dst[0] = (float*)(ws + W.dsend[b]);
        g.c.dot.dst_stride = (int64_t)P.S_l * P.qpd;
      }
      return e[0] ? cudaErrorInvalidValue : gemm_run(g, q, e, 512);
    });
  };
  const upipe_probe_t& pr = ctx->probe;   // test-only layout probe (stage -1: off)
  auto probe_in = [&](int s, int b, cudaStream_t q) {
    if (pr.stage != s) return;
    R.run(UPIPE_TRACE_AUX, q, "probe recv", [&](char*) {
      cudaError_t e = probe_copy(pr.q_recv, ws + W.qrecv[b], (size_t)P.S * qseg * 2, q);
      if (e == cudaSuccess && P.kv_sent(s)) e = probe_copy(pr.k_recv, ws + W.krecv[kvb(s)], (size_t)P.S * kseg * 2, q);
      if (e == cudaSuccess && P.kv_sent(s)) e = probe_copy(pr.v_recv, ws + W.vrecv[kvb(s)], (size_t)P.S * kseg * 2, q);
      if (e == cudaSuccess) e = probe_copy(pr.do_recv, ws + W.dorecv[b], (size_t)P.S * qseg * 2, q);
      if (e == cudaSuccess) e = probe_copy(pr.delta_recv, ws + W.drecv[b], (size_t)P.S * P.qpd * 4, q);
      return e;
    });
  };
  auto probe_out = [&](int s, int b, cudaStream_t q) {
    if (pr.stage != s) return;
    R.run(UPIPE_TRACE_AUX, q, "probe send back", [&](char*) {
      cudaError_t e = probe_copy(pr.dq_recv, ws + W.dqrecv[b], (size_t)P.S * qseg * 2, q);
      if (e == cudaSuccess && P.kv_last(s)) e = probe_copy(pr.dk_recv, ws + W.dkrecv, (size_t)P.S * kseg * 2, q);
      if (e == cudaSuccess && P.kv_last(s)) e = probe_copy(pr.dv_recv, ws + W.dvrecv, (size_t)P.S * kseg * 2, q);
      return e;
    });
  };
  // B1/B3: Q (+K, V) and dO + delta seq -> head ("during out_all_to_all", Table 4)
  auto inp = [&](int s, int b, cudaStream_t q) {
    a2a("a2a Q", ws + W.qsend[b], ws + W.qrecv[b], qbytes, q);
    if (P.kv_sent(s)) {
      const int kb = kvb(s);
      a2a("a2a K", ws + W.ksend, ws + W.krecv[kb], kbytes, q);
      a2a("a2a V", ws + W.vsend, ws + W.vrecv[kb], kbytes, q);
    }
    a2a("a2a dO", ws + W.dosend[b], ws + W.dorecv[b], qbytes, q);
    a2a("a2a delta", ws + W.dsend[b], ws + W.drecv[b], dbytes, q);
    probe_in(s, b, q);
  };
  // B4: attention backward (dK/dV accumulate over the sigma stages sharing the resident K/V), dQ -> bf16
  auto attn = [&](int s, int b, cudaStream_t q) {
    if (pr.stage == s && pr.dq_head) {     // test probe: injected head-layout dQ (dK, dV) replace the kernel's
      if (dir) {
        ctx->last_error = "layout probe dQ injection is not available with UPIPE_FLAG_DIRECT";
        R.status = UPIPE_ERR_INVALID_ARG;
        return;
      }
      R.run(UPIPE_TRACE_AUX, q, "probe inject dQ", [&](char*) {
        cudaError_t e = probe_copy(ws + W.dqsend[b], pr.dq_head, (size_t)P.S * qseg * 2, q);
        if (e == cudaSuccess && P.kv_last(s)) e = probe_copy(ws + W.dksend, pr.dk_head, (size_t)P.S * kseg * 2, q);
        if (e == cudaSuccess && P.kv_last(s)) e = probe_copy(ws + W.dvsend, pr.dv_head, (size_t)P.S * kseg * 2, q);
        return e;
      });
      return;
    }
    R.run(UPIPE_TRACE_AUX, q, "memset dQ", [&](char*) {
      return cudaMemsetAsync(ws + W.dqacc[b], 0, (size_t)((P.S + 3) & ~int64_t(3)) * qseg * 4, q);
    });
    const int r = P.kv_pos(s);
    const bool last = P.kv_last(s);
    if (qknorm) {                                     // normalised (+ RoPE) copies; the receive buffers keep the
      R.run(UPIPE_TRACE_AUX, q, "q norm", [&](char*) {   // pre-norm heads for the chain rule below
        return qk_prep_run(ws + W.qrecv[b], ws + W.qn[b], P.S, P.qpd, d, qseg, qkn->q_norm_w, P.sh.qk_norm_eps,
                           rope_head, q);
      });
      if (P.kv_sent(s))
        R.run(UPIPE_TRACE_AUX, q, "k norm", [&](char*) {
          return qk_prep_run(ws + W.krecv[kvb(s)], ws + W.kn[kvb(s)], P.S, P.kv_res, d, kseg, qkn->k_norm_w,
                             P.sh.qk_norm_eps, rope_head, q);
        });
    }
    AttnBwdProblem bp{};
    bp.q = qknorm ? ws + W.qn[b] : ws + W.qrecv[b];
    bp.k = qknorm ? ws + W.kn[kvb(s)] : ws + W.krecv[kvb(s)];
    bp.v = ws + W.vrecv[kvb(s)];
    bp.dout = ws + W.dorecv[b];
    bp.lse = lse_saved + (int64_t)s * P.qpd * P.S;
    bp.delta = (const float*)(ws + W.drecv[b]);
    bp.dq_acc = (float*)(ws + W.dqacc[b]);
    bp.dk_acc = P.sigma > 1 && !P.naive ? (float*)(ws + W.dkacc) : nullptr;
    bp.dv_acc = P.sigma > 1 && !P.naive ? (float*)(ws + W.dvacc) : nullptr;
    bp.dk_bf16 = last ? ws + W.dksend : nullptr;
    bp.dv_bf16 = last ? ws + W.dvsend : nullptr;
    SegPtrs dq_seg, dk_seg;                           // N2: dQ / dK / dV rows of rank p's tokens -> peer p
    if (dir) {
      bool ok = peer_blocks(T, first, C, me, ws + W.dqrecv[b], qbytes, P.S_l, dq_seg);
      if (last) {
        ok = ok && peer_blocks(T, first, C, me, ws + W.dkrecv, kbytes, P.S_l, dk_seg) &&
             peer_blocks(T, first, C, me, ws + W.dvrecv, kbytes, P.S_l, bp.dv_seg);
        bp.dk_seg = dk_seg;
        bp.dk_bf16 = bp.dv_bf16 = nullptr;
      }
      if (!ok) {
        ctx->last_error = "attn bwd: receive buffer outside the symmetric region";
        R.status = UPIPE_ERR_STATE;
        return;
      }
    }
    bp.S = P.S;
    bp.nq = P.qpd;
    bp.nkv = P.kv_res;
    bp.d = d;
    bp.causal = P.sh.causal;
    bp.ldq = qseg;
    bp.ldkv = kseg;
    bp.ldo_grad = qseg;
    bp.ld_lse = P.S;
    bp.ld_delta = P.qpd;
    bp.ld_kvb = kseg;
    bp.kv_accumulate = r > 0;
    bp.kv_write_acc = !last;
    bp.rope = rope_head;
    if (qknorm) {                                     // dK leaves in fp32 (pre-RoPE chain rule below)
      bp.dk_acc = (float*)(ws + W.dkacc);
      bp.kv_write_acc = 1;
      bp.dk_bf16 = nullptr;
      bp.dk_seg = SegPtrs{};
    }
    bp.dq_dim_major = attn_bwd_dq_dim_major(bp) ? 1 : 0;   // [qpd*d][S] accumulator (64-query kernel)
    bp.ld_dqt = (P.S + 3) & ~int64_t(3);                  // 16-byte TMA row stride
    // UPIPE_FLAG_DETERMINISTIC: dQ partials added in key-tile order; fresh semaphores per launch
    const bool det = (ctx->flags & UPIPE_FLAG_DETERMINISTIC) != 0;
    bp.dq_sem = det ? (int*)(ws + W.dqsem) : nullptr;
    auto bwd_launch = [&](const AttnBwdProblem& pb, const char* what) {
      if (det)
        R.run(UPIPE_TRACE_AUX, q, "memset dQ semaphores", [&](char*) {
          return cudaMemsetAsync(ws + W.dqsem, 0, (size_t)attn_bwd_sem_count(P.S, P.qpd) * 4, q);
        });
      R.run(UPIPE_TRACE_ATTN_BWD, q, what, [&](char* e) { return attn_bwd_run(pb, q, e, 512); });
    };
    if (P.ring == 1) {
      bwd_launch(bp, "attn bwd");
    } else {
      // Ring hybrid (DESIGN A27): the super-stage's fp32 dK/dV accumulators travel with their K/V block;
      // each rank adds the contributions of its queries (final lse and delta), dQ accumulates locally
      // (TMA reduce-add), and after the last hop every accumulator is back with its owner.
      const int rr = P.ring;
      const int nxt = ((ring_i + 1) % rr) * C + me, prv = ((ring_i + rr - 1) % rr) * C + me;
      const size_t kvbytes = (size_t)P.S * kseg * 2;
      bp.dk_acc = (float*)(ws + W.dkacc);
      bp.dv_acc = (float*)(ws + W.dvacc);
      bp.dk_bf16 = bp.dv_bf16 = nullptr;
      const SegPtrs dv_seg_dst = bp.dv_seg;             // N2: the home dK / dV go to the owners (below)
      bp.dk_seg = bp.dv_seg = SegPtrs{};                // the ring's kernels accumulate fp32 only
      bp.kv_write_acc = 1;
      // Overlapped ring (all ring collectives on the ctx's comm stream, same order on every rank): the
      // accumulators of step t travel right after this rank's attention of step t-1 (that dependency is
      // inherent), then step t+1's K/V block is forwarded while step t is attended.
      cudaStream_t cs = ctx->pipe.comm;
      cudaEvent_t* rev = ctx->pipe.ev + 13;             // [0] join, [1..2] step received, [3..4] step computed
      cudaEventRecord(rev[0], q);                       // the stage's K/V, dO, delta are in place
      cudaStreamWaitEvent(cs, rev[0], 0);
      R.comm(cs, "ring K", [&](std::string& m) { return T.sendrecv(bp.k, nxt, ws + W.kring[1], prv, kvbytes, cs, m); });
      R.comm(cs, "ring V", [&](std::string& m) { return T.sendrecv(bp.v, nxt, ws + W.vring[1], prv, kvbytes, cs, m); });
      bwd_launch(bp, "attn bwd (ring own block)");
      cudaEventRecord(rev[3], q);                       // step 0 computed (rev[3 + (t & 1)] for step t)
      for (int t = 1; t <= rr && R.status == UPIPE_OK; ++t) {
        const bool home = t == rr;                      // last hop: the accumulators return to their owner
        const float* dks = t == 1 ? (const float*)(ws + W.dkacc) : (const float*)(ws + W.dkring[(t - 1) & 1]);
        const float* dvs = t == 1 ? (const float*)(ws + W.dvacc) : (const float*)(ws + W.dvring[(t - 1) & 1]);
        float* dkn = home ? (float*)(ws + W.dkacc) : (float*)(ws + W.dkring[t & 1]);
        float* dvn = home ? (float*)(ws + W.dvacc) : (float*)(ws + W.dvring[t & 1]);
        cudaStreamWaitEvent(cs, rev[3 + ((t - 1) & 1)], 0);   // this rank's step t-1 contributions are in
        R.comm(cs, "ring dK", [&](std::string& m) { return T.sendrecv(dks, nxt, dkn, prv, kvbytes * 2, cs, m); });
        R.comm(cs, "ring dV", [&](std::string& m) { return T.sendrecv(dvs, nxt, dvn, prv, kvbytes * 2, cs, m); });
        cudaEventRecord(rev[1 + (t & 1)], cs);
        if (home) break;
        char* kn = ws + W.kring[t & 1];
        char* vn = ws + W.vring[t & 1];
        if (t + 1 < rr) {                               // forward block t while it is attended (read-only)
          R.comm(cs, "ring K", [&](std::string& m) {
            return T.sendrecv(kn, nxt, ws + W.kring[(t + 1) & 1], prv, kvbytes, cs, m);
          });
          R.comm(cs, "ring V", [&](std::string& m) {
            return T.sendrecv(vn, nxt, ws + W.vring[(t + 1) & 1], prv, kvbytes, cs, m);
          });
        }
        cudaStreamWaitEvent(q, rev[1 + (t & 1)], 0);
        const int j = (ring_i + rr - t) % rr;
        if (!(P.sh.causal && j > ring_i)) {
          AttnBwdProblem b2 = bp;
          b2.k = kn;
          b2.v = vn;
          b2.dk_acc = dkn;
          b2.dv_acc = dvn;
          b2.causal = 0;
          b2.kv_accumulate = 1;
          bwd_launch(b2, "attn bwd (ring block)");
        }
        cudaEventRecord(rev[3 + (t & 1)], q);
      }
      cudaStreamWaitEvent(q, rev[1 + (rr & 1)], 0);     // the home hop has landed
      if (last) {
        RopeRef rope_k = rope_head;                       // dK rows are the ring block's keys
        if (!qknorm)                                      // (q/k norm: the chain rule below converts dK)
          R.run(UPIPE_TRACE_AUX, q, "cvt dK", [&](char*) {
            if (dir)
              return cvt_f32_bf16_seg_run((const float*)(ws + W.dkacc), kseg, dk_seg, kseg, P.S, kseg, 1.0f, q, rope_k);
            return cvt_f32_bf16_run((const float*)(ws + W.dkacc), kseg, ws + W.dksend, kseg, P.S, kseg, 1.0f, q, rope_k);
          });
        R.run(UPIPE_TRACE_AUX, q, "cvt dV", [&](char*) {
          if (dir)
            return cvt_f32_bf16_seg_run((const float*)(ws + W.dvacc), kseg, dv_seg_dst, kseg, P.S, kseg, 1.0f, q,
                                        RopeRef{});
          return cvt_f32_bf16_run((const float*)(ws + W.dvacc), kseg, ws + W.dvsend, kseg, P.S, kseg, 1.0f, q);
        });
      }
    }
    if (qknorm) {
      // chain rule of the q/k norm fused into the gradients' fp32 -> bf16 conversion (A29): inverse RoPE, then
      // d(pre-norm) from the pre-norm heads still in the receive buffers; d(gamma) accumulates in the workspace
      R.run(UPIPE_TRACE_AUX, q, "dQ norm bwd", [&](char*) {
        return norm_bwd_run((const float*)(ws + W.dqacc[b]), bp.dq_dim_major ? bp.ld_dqt : qseg, bp.dq_dim_major != 0,
                            ws + W.qrecv[b], qseg, dir ? nullptr : ws + W.dqsend[b], qseg, dir ? &dq_seg : nullptr,
                            P.S, P.qpd, d, 1.0f, qkn->q_norm_w, P.sh.qk_norm_eps, rope_head, (float*)(ws + W.dgam), q,
                            det ? (float*)(ws + W.dgam) + 2 * d : nullptr);
      });
      if (last)
        R.run(UPIPE_TRACE_AUX, q, "dK norm bwd", [&](char*) {
          return norm_bwd_run((const float*)(ws + W.dkacc), kseg, false, ws + W.krecv[kvb(s)], kseg,
                              dir ? nullptr : ws + W.dksend, kseg, dir ? &dk_seg : nullptr, P.S, P.kv_res, d, 1.0f,
                              qkn->k_norm_w, P.sh.qk_norm_eps, rope_head, (float*)(ws + W.dgam) + d, q,
                              det ? (float*)(ws + W.dgam) + 2 * d : nullptr);
        });
      return;
    }
    R.run(UPIPE_TRACE_AUX, q, "cvt dQ", [&](char*) {
      if (bp.dq_dim_major)
        return cvt_dimmajor_f32_bf16_run((const float*)(ws + W.dqacc[b]), bp.ld_dqt, dir ? nullptr : ws + W.dqsend[b], qseg,
                                         P.S, qseg, 1.0f, q, rope_head, dir ? &dq_seg : nullptr);
      if (dir)
        return cvt_f32_bf16_seg_run((const float*)(ws + W.dqacc[b]), qseg, dq_seg, qseg, P.S, qseg, 1.0f, q, rope_head);
      return cvt_f32_bf16_run((const float*)(ws + W.dqacc[b]), qseg, ws + W.dqsend[b], qseg, P.S, qseg, 1.0f, q,
                              rope_head);
    });
  };
  // B5: dQ head -> seq ("during inp_all_to_all"); dK/dV when the super-stage's K/V retire
  auto outa = [&](int s, int b, cudaStream_t q) {
    a2a("a2a dQ", ws + W.dqsend[b], ws + W.dqrecv[b], qbytes, q);
    if (P.kv_last(s)) {
      a2a("a2a dK", ws + W.dksend, ws + W.dkrecv, kbytes, q);
      a2a("a2a dV", ws + W.dvsend, ws + W.dvrecv, kbytes, q);
    }
    probe_out(s, b, q);
  };
  // B6: dX and dW for the stage's heads (and the retired K/V heads). dX += dQ Wq + dK Wk + dV Wv is
  // one K-concatenated GEMM (one fp32 read-modify-write of the dX accumulator per stage) and
  // [dWq; dWk; dWv] = [dQ; dK; dV]^T X one M-concatenated GEMM (DESIGN A24).
  // Pre-allocated gradient buffer G [S_l][(Hq + 2 Hkv) d] bf16 (DESIGN A30; the backward analogue of the
  // pre-allocated output of P:329): each stage's received dQ (and the retired dK / dV) land in their head
  // columns, and dX = G [Wq; Wk; Wv] and [dWq; dWk; dWv] = G^T X run once after the stage loop -- one
  // long-K GEMM with a bf16 epilogue instead of a fp32 dX read-modify-write per stage. Not with the naive
  // ablation, whose stages send partial dK / dV, nor with one stage (Ulysses), whose dX GEMM stores bf16 directly.
  const bool gbuf = P.gbuf();
  const int64_t Gc = HqD + 2 * HkvD;
  auto post_g = [&](int s, int b, cudaStream_t q) {
    const int64_t q0 = P.q0(s, 0), kv0 = P.kv0(s, 0);
    upipe_bf16* G = reinterpret_cast<upipe_bf16*>(ws + W.gbuf);
    R.run(UPIPE_TRACE_AUX, q, "unpack dQ", [&](char*) {
      return unpack_cols_run(ws + W.dqrecv[b], P.S_l, C, (int)qseg, G, Gc, q0 * d, qstep, q);
    });
    if (P.kv_last(s)) {
      R.run(UPIPE_TRACE_AUX, q, "unpack dK", [&](char*) {
        return unpack_cols_run(ws + W.dkrecv, P.S_l, C, (int)kseg, G, Gc, HqD + kv0 * d, kseg, q);
      });
      R.run(UPIPE_TRACE_AUX, q, "unpack dV", [&](char*) {
        return unpack_cols_run(ws + W.dvrecv, P.S_l, C, (int)kseg, G, Gc, HqD + HkvD + kv0 * d, kseg, q);
      });
    }
  };
  auto final_g = [&](cudaStream_t q) {
    const upipe_bf16* G = reinterpret_cast<const upipe_bf16*>(ws + W.gbuf);
    const void* Ws[3] = {wq, wk, wv};
    float* dWs[3] = {dwq, dwk, dwv};
    const int64_t rows[3] = {HqD, HkvD, HkvD}, c0[3] = {0, HqD, HqD + HkvD};
    GemmProblem gx[3], gw[3];
    for (int i = 0; i < 3; ++i) {
      GemmProblem& x1 = gx[i];               // dX += G[:, c0 : c0 + rows] W_i   (B = W_i, N = D contiguous)
      x1.M = P.S_l;
      x1.N = P.D;
      x1.K = rows[i];
      x1.a = OperandMap{G, Gc, P.S_l, Gc, false};
      x1.a.k_base = c0[i];
      x1.b = OperandMap{Ws[i], P.D, rows[i], P.D, true};
      x1.c.out_bf16 = dx;
      x1.c.ld_bf16 = P.D;
      x1.c.epi = Epi::kStoreBF16;
      GemmProblem& w1 = gw[i];               // dW_i = G[:, c0 : c0 + rows]^T X   (A MN-major: rows along G)
      w1.M = rows[i];
      w1.N = P.D;
      w1.K = P.S_l;
      w1.a = OperandMap{G, Gc, P.S_l, Gc, true};
      w1.a.o_base = c0[i];
      w1.b = OperandMap{x, P.D, P.S_l, P.D, true};
      w1.c.out_f32 = dWs[i];
      w1.c.ld_f32 = P.D;
      w1.c.epi = Epi::kStoreF32;
      w1.c.zeroed = !det_order;              // split-K adds in arrival order: not in deterministic mode
    }
    R.run(UPIPE_TRACE_GEMM, q, "dX = G W", [&](char* e) { return gemm_run_group(gx, 3, GemmGroup::kKConcat, q, e, 512); });
    R.run(UPIPE_TRACE_GEMM, q, "dW = G^T X", [&](char* e) {
      return gemm_run_group(gw, 3, GemmGroup::kMConcat, q, e, 512);
    });
  };
  auto post = [&](int s, int b, cudaStream_t q) {
    if (gbuf) {
      post_g(s, b, q);
      return;
    }
    const int64_t q0 = P.q0(s, 0), kv0 = P.kv0(s, 0);
    GemmProblem gx[3], gw[3];
    int n = 1;
    gx[0] = dx_gemm(ws + W.dqrecv[b], qseg, wq, HqD, q0 * d, qstep);
    gw[0] = dw_gemm(ws + W.dqrecv[b], qseg, dwq, q0 * d, qstep);
    if (P.kv_last(s)) {
      gx[1] = dx_gemm(ws + W.dkrecv, kseg, wk, HkvD, kv0 * d, kseg);
      gx[2] = dx_gemm(ws + W.dvrecv, kseg, wv, HkvD, kv0 * d, kseg);
      gw[1] = dw_gemm(ws + W.dkrecv, kseg, dwk, kv0 * d, kseg);
      gw[2] = dw_gemm(ws + W.dvrecv, kseg, dwv, kv0 * d, kseg);
      if (P.naive && s % P.sigma != 0)      // naive schedule: later stages of a group add their partial dK/dV
        gw[1].c.epi = gw[2].c.epi = Epi::kAccF32;
      n = 3;
    }
    dx_epi(gx[0]);
    R.run(UPIPE_TRACE_GEMM, q, "dX(dQ,dK,dV)", [&](char* e) {
      return gemm_run_group(gx, n, GemmGroup::kKConcat, q, e, 512);
    });
    // M-concatenation needs the dWq / dWk row blocks in whole 128-row tiles
    if (gw[0].M % 128 == 0 && (n == 1 || gw[1].M % 128 == 0)) {
      R.run(UPIPE_TRACE_GEMM, q, "dW(q,k,v)", [&](char* e) {
        return gemm_run_group(gw, n, GemmGroup::kMConcat, q, e, 512);
      });
    } else {
      for (int i = 0; i < n; ++i)
        R.run(UPIPE_TRACE_GEMM, q, "dW", [&](char* e) { return gemm_run(gw[i], q, e, 512); });
    }
  };

  const int nu = P.nstages;
  if (dir) {
    // N2 (see the forward): Q/K/V and dO (+ delta) pushed by their projection epilogues, dQ by its
    // conversion, dK/dV by the attention-backward epilogue at the super-stage end
    for (int s = 0; s < nu && R.status == UPIPE_OK; ++s) {
      const uint32_t e_in = push_begin("direct Q/K/V/dO begin", st);
      pre(s, 0, st);
      push_end(e_in, "direct Q/K/V/dO end", st);
      probe_in(s, 0, st);
      const uint32_t e_out = push_begin("direct dQ/dK/dV begin", st);
      attn(s, 0, st);
      push_end(e_out, "direct dQ/dK/dV end", st);
      probe_out(s, 0, st);
      post(s, 0, st);
    }
  } else if (!ov) {
    for (int s = 0; s < nu && R.status == UPIPE_OK; ++s) {
      pre(s, 0, st);
      if (C > 1) inp(s, 0, st);
      else probe_in(s, 0, st);
      attn(s, 0, st);
      if (C > 1) outa(s, 0, st);
      else probe_out(s, 0, st);
      post(s, 0, st);
    }
  } else {
    // ---- overlapped schedule (same event protocol as the forward, plus the single dK/dV buffers)
    cudaStream_t cs = ctx->pipe.comm;
    cudaEvent_t* ev = ctx->pipe.ev;
    cudaEvent_t e_begin = ev[0], *e_pre = ev + 1, *e_in = ev + 3, *e_attn = ev + 5, *e_out = ev + 7,
                *e_post = ev + 9, e_kvout = ev[11], e_kvpost = ev[12];
    bool kv_inflight = false;
    cudaEventRecord(e_begin, st);
    cudaStreamWaitEvent(cs, e_begin, 0);
    pre(0, 0, st);
    cudaEventRecord(e_pre[0], st);
    cudaStreamWaitEvent(cs, e_pre[0], 0);
    inp(0, 0, cs);
    cudaEventRecord(e_in[0], cs);
    for (int s = 0; s < nu && R.status == UPIPE_OK; ++s) {
      const int b = s & 1;
      if (s + 1 < nu) {
        const int b1 = (s + 1) & 1;
        if (s >= 1) cudaStreamWaitEvent(st, e_in[b1], 0);
        if (P.kv_sent(s + 1)) cudaStreamWaitEvent(st, e_in[b], 0);
        pre(s + 1, b1, st);
        cudaEventRecord(e_pre[b1], st);
        cudaStreamWaitEvent(cs, e_pre[b1], 0);
        if (s >= 1) cudaStreamWaitEvent(cs, e_attn[b1], 0);
        inp(s + 1, b1, cs);
        cudaEventRecord(e_in[b1], cs);
      }
      cudaStreamWaitEvent(st, e_in[b], 0);
      if (P.kv_last(s) && kv_inflight) cudaStreamWaitEvent(st, e_kvout, 0);   // previous dK/dV a2a read dk/dvsend
      attn(s, b, st);
      cudaEventRecord(e_attn[b], st);
      // post(s-1) is enqueued before out(s) so that out(s) can wait for it when both use the dK/dV buffers
      if (s >= 1) {
        cudaStreamWaitEvent(st, e_out[(s - 1) & 1], 0);
        post(s - 1, (s - 1) & 1, st);
        cudaEventRecord(e_post[(s - 1) & 1], st);
        if (P.kv_last(s - 1)) cudaEventRecord(e_kvpost, st);
      }
      cudaStreamWaitEvent(cs, e_attn[b], 0);
      if (s >= 2) cudaStreamWaitEvent(cs, e_post[b], 0);                        // post(s-2) read dQ receive set b
      if (P.kv_last(s) && kv_inflight) cudaStreamWaitEvent(cs, e_kvpost, 0);  // previous post read dk/dvrecv
      outa(s, b, cs);
      cudaEventRecord(e_out[b], cs);
      if (P.kv_last(s)) {
        cudaEventRecord(e_kvout, cs);
        kv_inflight = true;
      }
    }
    cudaStreamWaitEvent(st, e_out[(nu - 1) & 1], 0);
    post(nu - 1, (nu - 1) & 1, st);
  }
  if (gbuf && R.status == UPIPE_OK) final_g(st);
  if (qknorm && R.status == UPIPE_OK)
    R.run(UPIPE_TRACE_AUX, st, "d(gamma) out", [&](char*) {
      cudaError_t e = cudaMemcpyAsync(qkn->dq_norm_w, ws + W.dgam, (size_t)d * 4, cudaMemcpyDeviceToDevice, st);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(qkn->dk_norm_w, ws + W.dgam + (size_t)d * 4, (size_t)d * 4, cudaMemcpyDeviceToDevice, st);
      return e;
    });
  // B7: dW summed over the CP group (the FSDP gradient reduction of P:437, A14)
  if (reduce_dw && T.size() > 1 && R.status == UPIPE_OK) {
    if (qknorm) {
      R.comm(st, "allreduce d(gamma_q)", [&](std::string& m) { return T.allreduce_sum_f32(qkn->dq_norm_w, d, st, m); });
      R.comm(st, "allreduce d(gamma_k)", [&](std::string& m) { return T.allreduce_sum_f32(qkn->dk_norm_w, d, st, m); });
    }
    R.comm(st, "allreduce dWq", [&](std::string& m) { return T.allreduce_sum_f32(dwq, (size_t)HqD * P.D, st, m); });
    R.comm(st, "allreduce dWk", [&](std::string& m) { return T.allreduce_sum_f32(dwk, (size_t)HkvD * P.D, st, m); });
    R.comm(st, "allreduce dWv", [&](std::string& m) { return T.allreduce_sum_f32(dwv, (size_t)HkvD * P.D, st, m); });
    R.comm(st, "allreduce dWo", [&](std::string& m) { return T.allreduce_sum_f32(dwo, (size_t)HqD * P.D, st, m); });
  }
  return R.status;
}

}  // namespace upipe
