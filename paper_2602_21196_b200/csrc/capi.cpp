// extern "C" boundary of libupipe (include/upipe.h). Validation before enqueue,
// status codes, no exceptions across the ABI.
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <atomic>
#include <map>
#include <string>
#include <new>

#include "kernels.h"
#include "upipe_internal.h"

static_assert(sizeof(upipe_shape_t) == 48, "upipe_shape_t layout is part of the ABI (Python mirror in upipe.py)");
static_assert(sizeof(upipe_probe_t) == 104, "upipe_probe_t layout (Python mirror in upipe.py)");

namespace upipe {
upipe_status_t layer_fwd(upipe_ctx_s* ctx, const Plan& P, const upipe_bf16* x, const upipe_bf16* wq,
                         const upipe_bf16* wk, const upipe_bf16* wv, const upipe_bf16* wo, const upipe_qk_norm_t* qkn,
                         upipe_bf16* y, upipe_bf16* o_saved, float* lse_saved, char* ws, cudaStream_t st);
upipe_status_t layer_bwd(upipe_ctx_s* ctx, const Plan& P, const upipe_bf16* x, const upipe_bf16* wq,
                         const upipe_bf16* wk, const upipe_bf16* wv, const upipe_bf16* wo, const upipe_qk_norm_t* qkn,
                         const upipe_bf16* dy, const upipe_bf16* o_saved, const float* lse_saved, upipe_bf16* dx,
                         float* dwq, float* dwk, float* dwv, float* dwo, int reduce_dw, char* ws, cudaStream_t st);
}  // namespace upipe

namespace upipe {
static std::atomic<uint64_t> g_launches{0};
void count_launches(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace upipe

using namespace upipe;

namespace {
thread_local std::string g_err;

upipe_status_t set_err(upipe_ctx_t ctx, upipe_status_t st, const std::string& m) {
  if (ctx) ctx->last_error = m;
  g_err = m;
  return st;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

upipe_status_t check_ctx(upipe_ctx_t ctx) {
  if (!ctx || !ctx->alive || !ctx->transport) return set_err(nullptr, UPIPE_ERR_STATE, "ctx not initialised or finalised");
  if (ctx->ipc_pending) return set_err(ctx, UPIPE_ERR_STATE, "IPC ctx not connected (upipe_ipc_connect)");
  return UPIPE_OK;
}

// The layer's workspace: the ctx's symmetric region for an IPC ctx, else the caller's.
bool resolve_ws(upipe_ctx_t ctx, void*& ws, size_t& ws_bytes) {
  if (char* w = ctx->transport->workspace()) {
    ws = w;
    ws_bytes = ctx->transport->workspace_bytes();
  }
  return ws != nullptr;
}

upipe_status_t cuda_status(cudaError_t e, const char* what, const char* detail = nullptr) {
  if (e == cudaSuccess) return UPIPE_OK;
  return set_err(nullptr, UPIPE_ERR_CUDA, std::string(what) + ": " + (detail && detail[0] ? detail : cudaGetErrorString(e)));
}

template <class... P>
bool all_aligned(P... ps) {
  return (aligned16(ps) && ...);
}
}  // namespace

extern "C" {

const char* upipe_status_string(upipe_status_t s) {
  switch (s) {
    case UPIPE_OK: return "UPIPE_OK";
    case UPIPE_ERR_INVALID_ARG: return "UPIPE_ERR_INVALID_ARG";
    case UPIPE_ERR_UNSUPPORTED: return "UPIPE_ERR_UNSUPPORTED";
    case UPIPE_ERR_CUDA: return "UPIPE_ERR_CUDA";
    case UPIPE_ERR_COMM: return "UPIPE_ERR_COMM";
    case UPIPE_ERR_WORKSPACE: return "UPIPE_ERR_WORKSPACE";
    case UPIPE_ERR_STATE: return "UPIPE_ERR_STATE";
  }
  return "UPIPE_ERR_UNKNOWN";
}

const char* upipe_last_error(upipe_ctx_t ctx) { return ctx ? ctx->last_error.c_str() : g_err.c_str(); }

upipe_status_t upipe_get_unique_id(uint8_t uid[UPIPE_UID_BYTES]) {
  if (!uid) return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "uid == NULL");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return set_err(nullptr, UPIPE_ERR_COMM, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  std::memset(uid, 0, UPIPE_UID_BYTES);
  std::memcpy(uid, &id, sizeof(id));
  return UPIPE_OK;
}

upipe_status_t upipe_init(upipe_ctx_t* out, const uint8_t uid[UPIPE_UID_BYTES], int cp_size, int cp_rank,
                          int cuda_device, uint32_t flags) {
  if (!out) return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "ctx == NULL");
  *out = nullptr;
  if (cp_size < 1 || cp_rank < 0 || cp_rank >= cp_size)
    return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "cp_rank must be in [0, cp_size)");
  if (cp_size > 1 && !uid) return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "uid == NULL with cp_size > 1");
  cudaError_t e = cudaSetDevice(cuda_device);
  if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
  auto* c = new (std::nothrow) upipe_ctx_s();
  if (!c) return set_err(nullptr, UPIPE_ERR_STATE, "out of host memory");
  c->device = cuda_device;
  c->C = cp_size;
  c->rank = cp_rank;
  c->flags = flags;
  std::string err;
  c->transport = cp_size == 1 ? make_self_transport() : make_nccl_transport(uid, cp_size, cp_rank, err);
  if (!c->transport) {
    delete c;
    return set_err(nullptr, UPIPE_ERR_COMM, err);
  }
  *out = c;
  return UPIPE_OK;
}

upipe_status_t upipe_init_local(upipe_ctx_t* out, upipe_fabric_t fabric, int cp_rank, int cuda_device,
                                uint32_t flags) {
  if (!out || !fabric) return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "ctx or fabric == NULL");
  *out = nullptr;
  cudaError_t e = cudaSetDevice(cuda_device);
  if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
  std::string err;
  auto t = make_fabric_transport(fabric, cp_rank, cuda_device, err);
  if (!t) return set_err(nullptr, UPIPE_ERR_INVALID_ARG, err);
  auto* c = new (std::nothrow) upipe_ctx_s();
  if (!c) return set_err(nullptr, UPIPE_ERR_STATE, "out of host memory");
  c->device = cuda_device;
  c->C = t->size();
  c->rank = cp_rank;
  c->flags = flags;
  c->transport = std::move(t);
  *out = c;
  return UPIPE_OK;
}

namespace {
// workspace + dW scratch of an IPC ctx for shapes up to sh
void ipc_sizes(int C, const upipe_shape_t& sh, uint32_t flags, size_t* ws, size_t* scratch) {
  Plan P = make_plan(C, sh);
  P.naive = (flags & UPIPE_FLAG_NAIVE_KV) != 0;
  const bool ov = overlap_enabled(flags, P), dir = direct_enabled(flags, P);
  *ws = std::max(fwd_workspace(P, ov, dir).total, bwd_workspace(P, ov, dir).total);
  const size_t hq = (size_t)sh.n_q_heads * sh.head_dim, hkv = (size_t)sh.n_kv_heads * sh.head_dim;
  *scratch = std::max(hq, hkv) * (size_t)sh.hidden * 4;
}
}  // namespace

upipe_status_t upipe_ipc_region_size(int cp_size, const upipe_shape_t* shape, uint32_t flags, size_t* bytes) {
  std::string m;
  if (upipe_status_t st = validate_shape(cp_size, shape, m)) return set_err(nullptr, st, m);
  if (!bytes) return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "bytes == NULL");
  size_t ws = 0, sc = 0;
  ipc_sizes(cp_size, *shape, flags, &ws, &sc);
  *bytes = ipc_region_bytes(ws, sc);
  return UPIPE_OK;
}

upipe_status_t upipe_ipc_create(upipe_ctx_t* out, int cp_size, int cp_rank, int cuda_device, uint32_t flags,
                                const upipe_shape_t* shape, uint8_t handle[UPIPE_IPC_HANDLE_BYTES]) {
  if (!out || !handle) return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "ctx or handle == NULL");
  *out = nullptr;
  if (cp_size < 1 || cp_rank < 0 || cp_rank >= cp_size)
    return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "cp_rank must be in [0, cp_size)");
  std::string m;
  if (upipe_status_t st = validate_shape(cp_size, shape, m)) return set_err(nullptr, st, m);
  cudaError_t e = cudaSetDevice(cuda_device);
  if (e != cudaSuccess) return cuda_status(e, "cudaSetDevice");
  size_t ws = 0, sc = 0;
  ipc_sizes(cp_size, *shape, flags, &ws, &sc);
  std::string err;
  auto t = make_ipc_transport(cp_size, cp_rank, cuda_device, ws, sc, handle, err);
  if (!t) return set_err(nullptr, UPIPE_ERR_CUDA, err);
  auto* c = new (std::nothrow) upipe_ctx_s();
  if (!c) return set_err(nullptr, UPIPE_ERR_STATE, "out of host memory");
  c->device = cuda_device;
  c->C = cp_size;
  c->rank = cp_rank;
  c->flags = flags;
  c->transport = std::move(t);
  c->ipc_pending = true;
  *out = c;
  return UPIPE_OK;
}

upipe_status_t upipe_ipc_connect(upipe_ctx_t ctx, const uint8_t* handles) {
  if (!ctx || !ctx->transport) return set_err(nullptr, UPIPE_ERR_STATE, "ctx not initialised");
  if (!handles) return set_err(ctx, UPIPE_ERR_INVALID_ARG, "handles == NULL");
  cudaSetDevice(ctx->device);
  std::string err;
  if (upipe_status_t st = ipc_connect(ctx->transport.get(), handles, err)) return set_err(ctx, st, err);
  ctx->ipc_pending = false;
  return UPIPE_OK;
}

upipe_status_t upipe_finalize(upipe_ctx_t ctx) {
  if (!ctx) return set_err(nullptr, UPIPE_ERR_STATE, "ctx == NULL");
  ctx->transport.reset();
  ctx->alive = false;
  delete ctx;
  return UPIPE_OK;
}

upipe_status_t upipe_wait(upipe_ctx_t ctx, void* stream, int64_t timeout_ms) {
  if (upipe_status_t st = check_ctx(ctx)) return st;
  cudaSetDevice(ctx->device);
  std::string err;
  const upipe_status_t st = ctx->transport->wait(static_cast<cudaStream_t>(stream), timeout_ms / 1000.0, err);
  if (st != UPIPE_OK) return set_err(ctx, st, "upipe_wait: " + err);
  return UPIPE_OK;
}

upipe_status_t upipe_comm_info(upipe_ctx_t ctx, upipe_comm_info_t* info) {
  if (upipe_status_t st = check_ctx(ctx)) return st;
  if (!info) return set_err(ctx, UPIPE_ERR_INVALID_ARG, "info == NULL");
  info->nranks = ctx->transport->size();
  info->rank = ctx->transport->rank();
  const int dev = ctx->transport->device();
  info->cuda_device = dev >= 0 ? dev : ctx->device;
  info->transport = ctx->transport->kind();
  info->max_ctas = ctx->transport->max_ctas();
  return UPIPE_OK;
}

upipe_status_t upipe_validate(int cp_size, const upipe_shape_t* shape, char* msg, size_t msg_len) {
  std::string m;
  upipe_status_t st = validate_shape(cp_size, shape, m);
  if (msg && msg_len) snprintf(msg, msg_len, "%s", m.c_str());
  if (st != UPIPE_OK) set_err(nullptr, st, m);
  return st;
}

upipe_status_t upipe_workspace_size(int cp_size, const upipe_shape_t* shape, int pass, size_t* bytes) {
  std::string m;
  upipe_status_t st = validate_shape(cp_size, shape, m);
  if (st != UPIPE_OK) return set_err(nullptr, st, m);
  if (!bytes || pass < 0 || (pass & 7) > 5 || pass > 15)
    return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "pass must be 0..5, plus 8 for UPIPE_FLAG_NAIVE_KV");
  Plan P = make_plan(cp_size, *shape);
  P.naive = (pass & 8) != 0;
  pass &= 7;
  const bool ov = pass < 2 && P.C > 1 && P.ring == 1;   // 0/1: default (overlapped for C > 1); 2/3: sequential
  const bool dir = pass >= 4 && direct_enabled(UPIPE_FLAG_DIRECT, P);   // 4/5: UPIPE_FLAG_DIRECT
  *bytes = (pass & 1) == 0 ? fwd_workspace(P, ov, dir).total : bwd_workspace(P, ov, dir).total;
  return UPIPE_OK;
}

upipe_status_t upipe_plan_stage(int cp_size, const upipe_shape_t* shape, int stage, int device,
                                upipe_stage_info_t* out) {
  std::string m;
  upipe_status_t st = validate_shape(cp_size, shape, m);
  if (st != UPIPE_OK) return set_err(nullptr, st, m);
  const Plan P = make_plan(cp_size, *shape);
  if (!out || stage < 0 || stage >= P.nstages || device < 0 || device >= P.C)   // device: Ulysses index
    return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "stage or device out of range");
  out->n_stages = P.nstages;
  out->qpd = P.qpd;
  out->kv_res = P.kv_res;
  out->sigma = P.sigma;
  out->q0 = P.q0(stage, device);
  out->kv0 = P.kv0(stage, device);
  out->kv_sent = P.kv_sent(stage) ? 1 : 0;
  return UPIPE_OK;
}

namespace {
// the q/k norm weights a shape with qk_norm_eps > 0 needs (fwd: weights; bwd: weights and gradients)
upipe_status_t check_qkn(upipe_ctx_t ctx, const upipe_shape_t* shape, const upipe_qk_norm_t* qkn, bool bwd) {
  if (shape->qk_norm_eps <= 0.f) return UPIPE_OK;
  if (!qkn || !qkn->q_norm_w || !qkn->k_norm_w || (bwd && (!qkn->dq_norm_w || !qkn->dk_norm_w)))
    return set_err(ctx, UPIPE_ERR_INVALID_ARG, "qk_norm_eps > 0 needs upipe_qk_norm_t weights (and gradients in bwd)");
  if (!all_aligned(qkn->q_norm_w, qkn->k_norm_w) || (bwd && !all_aligned(qkn->dq_norm_w, qkn->dk_norm_w)))
    return set_err(ctx, UPIPE_ERR_INVALID_ARG, "q/k norm weights must be 16-byte aligned");
  return UPIPE_OK;
}
}  // namespace

upipe_status_t upipe_attn_fwd(upipe_ctx_t ctx, const upipe_shape_t* shape, const upipe_bf16* x, const upipe_bf16* wq,
                              const upipe_bf16* wk, const upipe_bf16* wv, const upipe_bf16* wo, upipe_bf16* y,
                              upipe_bf16* o_saved, float* lse_saved, void* workspace, size_t ws_bytes,
                              void* stream) {
  return upipe_attn_fwd_ex(ctx, shape, x, wq, wk, wv, wo, nullptr, y, o_saved, lse_saved, workspace, ws_bytes, stream);
}

upipe_status_t upipe_attn_fwd_ex(upipe_ctx_t ctx, const upipe_shape_t* shape, const upipe_bf16* x,
                                 const upipe_bf16* wq, const upipe_bf16* wk, const upipe_bf16* wv, const upipe_bf16* wo,
                                 const upipe_qk_norm_t* qkn, upipe_bf16* y, upipe_bf16* o_saved, float* lse_saved,
                                 void* workspace, size_t ws_bytes, void* stream) {
  if (upipe_status_t st = check_ctx(ctx)) return st;
  std::string m;
  if (upipe_status_t st = validate_shape(ctx->C, shape, m)) return set_err(ctx, st, m);
  if (upipe_status_t st = check_qkn(ctx, shape, qkn, false)) return st;
  if (!x || !wq || !wk || !wv || !wo || !y || !o_saved || !lse_saved || !resolve_ws(ctx, workspace, ws_bytes))
    return set_err(ctx, UPIPE_ERR_INVALID_ARG, "null tensor pointer");
  if (!all_aligned(x, wq, wk, wv, wo, y, o_saved, lse_saved) || (reinterpret_cast<uintptr_t>(workspace) & 255))
    return set_err(ctx, UPIPE_ERR_INVALID_ARG, "tensors must be 16-byte aligned, workspace 256-byte aligned");
  Plan P = make_plan(ctx->C, *shape);
  P.naive = (ctx->flags & UPIPE_FLAG_NAIVE_KV) != 0;
  if (ws_bytes < fwd_workspace(P, overlap_enabled(ctx->flags, P), direct_enabled(ctx->flags, P)).total)
    return set_err(ctx, UPIPE_ERR_WORKSPACE, "ws_bytes < upipe_workspace_size(pass=0, or 2 with UPIPE_FLAG_SYNC_COMM)");
  cudaSetDevice(ctx->device);
  return layer_fwd(ctx, P, x, wq, wk, wv, wo, qkn, y, o_saved, lse_saved, static_cast<char*>(workspace),
                   static_cast<cudaStream_t>(stream));
}

upipe_status_t upipe_attn_bwd(upipe_ctx_t ctx, const upipe_shape_t* shape, const upipe_bf16* x, const upipe_bf16* wq,
                              const upipe_bf16* wk, const upipe_bf16* wv, const upipe_bf16* wo,
                              const upipe_bf16* dy, const upipe_bf16* o_saved, const float* lse_saved,
                              upipe_bf16* dx, float* dwq, float* dwk, float* dwv, float* dwo, int reduce_dw,
                              void* workspace, size_t ws_bytes, void* stream) {
  return upipe_attn_bwd_ex(ctx, shape, x, wq, wk, wv, wo, nullptr, dy, o_saved, lse_saved, dx, dwq, dwk, dwv, dwo,
                           reduce_dw, workspace, ws_bytes, stream);
}

upipe_status_t upipe_attn_bwd_ex(upipe_ctx_t ctx, const upipe_shape_t* shape, const upipe_bf16* x,
                                 const upipe_bf16* wq, const upipe_bf16* wk, const upipe_bf16* wv, const upipe_bf16* wo,
                                 const upipe_qk_norm_t* qkn, const upipe_bf16* dy, const upipe_bf16* o_saved,
                                 const float* lse_saved, upipe_bf16* dx, float* dwq, float* dwk, float* dwv, float* dwo,
                                 int reduce_dw, void* workspace, size_t ws_bytes, void* stream) {
  if (upipe_status_t st = check_ctx(ctx)) return st;
  std::string m;
  if (upipe_status_t st = validate_shape(ctx->C, shape, m)) return set_err(ctx, st, m);
  if (upipe_status_t st = check_qkn(ctx, shape, qkn, true)) return st;
  if (!x || !wq || !wk || !wv || !wo || !dy || !o_saved || !lse_saved || !dx || !dwq || !dwk || !dwv || !dwo ||
      !resolve_ws(ctx, workspace, ws_bytes))
    return set_err(ctx, UPIPE_ERR_INVALID_ARG, "null tensor pointer");
  if (!all_aligned(x, wq, wk, wv, wo, dy, o_saved, lse_saved, dx, dwq, dwk, dwv, dwo) ||
      (reinterpret_cast<uintptr_t>(workspace) & 255))
    return set_err(ctx, UPIPE_ERR_INVALID_ARG, "tensors must be 16-byte aligned, workspace 256-byte aligned");
  Plan P = make_plan(ctx->C, *shape);
  P.naive = (ctx->flags & UPIPE_FLAG_NAIVE_KV) != 0;
  if (ws_bytes < bwd_workspace(P, overlap_enabled(ctx->flags, P), direct_enabled(ctx->flags, P)).total)
    return set_err(ctx, UPIPE_ERR_WORKSPACE, "ws_bytes < upipe_workspace_size(pass=1, or 3 with UPIPE_FLAG_SYNC_COMM)");
  cudaSetDevice(ctx->device);
  return layer_bwd(ctx, P, x, wq, wk, wv, wo, qkn, dy, o_saved, lse_saved, dx, dwq, dwk, dwv, dwo, reduce_dw,
                   static_cast<char*>(workspace), static_cast<cudaStream_t>(stream));
}

upipe_status_t upipe_attn_core_fwd(const upipe_bf16* q, const upipe_bf16* k, const upipe_bf16* v, upipe_bf16* o,
                                   float* lse, int64_t S, int nq, int nkv, int d, int causal, int64_t ldq,
                                   int64_t ldkv, int64_t ldo, int64_t ld_lse, void* stream) {
  if (!q || !k || !v || !o || !lse || S < 1 || nq < 1 || nkv < 1 || nq % nkv)
    return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "attn_core_fwd: bad arguments");
  if (!all_aligned(q, k, v, o) || ldq % 8 || ldkv % 8 || ldo % 8)
    return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "attn_core_fwd: 16-byte alignment of tensors and strides");
  AttnFwdProblem p{q, k, v, o, lse, S, nq, nkv, d, causal, ldq, ldkv, ldo, ld_lse};
  char err[512] = {0};
  return cuda_status(attn_fwd_run(p, static_cast<cudaStream_t>(stream), err, sizeof err), "attn_fwd", err);
}

upipe_status_t upipe_attn_core_bwd(const upipe_bf16* q, const upipe_bf16* k, const upipe_bf16* v,
                                   const upipe_bf16* dout, const float* lse, const float* delta, float* dq_acc,
                                   float* dk_acc, float* dv_acc, int64_t S, int nq, int nkv, int d, int causal,
                                   int64_t ldq, int64_t ldkv, int64_t ldo_grad, int64_t ld_lse, int64_t ld_delta,
                                   int flags, int32_t* dq_sem, void* stream) {
  if (!q || !k || !v || !dout || !lse || !delta || !dq_acc || !dk_acc || !dv_acc || S < 1 || nq < 1 || nkv < 1 ||
      nq % nkv)
    return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "attn_core_bwd: bad arguments");
  if (!all_aligned(q, k, v, dout, dq_acc, dk_acc, dv_acc) || ldq % 8 || ldkv % 8 || ldo_grad % 8)
    return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "attn_core_bwd: 16-byte alignment of tensors and strides");
  AttnBwdProblem p{};
  p.q = q; p.k = k; p.v = v; p.dout = dout; p.lse = lse; p.delta = delta;
  p.dq_acc = dq_acc; p.dk_acc = dk_acc; p.dv_acc = dv_acc;
  p.S = S; p.nq = nq; p.nkv = nkv; p.d = d; p.causal = causal;
  p.ldq = ldq; p.ldkv = ldkv; p.ldo_grad = ldo_grad; p.ld_lse = ld_lse; p.ld_delta = ld_delta; p.ld_kvb = 0;
  p.kv_accumulate = (flags & UPIPE_CORE_ACCUMULATE) ? 1 : 0;
  p.kv_write_acc = 1;
  if (flags & UPIPE_CORE_DQ_DIM_MAJOR) {
    p.dq_dim_major = 1;
    p.ld_dqt = (S + 3) & ~int64_t(3);   // TMA: 16-byte row stride
    if (!attn_bwd_dq_dim_major_supported(p))
      return set_err(nullptr, UPIPE_ERR_UNSUPPORTED, "attn_core_bwd: dim-major dQ needs the 64-query kernel (d = 128)");
  }
  if (flags & UPIPE_CORE_DETERMINISTIC) {
    if (!dq_sem) return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "attn_core_bwd: deterministic mode needs dq_sem");
    p.dq_sem = dq_sem;
  }
  char err[512] = {0};
  return cuda_status(attn_bwd_run(p, static_cast<cudaStream_t>(stream), err, sizeof err), "attn_bwd", err);
}

int64_t upipe_core_bwd_sem_count(int64_t S, int nq) { return S < 1 || nq < 1 ? 0 : attn_bwd_sem_count(S, nq); }

upipe_status_t upipe_rowdot(const upipe_bf16* dO, int64_t ld_do, const upipe_bf16* O, int64_t ld_o, float* delta,
                            int64_t ld_delta, int64_t rows, int nheads, int d, void* stream) {
  if (!dO || !O || !delta || (d != 64 && d != 128) || !all_aligned(dO, O) || ld_do % 8 || ld_o % 8)
    return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "rowdot: bad arguments");
  return cuda_status(rowdot_run(dO, ld_do, O, ld_o, delta, ld_delta, rows, nheads, d, static_cast<cudaStream_t>(stream)),
                     "rowdot");
}

upipe_status_t upipe_gemm_xwT(const upipe_bf16* x, const upipe_bf16* w, void* y, int64_t M, int64_t N, int64_t K,
                              int mode, void* stream) {
  if (!x || !w || !y || M < 1 || N < 1 || K < 1 || N % 64 || K % 8 || (mode != 0 && mode != 1) ||
      !all_aligned(x, w, y))
    return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "gemm_xwT: bad arguments (N % 64, K % 8, alignment)");
  GemmProblem g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.a = OperandMap{x, K, M, K, false};
  g.b = OperandMap{w, K, N, K, false};
  if (mode == 0) {
    g.c.out_bf16 = y;
    g.c.ld_bf16 = N;
    g.c.epi = Epi::kStoreBF16;
  } else {
    g.c.out_f32 = y;
    g.c.ld_f32 = N;
    g.c.epi = Epi::kStoreF32;
  }
  char err[512] = {0};
  return cuda_status(gemm_run(g, static_cast<cudaStream_t>(stream), err, sizeof err), "gemm", err);
}

upipe_status_t upipe_synth_fill_bf16(upipe_bf16* dst, int64_t n, uint64_t seed, int tensor_id, int exponent,
                                     int64_t start, void* stream) {
  if (!dst || n < 0) return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "synth_fill: bad arguments");
  return cuda_status(synth_fill_bf16_run(dst, n, seed, tensor_id, exponent, start, static_cast<cudaStream_t>(stream)),
                     "synth_fill");
}

upipe_status_t upipe_kernel_launches(uint64_t* count) {
  if (!count) return set_err(nullptr, UPIPE_ERR_INVALID_ARG, "count == NULL");
  *count = g_launches.load();
  return UPIPE_OK;
}

upipe_status_t upipe_test_set_probe(upipe_ctx_t ctx, const upipe_probe_t* probe) {
  if (upipe_status_t st = check_ctx(ctx)) return st;
  if (!probe) return set_err(ctx, UPIPE_ERR_INVALID_ARG, "probe == NULL");
  ctx->probe = *probe;
  return UPIPE_OK;
}

upipe_status_t upipe_set_trace(upipe_ctx_t ctx, int on) {
  if (upipe_status_t st = check_ctx(ctx)) return st;
  ctx->tracer.on = on != 0;
  return UPIPE_OK;
}

upipe_status_t upipe_trace_read(upipe_ctx_t ctx, double ms[UPIPE_TRACE_NCAT], int64_t count[UPIPE_TRACE_NCAT]) {
  if (upipe_status_t st = check_ctx(ctx)) return st;
  if (!ms || !count) return set_err(ctx, UPIPE_ERR_INVALID_ARG, "ms/count == NULL");
  for (int i = 0; i < UPIPE_TRACE_NCAT; ++i) {
    ms[i] = 0;
    count[i] = 0;
  }
  cudaSetDevice(ctx->device);
  Tracer& T = ctx->tracer;
  // UPIPE_TRACE_LABELS=1: also print per-step-label totals (debugging aid) to stderr
  const char* lenv = getenv("UPIPE_TRACE_LABELS");
  std::map<std::string, std::pair<double, int>> by_label;
  for (auto& r : T.recs) {
    cudaError_t e = cudaEventSynchronize(r.b);
    float t = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.a, r.b);
    if (e != cudaSuccess) return set_err(ctx, UPIPE_ERR_CUDA, std::string("trace: ") + cudaGetErrorString(e));
    ms[r.cat] += t;
    count[r.cat] += 1;
    if (lenv && lenv[0] == '1') {
      auto& v = by_label[r.label ? r.label : ""];
      v.first += t;
      v.second += 1;
    }
    T.pool.push_back(r.a);
    T.pool.push_back(r.b);
  }
  T.recs.clear();
  for (auto& kv : by_label)
    fprintf(stderr, "[upipe trace] %-24s %4d x  %9.3f ms\n", kv.first.c_str(), kv.second.second, kv.second.first);
  return UPIPE_OK;
}

}  // extern "C"
