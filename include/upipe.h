/*
 * upipe.h -- C ABI of libupipe: UPipe ("Untied Ulysses", arXiv 2602.21196), the
 * headwise-chunked Ulysses context-parallel attention layer, forward and backward,
 * for NVIDIA B200 (sm_100a).
 *
 * Citations: P:n = PAPER.md line n (reference text of the paper), S:n = SPEC.md
 * line n. Readings of points the paper leaves open are numbered A1..A25 in
 * DESIGN.md ("Readings").
 *
 * What one layer call computes (§3.1, §3.3, §4.1):
 * the input is sequence-sharded (rank r holds tokens [r*S_l, (r+1)*S_l), P:274;
 * DESIGN A7). Heads are processed in nu = Hq/U stages of U heads. For
 * each stage the layer projects Q/K/V for only that stage's heads, runs
 * an all-to-all from sequence- to head-sharded layout (inp_all_to_all, P:317,
 * Q then K then V), computes causal GQA attention over the full sequence
 * for its U/C heads, runs the all-to-all back (out_all_to_all),
 * fills the pre-allocated output and accumulates the output
 * projection (BASELINE north_star). One chunk-sized buffer set in the caller's
 * workspace is reused by every stage. K/V heads are sent once
 * per super-stage and kept resident (GQA scheduling).
 * chunk_heads == n_q_heads is DeepSpeed-Ulysses on the same kernels.
 *
 * The result equals un-sharded multi-head causal GQA attention with projections
 * (SURVEY §8c c.1): U and C change only the order of the work.
 *
 * Conventions
 *  - bf16 tensors are passed as uint16_t storage (upipe_bf16). fp32 is float.
 *  - All tensor pointers are DEVICE pointers unless stated otherwise, 16-byte
 *    aligned, row-major, owned by the caller (PyTorch). The library never frees
 *    caller memory. Workspace is caller-owned too, so all activation memory is
 *    visible to the caller's allocator.
 *  - Weights use nn.Linear layout [out, in] (y = x W^T); q head h owns rows
 *    [h*d, (h+1)*d) of Wq and columns [h*d, (h+1)*d) of Wo; kv head g rows
 *    [g*d,(g+1)*d) of Wk/Wv; q head h reads kv head floor(h / (Hq/Hkv)) (A3, A4).
 *  - Scale 1/sqrt(head_dim) (A1); causal: key j visible to query i iff j <= i in
 *    the global token index (A2). No bias, RoPE, dropout (A6).
 *  - Calls are asynchronous: work is enqueued on `stream` (the ctx's transport
 *    may enqueue on it too) and outputs are valid when `stream` reaches that
 *    point. Inputs must stay alive and unmodified until then.
 *  - Errors: validation happens before anything is enqueued, so a failing call
 *    has no side effects; upipe_last_error(ctx) names the violated constraint.
 *    No C++ exception crosses the ABI. A ctx is not thread-safe; all ranks of a
 *    CP group must make the same sequence of calls (collective contract).
 */
#ifndef UPIPE_H_
#define UPIPE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define UPIPE_API __attribute__((visibility("default")))
#else
#define UPIPE_API
#endif

typedef uint16_t upipe_bf16;

typedef enum {
  UPIPE_OK = 0,
  UPIPE_ERR_INVALID_ARG = 1, /* a documented precondition is violated (named in upipe_last_error) */
  UPIPE_ERR_UNSUPPORTED = 2, /* valid for the method but not implemented (e.g. Hkv % C != 0, A9) */
  UPIPE_ERR_CUDA = 3,        /* a CUDA runtime error (message in upipe_last_error) */
  UPIPE_ERR_COMM = 4,        /* NCCL / fabric error or timeout */
  UPIPE_ERR_WORKSPACE = 5,   /* ws_bytes smaller than upipe_workspace_size */
  UPIPE_ERR_STATE = 6        /* ctx not initialised / already finalised */
} upipe_status_t;

typedef struct upipe_ctx_s* upipe_ctx_t;
typedef struct upipe_fabric_s* upipe_fabric_t;

/* Shape of one layer call on one rank. */
typedef struct {
  int64_t seq_local;   /* S_l = S / C tokens held by this rank (contiguous block r*S_l..); >= 1 */
  int32_t hidden;      /* D, model width (independent of Hq*d, A5); multiple of 64 */
  int32_t n_q_heads;   /* Hq */
  int32_t n_kv_heads;  /* Hkv; Hq % Hkv == 0; Hkv % C == 0 (A9) */
  int32_t head_dim;    /* d in {64, 128} */
  int32_t chunk_heads; /* U: heads per stage; U % C == 0; Hq % U == 0; U/C and Hq/Hkv divide one another (A8) */
  int32_t causal;      /* 1: causal mask (the paper's setting); 0: full attention */
  float rope_base;     /* 0: no rotary embedding; > 1: RoPE on Q and K at their global token positions
                          with angles p * rope_base^(-2i/d) on head-dim pairs (2i, 2i+1) (P:241,
                          SURVEY N3, DESIGN A26; Llama3: 500000). The ctx keeps the rotation tables. */
  int32_t ring_degree; /* r: UPipe x Ring hybrid (P:166 USP; DESIGN A27). 0 or 1:
                          plain UPipe over all C ranks. r > 1: C % r == 0; ranks g = i*a + u (a = C/r)
                          form r Ulysses groups of a consecutive ranks; group i holds the contiguous
                          ring block [i*S_b, (i+1)*S_b), S_b = a*S_l. Every constraint above that
                          names C then applies to a (U % a, Hkv % a, ...). Heads are resharded by
                          all-to-all inside the group; K/V blocks (and, in backward, their fp32
                          gradient accumulators) travel around the ring of the r ranks that share u,
                          and the partial outputs are merged by their log-sum-exp. */
  float qk_norm_eps;   /* 0: off. > 0: Qwen3 per-head RMSNorm of Q and K (the paper's second model family,
                          P:433, DESIGN A29): each head of the projection is divided by
                          sqrt(mean of its squares + qk_norm_eps) and scaled by its weight vector
                          (upipe_qk_norm_t), then rotated (RoPE) if rope_base > 0. Qwen3: 1e-6.
                          Needs upipe_attn_fwd_ex / upipe_attn_bwd_ex. */
} upipe_shape_t;

#define UPIPE_UID_BYTES 128

/* flags for upipe_init / upipe_init_local */
#define UPIPE_FLAG_NONE 0u
#define UPIPE_FLAG_SYNC_COMM 1u /* sequential schedule: collectives on the compute stream, one buffer set */
#define UPIPE_FLAG_NAIVE_KV 2u  /* ablation: re-project and re-send the stage's K/V heads at every
                                   stage instead of once per GQA super-stage ("naive" volume) */
#define UPIPE_FLAG_DETERMINISTIC 4u /* bitwise-reproducible backward: the attention backward
                                   adds the dQ partials of its key tiles in key-tile order (semaphores in
                                   the workspace) instead of in arrival order; slower */
#define UPIPE_FLAG_DIRECT 8u    /* direct-to-peer all-to-alls (P:296 the a2a buffers set the
                                   peak, "we only need buffers for 2 heads"): the producing kernels
                                   write straight into the owners' receive buffers over peer memory -- Q/K/V
                                   projection and dO projection epilogues (TMA stores), the attention
                                   epilogue (O, dK, dV), the dQ conversion -- so no send buffers exist and no
                                   copy or NCCL kernel moves the chunk; ordering by GPU front-end flags.
                                   Needs a ctx from upipe_ipc_create/connect, Ulysses degree <= 8; one
                                   buffer set (the transfers overlap inside the kernels, not on a side
                                   stream). Ignored at C = 1. */

/* ---------------------------------------------------------------- lifecycle */

/* Rank 0 creates the NCCL unique id that all CP ranks pass to upipe_init
 * (the Python binding broadcasts it over the torch process group). */
UPIPE_API upipe_status_t upipe_get_unique_id(uint8_t uid[UPIPE_UID_BYTES]);

/* Create a context for CP rank `cp_rank` of `cp_size` processes (one GPU each)
 * over NCCL (NVLink/NVSwitch). Collective across the group. cp_size == 1 needs no
 * uid (may be NULL). The ctx owns the communicator, a comm stream and events. */
UPIPE_API upipe_status_t upipe_init(upipe_ctx_t* ctx, const uint8_t uid[UPIPE_UID_BYTES], int cp_size, int cp_rank,
                          int cuda_device, uint32_t flags);

/* Single-process CP group: `cp_size` ranks driven by `cp_size` host threads of one
 * process (each with its own ctx and stream, possibly on the same device). The
 * all-to-alls are device-to-device copies between the ranks' buffers. Used to run
 * and test the sharded path (C = 2..8) on one GPU. */
UPIPE_API upipe_status_t upipe_fabric_create(upipe_fabric_t* fabric, int cp_size);
UPIPE_API upipe_status_t upipe_fabric_destroy(upipe_fabric_t fabric);
UPIPE_API upipe_status_t upipe_init_local(upipe_ctx_t* ctx, upipe_fabric_t fabric, int cp_rank, int cuda_device, uint32_t flags);

/* Direct-to-peer transport. One process per rank (one GPU each; several
 * ranks may share a GPU, e.g. in tests). The ctx allocates a symmetric region (cudaMalloc, the same
 * layout on every rank) that holds the layer's whole workspace -- every receive buffer at the same
 * offset on every rank -- plus synchronisation flags and the dW all-reduce scratch; peers map it with
 * CUDA IPC and PUSH their blocks straight into the owner's receive buffers (the projection GEMM's
 * epilogue, the attention epilogue and the dQ conversion write there directly; the remaining transfers
 * use the copy engines), ordered by flags the GPU front end writes and waits on. No NCCL, no send
 * buffers for the fused steps. Two phases; the caller exchanges the opaque handles (e.g. all_gather
 * over a torch process group):
 *   upipe_ipc_create(&ctx, C, rank, device, flags, max_shape, my_handle)
 *   upipe_ipc_connect(ctx, handles)   handles: [cp_size][UPIPE_IPC_HANDLE_BYTES], rank order
 * The region is sized for shapes up to `max_shape` (same heads, seq_local <= max_shape->seq_local);
 * upipe_attn_fwd / upipe_attn_bwd on such a ctx use it and ignore `workspace` (may be NULL, 0).
 * The region is library memory (not the caller's allocator): upipe_ipc_region_size reports it. */
#define UPIPE_IPC_HANDLE_BYTES 128
UPIPE_API upipe_status_t upipe_ipc_region_size(int cp_size, const upipe_shape_t* max_shape, uint32_t flags,
                                               size_t* bytes);
UPIPE_API upipe_status_t upipe_ipc_create(upipe_ctx_t* ctx, int cp_size, int cp_rank, int cuda_device, uint32_t flags,
                                          const upipe_shape_t* max_shape, uint8_t handle[UPIPE_IPC_HANDLE_BYTES]);
UPIPE_API upipe_status_t upipe_ipc_connect(upipe_ctx_t ctx, const uint8_t* handles);

UPIPE_API upipe_status_t upipe_finalize(upipe_ctx_t ctx);
UPIPE_API const char* upipe_status_string(upipe_status_t s);
UPIPE_API const char* upipe_last_error(upipe_ctx_t ctx); /* thread-local message if ctx == NULL */

/* Failure detection. Waits until `stream` has completed the work enqueued so far while
 * polling the ctx's communicator for asynchronous errors (NCCL: ncclCommGetAsyncError). An error, or
 * no completion within timeout_ms (a dead or stalled peer; <= 0: no limit), aborts the communicator
 * (ncclCommAbort: this rank's pending collectives return instead of hanging) and returns
 * UPIPE_ERR_COMM with the reason in upipe_last_error; the ctx must then be finalized. */
UPIPE_API upipe_status_t upipe_wait(upipe_ctx_t ctx, void* stream, int64_t timeout_ms);

/* What the ctx is connected to (for checking a launch: every rank should see nranks == cp_size). */
typedef struct {
  int32_t nranks, rank;
  int32_t cuda_device;  /* the communicator's device (NCCL) or the ctx's device */
  int32_t transport;    /* 0: none (C = 1), 1: NCCL, 2: single-process fabric, 3: IPC direct-to-peer */
  int32_t max_ctas;     /* NCCL CTA cap (UPIPE_NCCL_MAX_CTAS, default 16); 0 if not NCCL */
} upipe_comm_info_t;
UPIPE_API upipe_status_t upipe_comm_info(upipe_ctx_t ctx, upipe_comm_info_t* info);

/* ---------------------------------------------------------------- planning (host only, no GPU) */

/* Bytes of workspace one call needs, 256-byte aligned. pass 0: forward, 1: backward, for the
 * default schedule (C > 1: the next stage's all-to-all overlaps the current attention on the
 * ctx's comm stream, which needs a second chunk buffer set, DESIGN A23); pass 2: forward,
 * 3: backward for a ctx created with UPIPE_FLAG_SYNC_COMM (one buffer set, the paper's
 * memory-minimal schedule). At C = 1 all-to-alls are identities and 0 == 2, 1 == 3.
 * 4 / 5: forward / backward with UPIPE_FLAG_DIRECT (receive buffers only, one set; an IPC ctx holds
 * it in its symmetric region, see upipe_ipc_region_size). Add 8 for a ctx with UPIPE_FLAG_NAIVE_KV (its
 * backward keeps a fp32 dX accumulator instead of the pre-allocated gradient buffer, DESIGN A30). */
UPIPE_API upipe_status_t upipe_workspace_size(int cp_size, const upipe_shape_t* shape, int pass, size_t* bytes);

/* Stage plan of the GQA schedule (A8): for stage s and device p the
 * first local q head (q heads [q0, q0+qpd)), first resident kv head
 * (kv heads [kv0, kv0+kv_res)) and whether the kv heads are sent in this stage. */
typedef struct {
  int32_t n_stages, qpd, kv_res, sigma;
  int32_t q0, kv0, kv_sent;
} upipe_stage_info_t;
UPIPE_API upipe_status_t upipe_plan_stage(int cp_size, const upipe_shape_t* shape, int stage, int device,
                                upipe_stage_info_t* out);
/* Explain the first violated precondition of (cp_size, shape) into msg (may be NULL). */
UPIPE_API upipe_status_t upipe_validate(int cp_size, const upipe_shape_t* shape, char* msg, size_t msg_len);

/* ---------------------------------------------------------------- the layer */

/* Forward.
 *  x         [S_l, D]      bf16  this rank's sequence shard
 *  wq        [Hq*d, D]     bf16  wk, wv [Hkv*d, D]; wo [D, Hq*d]  (replicated on every rank)
 *  y         [S_l, D]      bf16  out
 *  o_saved   [S_l, Hq*d]   bf16  out: attention output before Wo (saved for backward)
 *  lse_saved [Hq/C, S]     fp32  out: natural-log LSE of this rank's heads, slot s*qpd + j
 *                                for local head j of stage s (A12, A17). Ring hybrid (r > 1):
 *                                [Hq/a, S_b] over the rank's ring block (same element count)
 *  workspace: >= upipe_workspace_size(C, shape, 0) bytes, 256-byte aligned. */
UPIPE_API upipe_status_t upipe_attn_fwd(upipe_ctx_t ctx, const upipe_shape_t* shape, const upipe_bf16* x, const upipe_bf16* wq,
                              const upipe_bf16* wk, const upipe_bf16* wv, const upipe_bf16* wo, upipe_bf16* y,
                              upipe_bf16* o_saved, float* lse_saved, void* workspace, size_t ws_bytes,
                              void* stream);

/* Backward, recomputing the stage projections (A12).
 *  dy                 [S_l, D] bf16 cotangent of y
 *  o_saved, lse_saved as produced by upipe_attn_fwd
 *  dx                 [S_l, D] bf16 out
 *  dwq dwk dwv dwo    fp32 out, weight shapes; if reduce_dw != 0 they are summed over
 *                     all C ranks (the FSDP reduction of P:437, A14), else this rank's part.
 *  workspace: >= upipe_workspace_size(C, shape, 1) bytes. */
UPIPE_API upipe_status_t upipe_attn_bwd(upipe_ctx_t ctx, const upipe_shape_t* shape, const upipe_bf16* x, const upipe_bf16* wq,
                              const upipe_bf16* wk, const upipe_bf16* wv, const upipe_bf16* wo,
                              const upipe_bf16* dy, const upipe_bf16* o_saved, const float* lse_saved,
                              upipe_bf16* dx, float* dwq, float* dwk, float* dwv, float* dwo, int reduce_dw,
                              void* workspace, size_t ws_bytes, void* stream);

/* Qwen3 q/k norm weights and their gradients (shape.qk_norm_eps > 0).
 *  q_norm_w, k_norm_w   [d] bf16 in (replicated on every rank)
 *  dq_norm_w, dk_norm_w [d] fp32 out of upipe_attn_bwd_ex: sum over this rank's heads and all S tokens,
 *                       summed over the CP group too when reduce_dw != 0 (ignored by the forward). */
typedef struct {
  const upipe_bf16* q_norm_w;
  const upipe_bf16* k_norm_w;
  float* dq_norm_w;
  float* dk_norm_w;
} upipe_qk_norm_t;

/* upipe_attn_fwd / upipe_attn_bwd with the Qwen3 q/k norm weights (qkn may be NULL when
 * shape->qk_norm_eps == 0; the plain entry points are these with qkn = NULL). */
UPIPE_API upipe_status_t upipe_attn_fwd_ex(upipe_ctx_t ctx, const upipe_shape_t* shape, const upipe_bf16* x,
                              const upipe_bf16* wq, const upipe_bf16* wk, const upipe_bf16* wv, const upipe_bf16* wo,
                              const upipe_qk_norm_t* qkn, upipe_bf16* y, upipe_bf16* o_saved, float* lse_saved,
                              void* workspace, size_t ws_bytes, void* stream);
UPIPE_API upipe_status_t upipe_attn_bwd_ex(upipe_ctx_t ctx, const upipe_shape_t* shape, const upipe_bf16* x,
                              const upipe_bf16* wq, const upipe_bf16* wk, const upipe_bf16* wv, const upipe_bf16* wo,
                              const upipe_qk_norm_t* qkn, const upipe_bf16* dy, const upipe_bf16* o_saved,
                              const float* lse_saved, upipe_bf16* dx, float* dwq, float* dwk, float* dwv, float* dwo,
                              int reduce_dw, void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- kernel-level entry points
 * The individual steps of the hot path, exposed for per-kernel parity tests and
 * roofline measurement. Same kernels the layer calls use. */

/* Attention core (F3): q [S][nq][d] (token stride ldq), k/v [S][nkv][d] (stride ldkv),
 * o at o + t*ldo + j*d, lse [nq][S] (stride ld_lse). */
UPIPE_API upipe_status_t upipe_attn_core_fwd(const upipe_bf16* q, const upipe_bf16* k, const upipe_bf16* v, upipe_bf16* o,
                                   float* lse, int64_t S, int nq, int nkv, int d, int causal, int64_t ldq,
                                   int64_t ldkv, int64_t ldo, int64_t ld_lse, void* stream);
/* Attention core backward (B4): dq_acc fp32 is ACCUMULATED into (zero it first) with dQ = (1/sqrt(d)) dS K;
 * layout [S][nq][d] (token-major), or with UPIPE_CORE_DQ_DIM_MAJOR [nq*d][S4]
 * (dims-major, row stride S4 = S rounded up to a multiple of 4 floats (TMA strides are 16-byte
 * multiples): the layer's layout for the 64-query kernel at d = 128);
 * dk_acc/dv_acc fp32 [S][nkv][d] are written (UPIPE_CORE_ACCUMULATE: added to their contents);
 * delta [S][nq] (stride ld_delta) = rowsum(dO*O) in fp32.
 * flags: UPIPE_CORE_ACCUMULATE | UPIPE_CORE_DQ_DIM_MAJOR (d = 128 only) | UPIPE_CORE_DETERMINISTIC
 * (dQ partials of the key tiles are added in key-tile order, so results are bitwise reproducible;
 * needs dq_sem: >= upipe_core_bwd_sem_count(S, nq) int32 of device memory, zeroed before the call;
 * may be NULL otherwise). */
#define UPIPE_CORE_ACCUMULATE 1
#define UPIPE_CORE_DQ_DIM_MAJOR 2
#define UPIPE_CORE_DETERMINISTIC 4
UPIPE_API upipe_status_t upipe_attn_core_bwd(const upipe_bf16* q, const upipe_bf16* k, const upipe_bf16* v,
                                   const upipe_bf16* dout, const float* lse, const float* delta, float* dq_acc,
                                   float* dk_acc, float* dv_acc, int64_t S, int nq, int nkv, int d, int causal,
                                   int64_t ldq, int64_t ldkv, int64_t ldo_grad, int64_t ld_lse, int64_t ld_delta,
                                   int flags, int32_t* dq_sem, void* stream);
/* Number of int32 semaphores the deterministic backward needs for (S, nq). */
UPIPE_API int64_t upipe_core_bwd_sem_count(int64_t S, int nq);
/* delta[t*ld_delta + j] = sum_e dO[t*ld_do + j*d + e] * O[t*ld_o + j*d + e] */
UPIPE_API upipe_status_t upipe_rowdot(const upipe_bf16* dO, int64_t ld_do, const upipe_bf16* O, int64_t ld_o, float* delta,
                            int64_t ld_delta, int64_t rows, int nheads, int d, void* stream);
/* Plain projection GEMM on the tcgen05 kernel: y[M,N] = x[M,K] w[N,K]^T, bf16 out
 * (mode 0) or fp32 out (mode 1). */
UPIPE_API upipe_status_t upipe_gemm_xwT(const upipe_bf16* x, const upipe_bf16* w, void* y, int64_t M, int64_t N, int64_t K,
                              int mode, void* stream);
/* Device copy of the seeded synthetic input generator (synth/__init__.py):
 * dst[i] = (2*m-255)/256 * 2^exponent, m = splitmix64(seed*G1 + tensor_id*G2 + start + i) >> 56. */
UPIPE_API upipe_status_t upipe_synth_fill_bf16(upipe_bf16* dst, int64_t n, uint64_t seed, int tensor_id, int exponent,
                                     int64_t start, void* stream);

/* ---------------------------------------------------------------- test-only layout probes
 * Not part of the public API (SURVEY §8b "test-only"). They make the integer permutations of the
 * hot path observable through the REAL layer code (projection epilogue -> transport -> receive
 * buffers, attention-output injection -> out all-to-all -> unpack into o_saved) so tests can check
 * them bit-exactly against the oracle's maps (§3.1 layout; SPEC S:150-152 round trip).
 * While a probe is set on a ctx, every upipe_attn_fwd / upipe_attn_bwd call of that ctx:
 *   - after the stage's inp all-to-all, copies the receive buffers of stage `stage` into the non-null
 *     outputs (q_recv [S][qpd*d], k_recv / v_recv [S][kv_res*d] when the stage sends K/V; in backward
 *     also do_recv [S][qpd*d] bf16 and delta_recv [S][qpd] fp32), S = tokens of the Ulysses group;
 *   - forward, o_head != NULL: SKIPS the stage's attention and uses o_head [S][qpd*d] (head layout,
 *     this device's heads) as its output, which then goes through the out all-to-all and the unpack
 *     into o_saved (lse of that stage is not written);
 *   - backward, dq_head != NULL: SKIPS the stage's attention backward and dQ conversion and sends
 *     dq_head [S][qpd*d] (and dk_head / dv_head [S][kv_res*d] at the stage that retires its K/V heads)
 *     head -> seq; dq_recv [C][S_l][qpd*d] (dk_recv / dv_recv [C][S_l][kv_res*d]) receive copies.
 * All pointers are device pointers owned by the caller; stage = -1 turns the probe off. The copies
 * are enqueued on the stream the probed step runs on; they are complete when the call's stream is. */
typedef struct {
  int32_t stage;
  upipe_bf16 *q_recv, *k_recv, *v_recv;
  const upipe_bf16* o_head;
  upipe_bf16* do_recv;
  float* delta_recv;
  const upipe_bf16 *dq_head, *dk_head, *dv_head;
  upipe_bf16 *dq_recv, *dk_recv, *dv_recv;
} upipe_probe_t;
UPIPE_API upipe_status_t upipe_test_set_probe(upipe_ctx_t ctx, const upipe_probe_t* probe);

/* ---------------------------------------------------------------- instrumentation */

/* Kernel-launch counter: number of CUDA kernels this library has launched in the
 * process so far (all contexts, including kernel-level entry points). */
UPIPE_API upipe_status_t upipe_kernel_launches(uint64_t* count);

/* Per-category device timing of the layer calls of one ctx. When tracing is on,
 * every step of upipe_attn_fwd/bwd is bracketed by CUDA events recorded on the
 * call's stream (the stream the kernels run on). upipe_trace_read waits for those
 * events, returns accumulated milliseconds and counts per category since the last
 * read, and clears them. Categories: */
#define UPIPE_TRACE_GEMM 0      /* projection / output / gradient GEMMs (tcgen05) */
#define UPIPE_TRACE_ATTN_FWD 1  /* attention forward kernel */
#define UPIPE_TRACE_ATTN_BWD 2  /* attention backward kernel */
#define UPIPE_TRACE_COMM 3      /* all-to-alls and the dW all-reduce */
#define UPIPE_TRACE_AUX 4       /* rowdot, dQ convert, unpack, memsets */
#define UPIPE_TRACE_NCAT 5
UPIPE_API upipe_status_t upipe_set_trace(upipe_ctx_t ctx, int on);
UPIPE_API upipe_status_t upipe_trace_read(upipe_ctx_t ctx, double ms[UPIPE_TRACE_NCAT], int64_t count[UPIPE_TRACE_NCAT]);

#ifdef __cplusplus
}
#endif
#endif /* UPIPE_H_ */
