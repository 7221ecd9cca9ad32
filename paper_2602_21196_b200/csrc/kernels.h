// Internal launcher declarations (host side). Not part of the C ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace upipe {

// process-wide kernel launch counter (upipe_kernel_launches)
void count_launches(uint64_t n);

// ---------------------------------------------------------------- GEMM
// D[m, n] = alpha * sum_k A(m, k) * B(n, k)   (bf16 in, fp32 accumulate in TMEM)
//
// Every operand is a 2-D row-major bf16 tensor in HBM addressed through a TMA map
// (inner dim contiguous). "K-major": the operand's K index runs along the inner
// dim; "MN-major": its M (or N) index does. Operands may be gathered in 64-element
// granules: for a logical outer index i and K index k,
//   outer_coord = o_base + (i / o_len) * o_istride + i % o_len + (k / k_len) * o_kstride
//   k_coord     = k_base + (k / k_len) * k_kstride + k % k_len + (i / o_len) * k_istride
// (o_len, k_len multiples of 64). This is how the per-stage head gather of the
// UPipe schedule (weights rows / columns of the stage's heads, the a2a buffers laid
// out [C][S_l][...]) is expressed without any copy.
struct OperandMap {
  const void* ptr = nullptr;
  int64_t inner = 0, outer = 0;  // tensor extents (elements): inner = contiguous dim
  int64_t ld = 0;                // row stride in elements
  bool mn_major = false;         // false: K along inner ; true: M/N along inner
  int64_t o_base = 0, o_len = 1 << 30, o_istride = 0, o_kstride = 0;
  int64_t k_base = 0, k_len = 1 << 30, k_kstride = 0, k_istride = 0;
};

// Output element (m, n) goes to
//   row = r_base + (m / m_len) * r_mstride + m % m_len + (n / n_len) * r_nstride
//   col = c_base + (n / n_len) * c_nstride + n % n_len + (m / m_len) * c_mstride
enum class Epi : int {
  kStoreBF16 = 0,     // out_bf16 = bf16(acc)
  kStoreF32 = 1,      // out_f32 = acc
  kAccF32 = 2,        // out_f32 += acc
  kAccF32ToBF16 = 3,  // out_bf16 = bf16(out_f32 + acc)   (last accumulation step)
};
// RoPE rotation tables (DESIGN A26), built once per (base, d, S) by the library in double precision:
//   hi[h][i] = (cos, sin)(h * 1024 * f_i mod 2pi),  lo[l][i] = (cos, sin)(l * f_i),  f_i = base^(-2i/d),
// so the angle of position p = 1024 h + l is composed exactly by one complex product (fp32 tables;
// an fp32 angle p * f_i would lose ~0.1 rad at p ~ 1e6).
struct RopeRef {
  const float2* hi = nullptr;   // null: no rotation
  const float2* lo = nullptr;
  int d = 0;                    // head_dim; pair index i = (column % d) / 2
  int64_t pos0 = 0;             // position of row 0
};

// Direct-to-peer destinations: a producer kernel writes block `seg` of its output
// straight into the receive buffer of the rank that owns it (a CUDA-IPC mapping of that rank's
// symmetric workspace) instead of into a local send buffer. kMaxSeg bounds the group (one box: 8 GPUs).
constexpr int kMaxSeg = 16;   // C <= 8 ranks x up to 2 N-concatenated outputs (K | V)
struct SegPtrs {
  void* p[kMaxSeg] = {};        // base of segment 0..n-1 (n = 0: not segmented)
  int n = 0;
  int64_t rows = 0;             // row-segmented outputs (attention O, dQ/dK/dV): rows per segment (S_l)
};

// Fused delta = rowsum(bf16(out) * O) per (row, head) in the bf16 store epilogue of the dO projection
// (DESIGN A13): the epilogue thread of row m holds the stored (bf16-rounded) dO values of
// its columns and reads the matching O columns of o_saved, so dO is never re-read from HBM.
//   output column n = (seg, nin) (seg = n / n_len) <-> O column col0 + seg * col_stride + nin of row m;
//   delta of (m, head nin / d) -> dst(seg)[m * ld_dst + nin / d], dst(seg) = dst[seg] if dst_stride == 0
//   else dst[0] + seg * dst_stride. Needs head-aligned tiles (the GEMM checks BN % d == 0).
struct RowDot {
  const void* o = nullptr;
  int64_t ld_o = 0, col0 = 0, col_stride = 0;
  float* dst[kMaxSeg] = {};
  int64_t dst_stride = 0;
  int ld_dst = 0, d = 0;
};

struct OutMap {
  void* out_f32 = nullptr;
  void* out_bf16 = nullptr;
  int64_t ld_f32 = 0, ld_bf16 = 0;
  int64_t r_base = 0, m_len = 1 << 30, r_mstride = 0, r_nstride = 0;
  int64_t c_base = 0, n_len = 1 << 30, c_nstride = 0, c_mstride = 0;
  Epi epi = Epi::kStoreBF16;
  RopeRef rope;                 // kStoreBF16 only: rotate column pairs by the row's position first
  // kStoreBF16, N2: column segment n / n_len goes to seg.p[n / n_len] + m * ld_bf16 + n % n_len (a peer's
  // receive block; replaces out_bf16 / r_nstride). Part 0 of a single (non-grouped) GEMM only.
  SegPtrs seg;
  RowDot dot;                   // part 0 of a single GEMM, kStoreBF16: fused row-dot (dot.o non-null)
  // kStoreF32: the caller zeroed the output, so the GEMM may split K across units that ADD their partial
  // products (atomically) -- used for the weight gradients, whose M x N tile count is below the SM count
  bool zeroed = false;
};

struct GemmProblem {
  int64_t M = 0, N = 0, K = 0;
  float alpha = 1.0f;
  OperandMap a, b;
  OutMap c;
};

cudaError_t gemm_run(const GemmProblem& p, cudaStream_t stream, char* err, size_t errlen);

// Grouped launches (one kernel, up to 3 parts):
//  kKConcat: C = sum_i A_i B_i^T  (equal M and N; each K_i a multiple of 64; output map of part 0)
//            e.g. dX = dQ Wq + dK Wk + dV Wv with one fp32 read-modify-write of dX;
//  kMConcat: rows of part i = A_i B^T (equal N and K; each M_i but the last a multiple of 128;
//            B operand of part 0; own output map per part), e.g. [dWq; dWk; dWv] = [dQ; dK; dV]^T X.
//  kNConcat: columns of part i = A B_i^T (equal M and K, one A operand: part 0's; each N_i a multiple of the
//            tile width; bf16 store outputs addressed as one segmented output: the parts' n_len-column
//            segments in order, e.g. [K | V] = X [Wk; Wv]^T into the K and V send (or peer receive) buffers).
enum class GemmGroup : int { kKConcat = 0, kMConcat = 1, kNConcat = 2 };
cudaError_t gemm_run_group(const GemmProblem* parts, int n, GemmGroup kind, cudaStream_t stream, char* err,
                           size_t errlen);

// ---------------------------------------------------------------- attention
// Causal GQA flash attention over the full sequence for the heads local to this
// device in one stage (head layout after the inp all-to-all).
//   q   [S][nq][d] bf16 (token-major, heads contiguous per token: row stride ldq elems)
//   k,v [S][nkv][d] bf16 (row stride ldkv)
//   o   [S][nq][d] bf16 written at o + t*ldo + j*d
//   lse [nq][S] fp32 natural-log log-sum-exp at lse + j*ld_lse + t
// q head j uses kv head kv_of_q(j) = j / (nq / nkv).
struct AttnFwdProblem {
  const void* q; const void* k; const void* v;
  void* o; float* lse;
  int64_t S; int nq, nkv, d; int causal;
  int64_t ldq, ldkv, ldo, ld_lse;
  float* o32 = nullptr;        // non-null: O in fp32 at o32 + t*ldo32 + j*d instead of bf16 (ring partials)
  int64_t ldo32 = 0;
  SegPtrs o_seg;               // N2 (n > 0): row t of O goes to o_seg.p[t / rows] + (t % rows)*ldo + j*d
};
cudaError_t attn_fwd_run(const AttnFwdProblem& p, cudaStream_t stream, char* err, size_t errlen);

// Backward: dq_acc fp32 [S][nq][d] (+= scale*dS K; must be zeroed by caller unless accumulate),
// dk/dv: fp32 accumulators [S][nkv][d] (kv_mode: 0 store, 1 accumulate) and/or bf16 output
// (kv_bf16 != null: write bf16(acc_prev + new) at kv_bf16 + t*ld_kvb + g*d).
struct AttnBwdProblem {
  const void* q; const void* k; const void* v; const void* dout;
  const float* lse; const float* delta;       // [nq][S] (ld_lse), delta = rowsum(dO*O) [S][nq] (ld_delta)
  float* dq_acc;                              // [S][nq][d]
  float* dk_acc; float* dv_acc;               // [S][nkv][d]
  void* dk_bf16; void* dv_bf16;               // optional bf16 outputs [S][nkv][d] row stride ld_kvb
  int64_t S; int nq, nkv, d; int causal;
  int64_t ldq, ldkv, ldo_grad, ld_lse, ld_delta, ld_kvb;
  int kv_accumulate;                          // 1: add the previous dk_acc/dv_acc contents
  int kv_write_acc;                           // 1: write fp32 accumulators back
  RopeRef rope;                               // dk_bf16 is rotated back by -angle(key) (RoPE on K)
  int dq_dim_major = 0;                       // 1 (only where attn_bwd_dq_dim_major() allows): dq_acc is
  int64_t ld_dqt = 0;                         //   [nq*d][S] fp32, row stride ld_dqt (tokens contiguous)
  int* dq_sem = nullptr;                      // non-null: deterministic dQ order (attn_bwd_sem_count ints, zeroed)
  SegPtrs dk_seg, dv_seg;                     // N2 (n > 0): bf16 dK / dV row t -> seg.p[t / rows] + (t % rows)*ld_kvb
};
// int32 semaphores the deterministic backward needs: one per (q head, 64-query tile, 32-dim box group).
inline int64_t attn_bwd_sem_count(int64_t S, int nq) { return (int64_t)nq * ((S + 63) / 64) * 4; }
cudaError_t attn_bwd_run(const AttnBwdProblem& p, cudaStream_t stream, char* err, size_t errlen);
// Whether attn_bwd_run can accumulate dQ dim-major for this problem (the 64-query kernel, whose dQ^T
// tile has one head dimension per TMEM lane, then stages 16-byte vectors instead of transposing).
bool attn_bwd_dq_dim_major(const AttnBwdProblem& p);
// Whether a dim-major dq_acc can be requested at all (the 64-query kernel serves it)
bool attn_bwd_dq_dim_major_supported(const AttnBwdProblem& p);

// ---------------------------------------------------------------- HBM-bound helpers
// delta[t][j] = sum_e dO[t][j*d+e] * O[t][j*d+e] over bf16 inputs, fp32 result.
cudaError_t rowdot_run(const void* dO, int64_t ld_do, const void* O, int64_t ld_o, float* delta, int64_t ld_delta,
                       int64_t rows, int nheads, int d, cudaStream_t s);
// bf16 = bf16(scale * f32) elementwise over a [rows][cols] block with strides.
cudaError_t cvt_f32_bf16_run(const float* src, int64_t lds, void* dst, int64_t ldd, int64_t rows, int64_t cols,
                             float scale, cudaStream_t s, const RopeRef& inverse_rope);
cudaError_t cvt_f32_bf16_run(const float* src, int64_t lds, void* dst, int64_t ldd, int64_t rows, int64_t cols,
                             float scale, cudaStream_t s);
// The same from a dim-major source: dst[t][c] = bf16(scale * src[c][t]) (src row stride lds, tokens
// contiguous), with the inverse RoPE of token rope.pos0 + t on column pairs; cols % 64 == 0.
cudaError_t cvt_dimmajor_f32_bf16_run(const float* src, int64_t lds, void* dst, int64_t ldd, int64_t rows,
                                      int64_t cols, float scale, cudaStream_t s, const RopeRef& inverse_rope,
                                      const SegPtrs* dst_seg = nullptr);
// N2 form of cvt_f32_bf16_run: dst row t -> dst_seg.p[t / dst_seg.rows] + (t % dst_seg.rows) * ldd.
cudaError_t cvt_f32_bf16_seg_run(const float* src, int64_t lds, const SegPtrs& dst_seg, int64_t ldd, int64_t rows,
                                 int64_t cols, float scale, cudaStream_t s, const RopeRef& inverse_rope);
// Ring-step combine (DESIGN A27), per row t and head j of [rows][nheads][d]:
//   lse' = log(e^lse_acc + e^lse_part) (max-subtracted), O' = e^(lse_acc-lse') O_acc + e^(lse_part-lse') O_part,
// O fp32, lse [nheads][ld_lse]; writes o_acc and lse_acc in place.
cudaError_t merge_partials_run(float* o_acc, const float* o_part, int64_t ld_o, float* lse_acc, const float* lse_part,
                               int64_t ld_lse, int64_t rows, int nheads, int d, cudaStream_t s);
// Column scatter: dst[t][col_of(seg)+e] = src[seg][t][e]   (unpack of the out all-to-all)
cudaError_t unpack_cols_run(const void* src, int64_t rows, int nseg, int seg_cols, void* dst, int64_t ldd,
                            int64_t col_base, int64_t col_stride, cudaStream_t s);
// Qwen3 per-head q/k RMSNorm: dst[t][h] = rope(src[t][h] / rms(src[t][h]) * gamma) per (row t,
// head h) of [rows][heads][d] bf16 (row stride ld; dst may alias src); rope.pos0 = position of row 0.
cudaError_t qk_prep_run(const void* src, void* dst, int64_t rows, int heads, int d, int64_t ld, const void* gamma,
                        float eps, const RopeRef& rope, cudaStream_t s);
constexpr int kNormBwdMaxBlocks = 148 * 6;
// Its chain rule fused into the fp32 -> bf16 gradient conversion: g = rope^-1(scale * src) (src row-major
// [rows][heads d] with row stride st, or dim_major [heads d][st]), x = the pre-norm rows (bf16, stride
// ldx); writes bf16 dx to dst (row stride ldd) or dst_seg (N2) and ADDS sum_t g * x_hat into dgamma[d] (fp32).
cudaError_t norm_bwd_run(const float* src, int64_t st, bool dim_major, const void* x, int64_t ldx, void* dst,
                         int64_t ldd, const SegPtrs* dst_seg, int64_t rows, int heads, int d, float scale,
                         const void* gamma, float eps, const RopeRef& inverse_rope, float* dgamma, cudaStream_t s,
                         float* det_partials = nullptr);   // non-null: [kNormBwdMaxBlocks][d] scratch, fixed order
cudaError_t synth_fill_bf16_run(void* dst, int64_t n, uint64_t seed, int tensor_id, int exponent, int64_t start,
                                cudaStream_t s);

}  // namespace upipe
