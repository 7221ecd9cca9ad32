// Causal GQA flash-attention backward for sm_100a (Table 4).
//
// KV-stationary: one CTA owns a 128-key tile of one KV head and loops over the
// query tiles (of every local query head of that KV group) that can see it.
// Per query tile, five tcgen05 MMAs (M=128, K=128 or d):
//   S^T  = K Q^T          (TMEM cols [0,128))      P^T  = exp2(S^T*c - lse2) -> bf16, back into TMEM
//   dP^T = V dO^T         (TMEM cols [128,256))    dS^T = P^T (dP^T - delta) -> bf16, smem
//   dV  += P^T dO         (TMEM [256, 256+d))      A operand P^T read from TMEM (TS form)
//   dK  += dS^T Q         (TMEM [256+d, 256+2d))
//   dQ   = dS K           (TMEM cols [128,128+d), reusing dP^T once consumed)
// P^T lives in the S^T columns it was computed from (two bf16 per 32-bit column),
// which frees the shared memory for double-buffered Q / dO tiles: the TMA loads of
// tile n+1 overlap the MMAs of tile n.
// dQ is reduced across KV tiles in HBM by TMA bulk reduce-add (fp32): the compute
// warps drain it TMEM -> shared memory (the dS^T buffer, free once the dQ MMA has
// completed) and one thread per warpgroup issues cp.reduce.async.bulk.tensor.
// dK/dV stay in TMEM for the whole CTA and are written (and optionally accumulated
// across the UPipe stages of one super-stage) at the end.
// Warps: 0-7 compute (two warpgroups splitting the 128 query columns; thread =
// one key row for S^T/dP^T, one query row for the dQ drain), 8 TMA producer,
// 9 MMA issuer.
#include <cstdio>

#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace upipe {
namespace {

using namespace dev;

struct BwdArgs {
  const float* lse;
  const float* delta;
  float* dk_acc;
  float* dv_acc;
  __nv_bfloat16* dk_bf16;
  __nv_bfloat16* dv_bf16;
  long long S, ld_lse, ld_delta, ld_kvb;
  int nq, nkv, causal, kv_accumulate, kv_write_acc;
  float scale;       // 1/sqrt(d)
  float scale_log2;  // log2(e)/sqrt(d)
};

__device__ __forceinline__ float ex2b(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int D>
struct BwdCfg {
  static constexpr int TB = 128 * D * 2;   // one 128 x D bf16 tile
  static constexpr int PB = 128 * 128 * 2; // 128 x 128 bf16
  static constexpr int OFF_K = 0, OFF_V = TB, OFF_Q = 2 * TB, OFF_DO = 4 * TB;  // Q, dO: 2 buffers each
  static constexpr int OFF_DS = 6 * TB;
  static constexpr int OFF_BAR = OFF_DS + PB;
  static constexpr int OFF_STAT = OFF_BAR + 256;             // lse2[2][128], delta[2][128] fp32
  static constexpr int SMEM = OFF_STAT + 2048;                // base is 1024-aligned (checked in-kernel)
  static constexpr uint32_t TM_S = 0, TM_DP = 128, TM_DQ = 128, TM_DV = 256, TM_DK = 256 + D;
  static constexpr int DQ_BOXES = D / 64;  // 32-float boxes of dQ per warpgroup (each drains D/2 columns)
};

template <int D>
__global__ void __launch_bounds__(320, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                    const __grid_constant__ CUtensorMap tmdQ, const BwdArgs a) {
  using C = BwdCfg<D>;
  constexpr int NCH = D / 64;
  extern __shared__ __align__(1024) uint8_t smem[];
  if (smem_u32(smem) & 1023) __trap();               // 128B-swizzle atoms need 1024-byte alignment
  float (*s_lse2)[128] = reinterpret_cast<float (*)[128]>(smem + C::OFF_STAT);
  float (*s_delta)[128] = reinterpret_cast<float (*)[128]>(smem + C::OFF_STAT + 1024);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* kv_full = bars + 0;
  uint64_t* q_full = bars + 1;     // [2]
  uint64_t* q_empty = bars + 3;    // [2]
  uint64_t* do_full = bars + 5;    // [2]
  uint64_t* do_empty = bars + 7;   // [2]
  uint64_t* sdp_full = bars + 9;
  uint64_t* ds_full = bars + 10;
  uint64_t* dq_full = bars + 11;
  uint64_t* dq_empty = bars + 12;
  uint64_t* dkv_full = bars + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int warp = warp_id(), lane = lane_id();
  const int jb = blockIdx.x;                      // key tile (small jb = most query tiles = longest)
  const int g = blockIdx.y;                       // kv head
  const int G = a.nq / a.nkv;
  const int nT = (int)((a.S + 127) / 128);
  const int qt_begin = a.causal ? jb : 0;
  const int n_qt = nT - qt_begin;
  const int N = G * n_qt;                         // (head, query tile) iterations

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV); tma_prefetch(&tmdO); tma_prefetch(&tmdQ);
    for (int i = 0; i < 14; ++i) mbar_init(&bars[i], (i == 10 || i == 12) ? 256 : 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      mbar_arrive_expect_tx(kv_full, 2 * C::TB);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        tma_load_3d(smem + C::OFF_K + c * 16384, &tmK, kv_full, c * 64, g, jb * 128);
        tma_load_3d(smem + C::OFF_V + c * 16384, &tmV, kv_full, c * 64, g, jb * 128);
      }
      for (int n = 0; n < N; ++n) {
        const int h = g * G + n / n_qt;
        const int qt = qt_begin + n % n_qt;
        const int b = n & 1;
        const uint32_t ph = ((n >> 1) & 1) ^ 1;
        mbar_wait(&q_empty[b], ph);
        mbar_arrive_expect_tx(&q_full[b], C::TB);
#pragma unroll
        for (int c = 0; c < NCH; ++c)
          tma_load_3d(smem + C::OFF_Q + b * C::TB + c * 16384, &tmQ, &q_full[b], c * 64, h, qt * 128);
        mbar_wait(&do_empty[b], ph);
        mbar_arrive_expect_tx(&do_full[b], C::TB);
#pragma unroll
        for (int c = 0; c < NCH; ++c)
          tma_load_3d(smem + C::OFF_DO + b * C::TB + c * 16384, &tmdO, &do_full[b], c * 64, h, qt * 128);
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer
      constexpr uint32_t id_kk = idesc_bf16(128, 128, false, false);  // S^T, dP^T: both K-major over d
      constexpr uint32_t id_kmn = idesc_bf16(128, D, false, true);    // dV (A in TMEM), dK: B MN-major
      constexpr uint32_t id_mnmn = idesc_bf16(128, D, true, true);    // dQ: A = dS^T viewed MN-major, B = K MN-major
      const uint32_t sK = smem_u32(smem + C::OFF_K), sV = smem_u32(smem + C::OFF_V);
      const uint32_t sQ0 = smem_u32(smem + C::OFF_Q), sdO0 = smem_u32(smem + C::OFF_DO);
      const uint32_t sdS = smem_u32(smem + C::OFF_DS);
      auto mma_kk = [&](uint32_t sa, uint32_t sb, uint32_t tm) {      // [128 x D] x [128 x D]^T
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ss(tm, desc_sw128(sa + c * 16384 + kk * 32, 16, 1024), desc_sw128(sb + c * 16384 + kk * 32, 16, 1024),
                   id_kk, (c | kk) != 0);
      };
      auto mma_kmn = [&](uint32_t sa, uint32_t sb, uint32_t tm, bool acc) {  // A [128 x 128 q] K-major smem
#pragma unroll
        for (int kb = 0; kb < 2; ++kb)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ss(tm, desc_sw128(sa + kb * 16384 + kk * 32, 16, 1024),
                   desc_sw128(sb + kb * 8192 + kk * 2048, 16384, 1024), id_kmn, (acc || kb || kk) ? 1u : 0u);
      };
      auto mma_tmn = [&](uint32_t ta, uint32_t sb, uint32_t tm, bool acc) {  // A = P^T in TMEM (q 0-63 at +0, 64-127 at +64)
#pragma unroll
        for (int kb = 0; kb < 2; ++kb)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ts(tm, ta + kb * 64 + kk * 8, desc_sw128(sb + kb * 8192 + kk * 2048, 16384, 1024), id_kmn,
                   (acc || kb || kk) ? 1u : 0u);
      };
      auto mma_mnmn = [&](uint32_t sa, uint32_t sb, uint32_t tm) {  // dQ = dS K: K dim = keys (rows of both)
#pragma unroll
        for (int kb = 0; kb < 2; ++kb)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ss(tm, desc_sw128(sa + kb * 8192 + kk * 2048, 16384, 1024),
                   desc_sw128(sb + kb * 8192 + kk * 2048, 16384, 1024), id_mnmn, (kb | kk) != 0);
      };
      mbar_wait(kv_full, 0);
      mbar_wait(&q_full[0], 0);
      tc_fence_after();
      mma_kk(sK, sQ0, tmem + C::TM_S);
      mbar_wait(&do_full[0], 0);
      tc_fence_after();
      mma_kk(sV, sdO0, tmem + C::TM_DP);
      mma_commit(sdp_full);
      for (int n = 0; n < N; ++n) {
        const int b = n & 1;
        const uint32_t sQ = sQ0 + b * C::TB, sdO = sdO0 + b * C::TB;
        mbar_wait(ds_full, n & 1);
        tc_fence_after();
        mma_tmn(tmem + C::TM_S, sdO, tmem + C::TM_DV, n > 0);
        mma_commit(&do_empty[b]);
        mma_kmn(sdS, sQ, tmem + C::TM_DK, n > 0);
        mma_commit(&q_empty[b]);
        mma_mnmn(sdS, sK, tmem + C::TM_DQ);
        mma_commit(dq_full);
        if (n + 1 < N) {
          const int b1 = (n + 1) & 1;
          const uint32_t ph1 = ((n + 1) >> 1) & 1;
          mbar_wait(&q_full[b1], ph1);
          tc_fence_after();
          mma_kk(sK, sQ0 + b1 * C::TB, tmem + C::TM_S);   // in-order after dV(n), which reads P^T from these columns
          mbar_wait(dq_empty, n & 1);
          mbar_wait(&do_full[b1], ph1);
          tc_fence_after();
          mma_kk(sV, sdO0 + b1 * C::TB, tmem + C::TM_DP);
          mma_commit(sdp_full);
        }
      }
      mma_commit(dkv_full);
    }
  } else {
    // ------------------------------------------------ compute warpgroups (warps 0-7)
    const int wg = warp >> 2;                         // query columns [64 wg, 64 wg + 64) ; dQ cols [wg D/2, ...)
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const long long key = (long long)jb * 128 + r;
    const float sl2 = a.scale_log2;
    const bool issuer = (warp & 3) == 0 && lane == 0;
    uint8_t* staging = smem + C::OFF_DS + wg * 16384;  // this warpgroup's half of dS^T, free after the dQ MMA
    const uint32_t dsbase = smem_u32(smem + C::OFF_DS);
    for (int n = 0; n < N; ++n) {
      const int h = g * G + n / n_qt;
      const int qt = qt_begin + n % n_qt;
      const long long q0 = (long long)qt * 128;
      const int sb = n & 1;
      {
        const long long q = q0 + r;
        if (wg == 0) s_lse2[sb][r] = q < a.S ? a.lse[(long long)h * a.ld_lse + q] * 1.4426950408889634f : 0.f;
        else s_delta[sb][r] = q < a.S ? a.delta[q * a.ld_delta + h] : 0.f;
      }
      if (issuer) bulk_wait_read0();                  // previous dQ reduce has finished reading dS^T smem
      named_bar_sync(1, 256);
      mbar_wait(sdp_full, n & 1);
      tc_fence_after();
      const bool diag = a.causal && qt == jb;
      const bool tail = q0 + 128 > a.S || (long long)jb * 128 + 128 > a.S;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int col0 = wg * 64 + c * 32;
        uint32_t rs[32], rp[32];
        tmem_ld32(tmem + C::TM_S + lane_off + col0, rs);
        tmem_ld32(tmem + C::TM_DP + lane_off + col0, rp);
        tmem_wait_ld();
        float p[32], ds[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int qi = col0 + i;
          float pv = ex2b(__uint_as_float(rs[i]) * sl2 - s_lse2[sb][qi]);
          if (diag || tail) {
            const long long q = q0 + qi;
            if ((a.causal && key > q) || q >= a.S || key >= a.S) pv = 0.f;
          }
          p[i] = pv;
          ds[i] = pv * (__uint_as_float(rp[i]) - s_delta[sb][qi]);
        }
        // P^T (bf16 pairs) back into the S^T columns already read: q [col0, col0+32) -> cols wg*64 + c*16 + [0,16)
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(p[2 * i], p[2 * i + 1]);
        tmem_st16(tmem + C::TM_S + lane_off + wg * 64 + c * 16, pk);
#pragma unroll
        for (int v8 = 0; v8 < 4; ++v8) {
          const int qc = col0 + v8 * 8;
          const uint32_t off = (qc >> 6) * 16384 + sw128_offset(r, qc & 63);
          st_shared_v4(dsbase + off, pack_bf16(ds[v8 * 8 + 0], ds[v8 * 8 + 1]),
                       pack_bf16(ds[v8 * 8 + 2], ds[v8 * 8 + 3]), pack_bf16(ds[v8 * 8 + 4], ds[v8 * 8 + 5]),
                       pack_bf16(ds[v8 * 8 + 6], ds[v8 * 8 + 7]));
        }
      }
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(ds_full);
      // ---- dQ drain: TMEM lane = query row; this warpgroup takes dQ columns [wg D/2, (wg+1) D/2)
      mbar_wait(dq_full, n & 1);
      tc_fence_after();
      uint32_t rq[C::DQ_BOXES][32];
#pragma unroll
      for (int b = 0; b < C::DQ_BOXES; ++b) tmem_ld32(tmem + C::TM_DQ + lane_off + wg * (D / 2) + b * 32, rq[b]);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(dq_empty);
      const uint32_t stbase = smem_u32(staging);
#pragma unroll
      for (int b = 0; b < C::DQ_BOXES; ++b) {
        if (b > 0) {                      // staging holds one 32-column box: wait for the previous reduce to read it
          if (issuer) bulk_wait_read0();
          named_bar_sync(2 + wg, 128);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {     // 16-byte chunk j of the 128-byte row, swizzled by row % 8
          const uint32_t addr = stbase + r * 128 + ((j ^ (r & 7)) << 4);
          st_shared_v4(addr, __float_as_uint(__uint_as_float(rq[b][4 * j + 0]) * a.scale),
                       __float_as_uint(__uint_as_float(rq[b][4 * j + 1]) * a.scale),
                       __float_as_uint(__uint_as_float(rq[b][4 * j + 2]) * a.scale),
                       __float_as_uint(__uint_as_float(rq[b][4 * j + 3]) * a.scale));
        }
        fence_proxy_async_smem();
        named_bar_sync(2 + wg, 128);
        if (issuer) {
          tma_reduce_add_2d(&tmdQ, staging, h * D + wg * (D / 2) + b * 32, (int)q0);
          bulk_commit();
        }
      }
    }
    if (issuer) bulk_wait0();
    // ---- dK / dV epilogue (TMEM lane = key row): warpgroup 0 writes dV, warpgroup 1 writes dK
    mbar_wait(dkv_full, 0);
    tc_fence_after();
    const long long ldacc = (long long)a.nkv * D;
    const int which = wg;
    const uint32_t tcol = which ? C::TM_DK : C::TM_DV;
    const float sc = which ? a.scale : 1.f;
    float* acc = (which ? a.dk_acc : a.dv_acc);
    __nv_bfloat16* ob = which ? a.dk_bf16 : a.dv_bf16;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t rr[32];
      tmem_ld32(tmem + tcol + lane_off + c * 32, rr);
      tmem_wait_ld();
      if (key >= a.S || N == 0) continue;
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(rr[i]) * sc;
      float4* accp = acc ? reinterpret_cast<float4*>(acc + key * ldacc + (long long)g * D + c * 32) : nullptr;
      if (a.kv_accumulate && accp) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 o = accp[i];
          v[4 * i] += o.x; v[4 * i + 1] += o.y; v[4 * i + 2] += o.z; v[4 * i + 3] += o.w;
        }
      }
      if (a.kv_write_acc && accp) {
#pragma unroll
        for (int i = 0; i < 8; ++i) accp[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      }
      if (ob) {
        uint4* dst = reinterpret_cast<uint4*>(ob + key * a.ld_kvb + (long long)g * D + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_uint4(pack_bf16(v[8 * i + 0], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                              pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

cudaError_t attn_bwd_run(const AttnBwdProblem& p, cudaStream_t stream, char* err, size_t errlen) {
  if (p.S <= 0 || p.nkv <= 0) return cudaSuccess;
  if ((p.d != 64 && p.d != 128) || p.nq % p.nkv) {
    snprintf(err, errlen, "attn_bwd: unsupported head_dim %d or head counts %d/%d", p.d, p.nq, p.nkv);
    return cudaErrorInvalidValue;
  }
  CUtensorMap tq, tk, tv, tdo, tdq;
  if (!make_tmap_3d(&tq, p.q, p.d, p.nq, p.S, p.d, p.ldq, 64, 1, 128, err, errlen)) return cudaErrorInvalidValue;
  if (!make_tmap_3d(&tk, p.k, p.d, p.nkv, p.S, p.d, p.ldkv, 64, 1, 128, err, errlen)) return cudaErrorInvalidValue;
  if (!make_tmap_3d(&tv, p.v, p.d, p.nkv, p.S, p.d, p.ldkv, 64, 1, 128, err, errlen)) return cudaErrorInvalidValue;
  if (!make_tmap_3d(&tdo, p.dout, p.d, p.nq, p.S, p.d, p.ldo_grad, 64, 1, 128, err, errlen))
    return cudaErrorInvalidValue;
  // dq_acc fp32 [S][nq*d]: boxes of 32 columns x 128 rows, TMA reduce-add
  if (!make_tmap_2d_f32(&tdq, p.dq_acc, (uint64_t)p.nq * p.d, p.S, (uint64_t)p.nq * p.d, 32, 128, err, errlen))
    return cudaErrorInvalidValue;
  BwdArgs a;
  a.lse = p.lse;
  a.delta = p.delta;
  a.dk_acc = p.dk_acc;
  a.dv_acc = p.dv_acc;
  a.dk_bf16 = reinterpret_cast<__nv_bfloat16*>(p.dk_bf16);
  a.dv_bf16 = reinterpret_cast<__nv_bfloat16*>(p.dv_bf16);
  a.S = p.S;
  a.ld_lse = p.ld_lse;
  a.ld_delta = p.ld_delta;
  a.ld_kvb = p.ld_kvb;
  a.nq = p.nq;
  a.nkv = p.nkv;
  a.causal = p.causal;
  a.kv_accumulate = p.kv_accumulate;
  a.kv_write_acc = p.kv_write_acc;
  a.scale = 1.f / sqrtf((float)p.d);
  a.scale_log2 = 1.4426950408889634f / sqrtf((float)p.d);
  const int nT = (int)((p.S + 127) / 128);
  dim3 grid(nT, p.nkv);
  cudaError_t e;
  if (p.d == 128) {
    static const cudaError_t attr =
        cudaFuncSetAttribute(attn_bwd_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, BwdCfg<128>::SMEM);
    if (attr != cudaSuccess) { snprintf(err, errlen, "attn_bwd attr: %s", cudaGetErrorString(attr)); return attr; }
    attn_bwd_kernel<128><<<grid, 320, BwdCfg<128>::SMEM, stream>>>(tq, tk, tv, tdo, tdq, a);
    count_launches(1);
  } else {
    static const cudaError_t attr =
        cudaFuncSetAttribute(attn_bwd_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, BwdCfg<64>::SMEM);
    if (attr != cudaSuccess) { snprintf(err, errlen, "attn_bwd attr: %s", cudaGetErrorString(attr)); return attr; }
    attn_bwd_kernel<64><<<grid, 320, BwdCfg<64>::SMEM, stream>>>(tq, tk, tv, tdo, tdq, a);
    count_launches(1);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) snprintf(err, errlen, "attn_bwd launch: %s", cudaGetErrorString(e));
  return e;
}

}  // namespace upipe
