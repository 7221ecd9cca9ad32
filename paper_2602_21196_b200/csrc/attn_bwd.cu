// Causal GQA flash-attention backward for sm_100a (Table 4).
// Two kernels: attn_bwd_q64_kernel (below the first, d = 128, the default: 64-query tiles in two TMEM
// slots, ping-pong) and attn_bwd_kernel<d> (128-query tiles; d = 64, and d = 128 with UPIPE_BWD_Q64=0),
// described here.
//
// KV-stationary: one CTA owns a 128-key tile of one KV head and loops over the
// query tiles (of every local query head of that KV group) that can see it.
// Per query tile, five tcgen05 MMAs (M=128, K=128 or d):
//   S^T  = K Q^T          (TMEM cols [0,128))      P^T  = exp2(S^T*c - lse2) -> bf16, back into TMEM
//   dP^T = V dO^T         (TMEM cols [128,256))    dS^T = P^T (dP^T - delta) -> bf16, smem
//   dV  += P^T dO         (TMEM [256, 256+d))      A operand P^T read from TMEM (TS form)
//   dK  += dS^T Q         (TMEM [256+d, 256+2d))
//   dQ   = dS K           (TMEM cols [128,128+d), reusing dP^T once consumed)
// P^T lives in the S^T columns it was computed from (two bf16 per 32-bit column).
// dQ is reduced across KV tiles in HBM by TMA bulk reduce-add (fp32): each compute
// warpgroup drains its half of dQ TMEM -> shared memory (32-column boxes) and one
// of its threads issues cp.reduce.async.bulk.tensor; the 1/sqrt(d) scale of dQ is
// applied when the accumulator is converted to bf16.
// Issue order per query tile n: dV(n), dQ(n), S(n+1), dP(n+1), dK(n). The TMEM budget
// (S|dP|dV|dK = 512 columns at d = 128) rules out double-buffering S/dP, so the tile-to-tile
// chain is E(n) -> 4 MMAs -> E(n+1); dK(n) is issued last and overlaps E(n+1) (which only
// waits for it before overwriting dS^T in shared memory), and the dQ(n) drain overlaps
// S(n+1)/dP(n+1).
// dK/dV stay in TMEM for the whole CTA and are written (and optionally accumulated
// across the UPipe stages of one super-stage) at the end.
// Warps: 0-7 compute (two warpgroups, each owning 64 of the 128 query columns of
// S^T/dP^T; thread = one key row there, one query row for the dQ drain), warp 8
// TMA producer, warp 9 MMA issuer. The elementwise math runs on fp32 pairs (FFMA2/FADD2/FMUL2);
// the exponentials take MUFU.EX2 (UPIPE_BWD_MUFU_EVERY selects a polynomial share on the FMA pipe).
#include <cstdio>
#include <cstdlib>

#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace upipe {
namespace {

using namespace dev;

struct BwdArgs {
  float* dq_acc;
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
  RopeRef rope;      // dK (bf16 output) rotated back by -angle(key) when set (RoPE on K, DESIGN A26)
  int dq_dim_major;  // q64 kernel: dq_acc is [nq*d][S] (TMA boxes of 32 dims x 32 tokens)
  int* dq_sem;       // deterministic dQ (UPIPE_FLAG_DETERMINISTIC): per (head, query tile, box group) the
                     // number of key tiles that have added their partial; key tile jb adds when it reads jb
  long long* dbg;    // optional per-role cycle breakdown of CTA (0,0) (UPIPE_BWD_TIMELINE=1)
  // N2 (nkseg / nvseg > 0): bf16 dK / dV row t -> {dk,dv}seg[t / kvseg_rows] + (t % kvseg_rows) * ld_kvb (a
  // peer's receive block) instead of dk_bf16 / dv_bf16
  __nv_bfloat16* dkseg[kMaxSeg];
  __nv_bfloat16* dvseg[kMaxSeg];
  long long kvseg_rows;
  int nkseg, nvseg;
};

// Destination row of the bf16 dK / dV epilogue (plain or N2 segmented); key < S.
__device__ __forceinline__ __nv_bfloat16* kv_out_row(const BwdArgs& a, int which, long long key) {
  if (which ? a.nkseg : a.nvseg) return (which ? a.dkseg : a.dvseg)[key / a.kvseg_rows] + (key % a.kvseg_rows) * a.ld_kvb;
  return (which ? a.dk_bf16 : a.dv_bf16) + key * a.ld_kvb;
}

__device__ __forceinline__ float ex2b(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

#ifndef UPIPE_BWD_MUFU_EVERY
// element pairs j with j % N == 0 take MUFU.EX2, the rest the FMA polynomial (ex2_fma2). Measured at
// S = 32K (profiles/bwd_timeline.py): N = 1 (all MUFU) 5.39-5.44 ms, 2: 5.43, 4: 5.58, 8: 5.65; moving the
// bf16 packs to the ALU pipe (round-half-away PRMT packs) was slower in every combination.
#define UPIPE_BWD_MUFU_EVERY 1
#endif
constexpr int kSoftmaxWarps = 8;                  // two warpgroups: P^T, dS^T (+ dK/dV epilogue)
constexpr int kRegsSoftmax = 144, kRegsDrain = 152, kRegsOther = 72;   // setmaxnreg split of the 64K registers
constexpr int kThreads = (kSoftmaxWarps + 8) * 32;  // + dQ drain warpgroup + {TMA, MMA, 2 idle}
constexpr int kTmaWarp = kSoftmaxWarps + 4, kMmaWarp = kSoftmaxWarps + 5;
static_assert(2 * 128 * kRegsSoftmax + 128 * kRegsDrain + 128 * kRegsOther <= 65536, "register split");

template <int D>
struct BwdCfg {
  static constexpr int TB = 128 * D * 2;   // one 128 x D bf16 tile
  static constexpr int PB = 128 * 128 * 2; // 128 x 128 bf16
  static constexpr int OFF_K = 0, OFF_V = TB, OFF_Q = 2 * TB;   // Q: 2 buffers
  static constexpr int OFF_DO = 4 * TB;
  static constexpr int OFF_DS = 5 * TB;
  static constexpr int OFF_STG = OFF_DS + PB;                    // dQ staging slots 0,1 (16 KB each); 2,3 alias dS^T
  static constexpr int OFF_BAR = OFF_STG + 32768;
  static constexpr int OFF_STAT = OFF_BAR + 256;                 // lse2[2][128], delta[2][128] fp32
  static constexpr int SMEM = OFF_STAT + 2048;                    // base is 1024-aligned (checked in-kernel)
  static constexpr uint32_t TM_S = 0, TM_DP = 128, TM_DQ = 128, TM_DV = 256, TM_DK = 256 + D;
  static constexpr int DQ_BOXES = D / 32;                         // 32-column fp32 boxes of dQ per query tile
};

// Cycle counters of the per-role timeline; compiled out unless the timeline variant is launched.
template <bool TL>
__device__ __forceinline__ long long tick() { if constexpr (TL) return clock64(); else return 0; }

// DET (UPIPE_FLAG_DETERMINISTIC): heads-inner lockstep order and the dQ semaphores; compiled out of the
// default variant (measured: carrying them as runtime branches cost the q64 kernel ~20 %).
template <int D, bool TL, bool DET = false>
__global__ void __launch_bounds__(kThreads, 1)
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
  uint64_t* do_full = bars + 5;
  uint64_t* do_empty = bars + 6;
  uint64_t* sdp_full = bars + 7;
  uint64_t* ds_full = bars + 8;
  uint64_t* dq_full = bars + 9;
  uint64_t* dq_empty = bars + 10;
  uint64_t* dkv_full = bars + 11;
  uint64_t* ds_empty = bars + 12;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int warp = warp_id(), lane = lane_id();
  const int jb = blockIdx.x;                      // key tile (small jb = most query tiles = longest)
  const int g = blockIdx.y;                       // kv head
  const int G = a.nq / a.nkv;
  const int nT = (int)((a.S + 127) / 128);
  const int qt_begin = a.causal ? jb : 0;
  const int n_qt = nT - qt_begin;
  const int N = G * n_qt;                         // (head, query tile) iterations
  constexpr int kSoftmax = kSoftmaxWarps * 32;
  // visiting order: heads outer, query tiles up from the diagonal (default), or heads inner and query
  // tiles down to the diagonal (DET: all CTAs of the launch in lockstep, for dq_sem)
  auto tile_h = [&](int n) { return g * G + (DET ? n % G : n / n_qt); };
  auto tile_qt = [&](int n) { return DET ? nT - 1 - n / G : qt_begin + n % n_qt; };

  if (warp == kTmaWarp && lane == 0) {
    tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV); tma_prefetch(&tmdO); tma_prefetch(&tmdQ);
    for (int i = 0; i < 13; ++i) mbar_init(&bars[i], i == 8 ? kSoftmax : i == 10 ? 128 : 1);
    fence_barrier_init();
    tmem_slot[1] = smem_u32(smem);
  }
  if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= kTmaWarp) regs_dec<kRegsOther>();   // warpgroup 3 hands registers to the others
  if (warp == kTmaWarp) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      mbar_arrive_expect_tx(kv_full, 2 * C::TB);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        tma_load_3d(smem + C::OFF_K + c * 16384, &tmK, kv_full, c * 64, g, jb * 128);
        tma_load_3d(smem + C::OFF_V + c * 16384, &tmV, kv_full, c * 64, g, jb * 128);
      }
      for (int n = 0; n < N; ++n) {
        const int h = tile_h(n);
        const int qt = tile_qt(n);
        const int b = n & 1;
        mbar_wait(&q_empty[b], ((n >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[b], C::TB);
#pragma unroll
        for (int c = 0; c < NCH; ++c)
          tma_load_3d(smem + C::OFF_Q + b * C::TB + c * 16384, &tmQ, &q_full[b], c * 64, h, qt * 128);
        mbar_wait(do_empty, (n & 1) ^ 1);
        mbar_arrive_expect_tx(do_full, C::TB);
#pragma unroll
        for (int c = 0; c < NCH; ++c)
          tma_load_3d(smem + C::OFF_DO + c * 16384, &tmdO, do_full, c * 64, h, qt * 128);
      }
    }
  } else if (warp == kMmaWarp) {
    {
      // ------------------------------------------------ MMA issuer (whole warp; elect.sync inside the MMA asm)
      long long tl[5] = {0, 0, 0, 0, 0};
      constexpr uint32_t id_kk = idesc_bf16(128, 128, false, false);  // S^T, dP^T: both K-major over d
      constexpr uint32_t id_kmn = idesc_bf16(128, D, false, true);    // dV (A in TMEM), dK: B MN-major
      constexpr uint32_t id_mnmn = idesc_bf16(128, D, true, true);    // dQ: A = dS^T viewed MN-major, B = K MN-major
      // Shared-memory bases are re-read (volatile) every tile so the compiler cannot hoist ~40
      // loop-invariant 64-bit descriptors into this warp's small register budget; each MMA's
      // descriptor is base + immediate, computed right before the instruction.
      uint32_t sK, sV, sQ0, sdO, sdS;
      auto load_bases = [&]() {
        const uint32_t base = ld_volatile_shared_u32(tmem_slot + 1);
        sK = base + C::OFF_K; sV = base + C::OFF_V; sQ0 = base + C::OFF_Q; sdO = base + C::OFF_DO; sdS = base + C::OFF_DS;
      };
      load_bases();
      auto mma_kk = [&](uint32_t sa, uint32_t sb, uint32_t tm) {      // [128 x D] x [128 x D]^T
        const uint64_t da = desc_sw128(sa, 16, 1024), db = desc_sw128(sb, 16, 1024);
#pragma unroll
        for (int i = 0; i < 4 * NCH; ++i) {
          const uint32_t off = ((i >> 2) * 16384 + (i & 3) * 32) >> 4;
          mma_ss_w(tm, da + off, db + off, id_kk, i != 0);
        }
      };
      auto mma_kmn = [&](uint32_t sa, uint32_t sb, uint32_t tm, bool acc) {  // A [128 x 128 q] K-major smem
        const uint64_t da = desc_sw128(sa, 16, 1024), db = desc_sw128(sb, 16384, 1024);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          mma_ss_w(tm, da + (((i >> 2) * 16384 + (i & 3) * 32) >> 4), db + i * (2048 >> 4), id_kmn, (acc || i) ? 1u : 0u);
      };
      // A = P^T in TMEM: queries [16 ks, 16 ks + 16) are packed at TMEM cols 64 (ks / 4) + 8 (ks % 4)
      auto mma_tmn = [&](uint32_t ta, uint32_t sb, uint32_t tm, bool acc) {
        const uint64_t db = desc_sw128(sb, 16384, 1024);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          mma_ts_w(tm, ta + (ks >> 2) * 64 + (ks & 3) * 8, db + ks * (2048 >> 4), id_kmn, (acc || ks) ? 1u : 0u);
      };
      auto mma_mnmn = [&](uint32_t sa, uint32_t sb, uint32_t tm) {  // dQ = dS K: K dim = keys (rows of both)
        const uint64_t da = desc_sw128(sa, 16384, 1024), db = desc_sw128(sb, 16384, 1024);
#pragma unroll
        for (int i = 0; i < 8; ++i) mma_ss_w(tm, da + i * (2048 >> 4), db + i * (2048 >> 4), id_mnmn, i != 0);
      };
      mbar_wait(kv_full, 0);
      mbar_wait(&q_full[0], 0);
      tc_fence_after();
      mma_kk(sK, sQ0, tmem + C::TM_S);
      mbar_wait(do_full, 0);
      tc_fence_after();
      mma_kk(sV, sdO, tmem + C::TM_DP);
      mma_commit_w(sdp_full);
      for (int n = 0; n < N; ++n) {
        const int b = n & 1;
        long long t0 = tick<TL>();
        mbar_wait(ds_full, n & 1);
        long long t1 = tick<TL>();
        tl[0] += t1 - t0;
        tc_fence_after();
        load_bases();
        mma_tmn(tmem + C::TM_S, sdO, tmem + C::TM_DV, n > 0);
        mma_commit_w(do_empty);                           // dO(n) consumed: the producer loads dO(n+1)
        mma_mnmn(sdS, sK, tmem + C::TM_DQ);
        mma_commit_w(dq_full);                            // drained while S(n+1), dP(n+1) run
        tl[1] += tick<TL>() - t1;
        if (n + 1 < N) {
          const int b1 = (n + 1) & 1;
          long long t2 = tick<TL>();
          mbar_wait(&q_full[b1], ((n + 1) >> 1) & 1);
          tl[2] += tick<TL>() - t2;
          tc_fence_after();
          mma_kk(sK, sQ0 + b1 * C::TB, tmem + C::TM_S);   // in-order after dV(n), which reads P^T from these columns
          long long t3 = tick<TL>();
          mbar_wait(dq_empty, n & 1);
          long long t4 = tick<TL>();
          mbar_wait(do_full, (n + 1) & 1);
          tl[3] += t4 - t3;
          tl[4] += tick<TL>() - t4;
          tc_fence_after();
          mma_kk(sV, sdO, tmem + C::TM_DP);
          mma_commit_w(sdp_full);
        }
        // dK(n) last: it runs on the tensor core while the compute warps start on tile n+1
        mma_kmn(sdS, sQ0 + b * C::TB, tmem + C::TM_DK, n > 0);
        mma_commit_w(&q_empty[b]);
        mma_commit_w(ds_empty);                           // dS^T(n) consumed: tile n+1 may overwrite it
      }
      mma_commit_w(dkv_full);
      if (a.dbg && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0)
        for (int i = 0; i < 5; ++i) a.dbg[5 + i] = tl[i];
    }
  } else if (warp < kSoftmaxWarps) {
    // ------------------------------------------------ softmax-gradient warpgroups (warps 0-7)
    regs_inc<kRegsSoftmax>();
    const int wg = warp >> 2;                         // query columns [64 wg, 64 wg + 64) in two 32-column chunks
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const long long key = (long long)jb * 128 + r;
    const float sl2 = a.scale_log2;
    const uint32_t dsbase = smem_u32(smem + C::OFF_DS) + wg * 16384;   // dS^T chunk of this warpgroup's 64 queries
    float stat_next = 0.f;                            // warpgroup 0 prefetches lse, warpgroup 1 delta, one tile ahead
    auto load_stat = [&](int n) -> float {
      const int h = tile_h(n);
      const long long q = (long long)tile_qt(n) * 128 + r;
      if (q >= a.S) return 0.f;
      return wg == 0 ? a.lse[(long long)h * a.ld_lse + q] * -1.4426950408889634f : a.delta[q * a.ld_delta + h];
    };
    if (N > 0) stat_next = load_stat(0);
    long long tl[4] = {0, 0, 0, 0}, te[4] = {0, 0, 0, 0};   // te: E split into ld / math / store / wait_st
    for (int n = 0; n < N; ++n) {
      const int qt = tile_qt(n);
      const long long q0 = (long long)qt * 128;
      const int sb = n & 1;
      if (wg == 0) s_lse2[sb][r] = stat_next;
      else s_delta[sb][r] = stat_next;
      if (n + 1 < N) stat_next = load_stat(n + 1);
      // One warp polls the mbarrier; the others block in bar.sync (no issue slots spent spinning:
      // every waiting warp's try_wait/nanosleep loop competes with the softmax math for issue)
      long long c0 = tick<TL>();
      if (warp == 0) mbar_wait(sdp_full, n & 1);
      long long c1 = tick<TL>();
      named_bar_sync(1, kSoftmax);
      long long c2 = tick<TL>();
      tl[0] += c1 - c0;
      tl[1] += c2 - c1;
      tc_fence_after();
      const bool need_mask = (a.causal && qt == jb) || q0 + 128 > a.S || (long long)jb * 128 + 128 > a.S;
      const long long qmin = key >= a.S ? a.S : (a.causal ? key : 0);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int col0 = wg * 64 + c * 32;
        uint32_t rs[32], rp[32];
        const long long e0 = tick<TL>();
        tmem_ld32(tmem + C::TM_S + lane_off + col0, rs);
        tmem_ld32(tmem + C::TM_DP + lane_off + col0, rp);
        const float4* l4 = reinterpret_cast<const float4*>(&s_lse2[sb][col0]);
        const float4* d4 = reinterpret_cast<const float4*>(&s_delta[sb][col0]);
        // lse / delta (shared-memory broadcasts) are fetched while the TMEM loads are in flight
        float4 lx[8], dl[8];
#pragma unroll
        for (int i4 = 0; i4 < 8; ++i4) lx[i4] = l4[i4];
        tmem_wait_ld();
        const long long e1 = tick<TL>();
        te[0] += e1 - e0;
#pragma unroll
        for (int i4 = 0; i4 < 8; ++i4) dl[i4] = d4[i4];
        // P = 2^(s*c - lse2) on element pairs (FFMA2/FADD2/FMUL2 halve the issue slots); pairs with
        // j % UPIPE_BWD_MUFU_EVERY == 0 on MUFU, the rest as the polynomial on the FMA pipe.
        // s_lse2 holds -lse*log2(e).
        const uint64_t sl2x2 = f2_pack(sl2, sl2);
        uint64_t pp[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float4 x = lx[j >> 1];
          const uint64_t nl = (j & 1) ? f2_pack(x.z, x.w) : f2_pack(x.x, x.y);
          const uint64_t t = f2_fma(f2_pack(__uint_as_float(rs[2 * j]), __uint_as_float(rs[2 * j + 1])), sl2x2, nl);
          if ((j % UPIPE_BWD_MUFU_EVERY) == 0) {
            float t0, t1;
            f2_unpack(t, t0, t1);
            pp[j] = f2_pack(ex2b(t0), ex2b(t1));
          } else {
            pp[j] = ex2_fma2(t);
          }
        }
        if (need_mask) {                               // uniform branch: only diagonal / ragged tiles
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float p0, p1;
            f2_unpack(pp[j], p0, p1);
            const long long qa = q0 + col0 + 2 * j;
            p0 = (qa >= qmin && qa < a.S) ? p0 : 0.f;
            p1 = (qa + 1 >= qmin && qa + 1 < a.S) ? p1 : 0.f;
            pp[j] = f2_pack(p0, p1);
          }
        }
        // dS = P (dP - delta)
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float4 y = dl[j >> 1];
          const uint64_t dlt = (j & 1) ? f2_pack(y.z, y.w) : f2_pack(y.x, y.y);
          const uint64_t ds = f2_mul(pp[j], f2_sub(f2_pack(__uint_as_float(rp[2 * j]), __uint_as_float(rp[2 * j + 1])), dlt));
          float d0, d1, p0, p1;
          f2_unpack(ds, d0, d1);
          f2_unpack(pp[j], p0, p1);
          rp[2 * j] = __float_as_uint(d0);
          rp[2 * j + 1] = __float_as_uint(d1);
          rs[2 * j] = __float_as_uint(p0);
          rs[2 * j + 1] = __float_as_uint(p1);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i)
          rs[i] = pack_bf16(__uint_as_float(rs[2 * i]), __uint_as_float(rs[2 * i + 1]));
        const long long e2 = tick<TL>();
        te[1] += e2 - e1;
        // P^T (bf16 pairs) back into S^T columns already read: queries [col0, col0+32) -> cols 64 wg + 16 c
        tmem_st16(tmem + C::TM_S + lane_off + wg * 64 + c * 16, *reinterpret_cast<uint32_t(*)[16]>(rs));
        if (c == 0 && n > 0) {                         // dK(n-1) has read dS^T(n-1)
          long long w0 = tick<TL>();
          mbar_wait(ds_empty, (n - 1) & 1);
          tl[3] += tick<TL>() - w0;
        }
#pragma unroll
        for (int v8 = 0; v8 < 4; ++v8) {
          const int qc = c * 32 + v8 * 8;
          auto pk = [](uint32_t lo, uint32_t hi) { return pack_bf16(__uint_as_float(lo), __uint_as_float(hi)); };
          st_shared_v4(dsbase + sw128_offset(r, qc), pk(rp[v8 * 8 + 0], rp[v8 * 8 + 1]), pk(rp[v8 * 8 + 2], rp[v8 * 8 + 3]),
                       pk(rp[v8 * 8 + 4], rp[v8 * 8 + 5]), pk(rp[v8 * 8 + 6], rp[v8 * 8 + 7]));
        }
        te[2] += tick<TL>() - e2;
      }
      const long long e3 = tick<TL>();
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(ds_full);
      te[3] += tick<TL>() - e3;
      tl[2] += tick<TL>() - c2;
    }
    if (a.dbg && blockIdx.x == 0 && blockIdx.y == 0 && warp == 0 && lane == 0) {
      for (int i = 0; i < 3; ++i) a.dbg[i] = tl[i];
      a.dbg[11] = tl[3];
      a.dbg[10] = N;
      for (int i = 0; i < 4; ++i) a.dbg[12 + i] = te[i];
    }
    // ---- dK / dV epilogue (TMEM lane = key row): warpgroup 0 writes dV, warpgroup 1 dK
    mbar_wait(dkv_full, 0);
    tc_fence_after();
    const long long ldacc = (long long)a.nkv * D;
    const int which = wg;                           // 0: dV, 1: dK
    const int cbeg = 0;
    const uint32_t tcol = which ? C::TM_DK : C::TM_DV;
    const float sc = which ? a.scale : 1.f;
    float* acc = (which ? a.dk_acc : a.dv_acc);
    const bool ob = which ? (a.nkseg || a.dk_bf16) : (a.nvseg || a.dv_bf16);
#pragma unroll 1
    for (int c = cbeg; c < cbeg + D; c += 32) {
      uint32_t rr[32];
      tmem_ld32(tmem + tcol + lane_off + c, rr);
      tmem_wait_ld();
      if (key >= a.S || N == 0) continue;
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(rr[i]) * sc;
      float4* accp = acc ? reinterpret_cast<float4*>(acc + key * ldacc + (long long)g * D + c) : nullptr;
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
        if (which && a.rope.hi) rope_rotate<16>(v, a.rope.hi, a.rope.lo, D, a.rope.pos0 + key, c, -1.f);
        uint4* dst = reinterpret_cast<uint4*>(kv_out_row(a, which, key) + (long long)g * D + c);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_uint4(pack_bf16(v[8 * i + 0], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                              pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
      }
    }
  } else if (warp < kSoftmaxWarps + 4) {
    // ------------------------------------------------ dQ drain warpgroup (warps 8-11)
    // TMEM lane = query row. The whole dQ tile is loaded to registers first so the MMA
    // warp can reuse the columns for dP(n+1); it is then staged box by box (32 fp32
    // columns) through two 16 KB shared-memory slots and reduced into dq_acc by TMA.
    regs_inc<kRegsDrain>();
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const bool issuer = quad == 0 && lane == 0;
    long long tl[2] = {0, 0};
    int* sem_prev = nullptr;                          // deterministic dQ (see the q64 kernel's drain)
    for (int n = 0; n < N; ++n) {
      const int h = tile_h(n);
      const int q0 = tile_qt(n) * 128;
      int* const sem = DET ? a.dq_sem + (long long)h * nT + q0 / 128 : nullptr;
      long long c0 = tick<TL>();
      if (quad == 0) mbar_wait(dq_full, n & 1);   // one polling warp, the others wait in bar.sync
      named_bar_sync(2, 128);
      long long c1 = tick<TL>();
      tc_fence_after();
      uint32_t rq[C::DQ_BOXES][32];
#pragma unroll
      for (int b = 0; b < C::DQ_BOXES; ++b) tmem_ld32(tmem + C::TM_DQ + lane_off + b * 32, rq[b]);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(dq_empty);
#pragma unroll
      for (int b = 0; b < C::DQ_BOXES; ++b) {
        uint8_t* const slot = smem + C::OFF_STG + (b & 1) * 16384;
        if (issuer) bulk_wait_read1();   // the reduce that last used this slot (two groups back) has read it
        named_bar_sync(2, 128);
        const uint32_t stbase = smem_u32(slot);
#pragma unroll
        for (int j = 0; j < 8; ++j)       // 16-byte chunk j of the 128-byte row, swizzled by row % 8
          st_shared_v4(stbase + r * 128 + ((j ^ (r & 7)) << 4),
                       __float_as_uint(__uint_as_float(rq[b][4 * j + 0]) * a.scale),
                       __float_as_uint(__uint_as_float(rq[b][4 * j + 1]) * a.scale),
                       __float_as_uint(__uint_as_float(rq[b][4 * j + 2]) * a.scale),
                       __float_as_uint(__uint_as_float(rq[b][4 * j + 3]) * a.scale));
        fence_proxy_async_smem();
        named_bar_sync(2, 128);
        if (issuer) {
          if (b == 0 && sem) sem_wait_eq(sem, jb);
          tma_reduce_add_2d(&tmdQ, slot, h * D + b * 32, q0);
          bulk_commit();
          if (b == C::DQ_BOXES - 1) {
            if (sem_prev) {                             // the previous tile's boxes have completed
              bulk_wait_n<C::DQ_BOXES>();
              fence_proxy_async_global();
              st_release_gpu(sem_prev, jb + 1);
            }
            sem_prev = sem;
          }
        }
      }
      tl[0] += c1 - c0;
      tl[1] += tick<TL>() - c1;
    }
    if (issuer) {
      bulk_wait0();
      if (sem_prev) {
        fence_proxy_async_global();
        st_release_gpu(sem_prev, jb + 1);
      }
    }
    if (a.dbg && blockIdx.x == 0 && blockIdx.y == 0 && warp == kSoftmaxWarps && lane == 0) {
      a.dbg[3] = tl[0];
      a.dbg[4] = tl[1];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}


// ---------------------------------------------------------------------------------------------
// Q64 variant (d = 128): 64-query tiles in two TMEM slots, so one slot's softmax-gradient work
// overlaps the other slot's MMAs (ping-pong, as in the forward). TMEM: S_A | dP_A | S_B | dP_B
// (64 columns each) | dV | dK; per tile n in slot x = n & 1 the tensor core runs
//   dV(n) += P^T dO, dQ^T(n) = K^T dS (into dP_x), dK(n) += dS^T Q, S(n+2), dP(n+2)
// where S / dP / dQ^T are N = 64 MMAs. dQ^T leaves TMEM with one dimension per lane and is staged
// transposed (one 64 x 32 fp32 box per drain warp) for the TMA reduce-add into dq_acc.
// kDkTs (UPIPE_BWD_DK_TS=1 at build time): the q64 kernel's dK MMA takes dS^T from TMEM (TS form; the softmax
// warps store it next to P^T in the slot's S columns, which the S^T read has freed) instead of from shared
// memory: 16 KB less shared-memory operand traffic per 64-query tile. Measured neutral (same-box A/B at 128K,
// profiles/r02_ab_bwd_dkts.txt: attn bwd 82.5 vs 82.7 ms per launch, 339.9 vs 338.7 ms per bench step), so the
// tensor pipe's operand reads do not compete with the other shared-memory traffic here; off by default.
#ifndef UPIPE_BWD_DK_TS
#define UPIPE_BWD_DK_TS 0
#endif
constexpr bool kDkTs = UPIPE_BWD_DK_TS != 0;

struct Q64Cfg {
  static constexpr int D = 128;
  static constexpr int KT = 128 * D * 2;            // K or V tile: 128 keys x 128 d bf16 (two 16 KB chunks)
  static constexpr int QT = 64 * D * 2;             // Q or dO tile: 64 queries x 128 d (two 8 KB chunks)
  static constexpr int NQ = 3;                      // Q / dO ring depth
  static constexpr int OFF_K = 0, OFF_V = KT, OFF_Q = 2 * KT, OFF_DO = OFF_Q + NQ * QT;
  static constexpr int OFF_DS = OFF_DO + NQ * QT;   // dS^T [128 keys][64 q] bf16 per slot (16 KB)
  static constexpr int OFF_STG = OFF_DS + 2 * 16384; // dQ^T staging: 4 warps x (64 q x 32 d fp32 = 8 KB)
  static constexpr int OFF_STAT = OFF_STG + 32768;  // [slot][parity] lse2[64], delta[64]
  static constexpr int OFF_BAR = OFF_STAT + 2048;
  static constexpr int SMEM = OFF_BAR + 256;
  static_assert(SMEM <= 232448, "shared memory");
  static constexpr uint32_t TM_S0 = 0, TM_DP0 = 64, TM_S1 = 128, TM_DP1 = 192, TM_DV = 256, TM_DK = 384;
};

// PAIR (UPIPE_BWD_PAIR): clusters of two CTAs on adjacent key tiles (2i, 2i+1) of one KV head visit the same
// query tiles in the same order (the even tile's range; the odd CTA's extra tiles are fully masked for it), so
// each CTA loads one half of every Q / dO tile and multicasts it to both: half the L2 -> SM operand traffic.
// UPIPE_BWD_CLUSTER (build time, 2 or 4): CTAs per cluster of the PAIR launch. With 4, each CTA loads one quarter of
// every Q / dO tile (one 64-dimension chunk, 32 query rows) and multicasts it to all four.
#ifndef UPIPE_BWD_CLUSTER
#define UPIPE_BWD_CLUSTER 2
#endif
constexpr int kBwdCluster = UPIPE_BWD_CLUSTER;
static_assert(kBwdCluster == 2 || kBwdCluster == 4, "UPIPE_BWD_CLUSTER: 2 or 4");

template <bool TL, bool DET = false, bool PAIR = false>
__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_q64_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                        const __grid_constant__ CUtensorMap tmdQ, const BwdArgs a) {
  using C = Q64Cfg;
  constexpr int D = C::D;
  extern __shared__ __align__(1024) uint8_t smem[];
  if (smem_u32(smem) & 1023) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* kv_full = bars + 0;
  uint64_t* q_full = bars + 1;      // [3]
  uint64_t* q_empty = bars + 4;     // [3]
  uint64_t* do_full = bars + 7;     // [3]
  uint64_t* do_empty = bars + 10;   // [3]
  uint64_t* sdp_full = bars + 13;   // [2] S(n), dP(n) of slot n & 1 in TMEM
  uint64_t* ds_full = bars + 15;    // [2] P^T in TMEM, dS^T in smem (128 arrivals)
  uint64_t* dq_full = bars + 17;    // [2]
  uint64_t* dq_empty = bars + 19;   // [2] (128 arrivals)
  uint64_t* dkv_full = bars + 21;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);
  float* stats = reinterpret_cast<float*>(smem + C::OFF_STAT);   // [(slot*2 + parity)*2 + {lse2, delta}][64]

  const int warp = warp_id(), lane = lane_id();
  const int jb = blockIdx.x;
  const int g = blockIdx.y;
  const int G = a.nq / a.nkv;
  const int nT64 = (int)((a.S + 63) / 64);
  constexpr int CLN = PAIR ? kBwdCluster : 1;
  constexpr uint16_t kMask = (uint16_t)((1u << CLN) - 1);
  const uint32_t crank = PAIR ? cluster_ctarank() : 0;
  const int qt_begin = a.causal ? 2 * (jb & ~(CLN - 1)) : 0;   // PAIR: the cluster's common range (its first tile's)
  const int n_qt = nT64 - qt_begin;
  const int N = G * n_qt;
  // Query tiles are visited from the last one down to the diagonal: CTAs that run at the same time then
  // reduce their dQ partials into the same rows of dq_acc (L2 hits) instead of each starting at its own
  // diagonal and sweeping a different region (measured: the dQ reduce-adds dominated the energy).
  // Heads of the KV group outer (default) or inner (DET, the deterministic lockstep order).
  auto tile_h = [&](int n) { return g * G + (DET ? n % G : n / n_qt); };
  auto tile_qt = [&](int n) { return nT64 - 1 - (DET ? n / G : n % n_qt); };
  constexpr int kWg = 128;

  if (warp == kTmaWarp && lane == 0) {
    tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV); tma_prefetch(&tmdO); tma_prefetch(&tmdQ);
    for (int i = 0; i < 22; ++i) {
      const bool slot_empty = (i >= 4 && i < 7) || (i >= 10 && i < 13);   // q_empty, do_empty: both CTAs release
      mbar_init(&bars[i], (i == 15 || i == 16 || i == 19 || i == 20) ? kWg : (slot_empty ? CLN : 1));
    }
    fence_barrier_init();
    tmem_slot[1] = smem_u32(smem);
  }
  if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();                // the peer's barriers exist before any multicast lands in them
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= kTmaWarp) regs_dec<kRegsOther>();
  if (warp == kTmaWarp) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * C::KT);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        tma_load_3d(smem + C::OFF_K + c * 16384, &tmK, kv_full, c * 64, g, jb * 128);
        tma_load_3d(smem + C::OFF_V + c * 16384, &tmV, kv_full, c * 64, g, jb * 128);
      }
      for (int n = 0; n < N; ++n) {
        const int h = tile_h(n);
        const int qt = tile_qt(n);
        const int st = n % C::NQ;
        const uint32_t ph = ((n / C::NQ) & 1) ^ 1;
        mbar_wait(&q_empty[st], ph);              // PAIR: this slot is free in both CTAs
        mbar_arrive_expect_tx(&q_full[st], C::QT);
        if (PAIR && CLN == 4) {                   // this CTA's quarter (chunk crank & 1, rows 32 (crank >> 1)) to all
          tma_load_3d_mc(smem + C::OFF_Q + st * C::QT + (crank & 1) * 8192 + (crank >> 1) * 4096, &tmQ, &q_full[st],
                         (crank & 1) * 64, h, qt * 64 + (crank >> 1) * 32, kMask);
        } else if (PAIR) {                        // this CTA's half (one 64-dim chunk) to both CTAs
          tma_load_3d_mc(smem + C::OFF_Q + st * C::QT + crank * 8192, &tmQ, &q_full[st], crank * 64, h, qt * 64, 0x3);
        } else {
#pragma unroll
          for (int c = 0; c < 2; ++c) tma_load_3d(smem + C::OFF_Q + st * C::QT + c * 8192, &tmQ, &q_full[st], c * 64, h, qt * 64);
        }
        mbar_wait(&do_empty[st], ph);
        mbar_arrive_expect_tx(&do_full[st], C::QT);
        if (PAIR && CLN == 4) {
          tma_load_3d_mc(smem + C::OFF_DO + st * C::QT + (crank & 1) * 8192 + (crank >> 1) * 4096, &tmdO, &do_full[st],
                         (crank & 1) * 64, h, qt * 64 + (crank >> 1) * 32, kMask);
        } else if (PAIR) {
          tma_load_3d_mc(smem + C::OFF_DO + st * C::QT + crank * 8192, &tmdO, &do_full[st], crank * 64, h, qt * 64,
                         0x3);
        } else {
#pragma unroll
          for (int c = 0; c < 2; ++c)
            tma_load_3d(smem + C::OFF_DO + st * C::QT + c * 8192, &tmdO, &do_full[st], c * 64, h, qt * 64);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    constexpr uint32_t id_sp = idesc_bf16(128, 64, false, false);    // S^T, dP^T: K-major A (K/V) and B (Q/dO)
    constexpr uint32_t id_kmn = idesc_bf16(128, D, false, true);     // dV (A in TMEM), dK: B = Q / dO MN-major
    constexpr uint32_t id_dq = idesc_bf16(128, 64, true, true);      // dQ^T = K^T dS: both MN-major
    uint32_t base;
    auto load_base = [&]() { base = ld_volatile_shared_u32(tmem_slot + 1); };
    load_base();
    auto mma_sp = [&](uint32_t skv, uint32_t sqt, uint32_t tm) {   // [128 keys x d] x [64 q x d]^T
      const uint64_t da = desc_sw128(skv, 16, 1024), db = desc_sw128(sqt, 16, 1024);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        mma_ss_w(tm, da + (((i >> 2) * 16384 + (i & 3) * 32) >> 4), db + (((i >> 2) * 8192 + (i & 3) * 32) >> 4),
                 id_sp, i != 0);
    };
    // TMEM column of the 16-query A chunk ks (P^T, or dS^T at +16) in a slot's S columns: see kDkTs
    auto a_col = [](int ks) -> uint32_t { return kDkTs ? (ks >> 1) * 32 + (ks & 1) * 8 : ks * 8; };
    auto mma_dv = [&](uint32_t tp, uint32_t sdo, bool acc) {       // dV += P^T dO: A = P^T (TMEM, 64 q)
      const uint64_t db = desc_sw128(sdo, 8192, 1024);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
        mma_ts_w(tmem + C::TM_DV, tp + a_col(ks), db + ks * (2048 >> 4), id_kmn, (acc || ks) ? 1u : 0u);
    };
    auto mma_dk = [&](uint32_t sds, uint32_t tp, uint32_t sq, bool acc) {   // dK += dS^T Q (64 q)
      const uint64_t da = desc_sw128(sds, 16, 1024), db = desc_sw128(sq, 8192, 1024);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        if constexpr (kDkTs)   // A = dS^T from TMEM (the slot's S columns next to P^T)
          mma_ts_w(tmem + C::TM_DK, tp + a_col(ks) + 16, db + ks * (2048 >> 4), id_kmn, (acc || ks) ? 1u : 0u);
        else                   // A = dS^T from shared memory (K-major)
          mma_ss_w(tmem + C::TM_DK, da + ((ks * 32) >> 4), db + ks * (2048 >> 4), id_kmn, (acc || ks) ? 1u : 0u);
      }
    };
    auto mma_dq = [&](uint32_t sk, uint32_t sds, uint32_t tm) {    // dQ^T = K^T dS over the 128 keys
      const uint64_t da = desc_sw128(sk, 16384, 1024), db = desc_sw128(sds, 8192, 1024);
#pragma unroll
      for (int i = 0; i < 8; ++i) mma_ss_w(tm, da + i * (2048 >> 4), db + i * (2048 >> 4), id_dq, i != 0);
    };
    auto slot_s = [](int x) { return x ? C::TM_S1 : C::TM_S0; };
    auto slot_dp = [](int x) { return x ? C::TM_DP1 : C::TM_DP0; };
    mbar_wait(kv_full, 0);
    for (int t = 0; t < 2 && t < N; ++t) {
      mbar_wait(&q_full[t], 0);
      tc_fence_after();
      mma_sp(base + C::OFF_K, base + C::OFF_Q + t * C::QT, tmem + slot_s(t));
      mbar_wait(&do_full[t], 0);
      tc_fence_after();
      mma_sp(base + C::OFF_V, base + C::OFF_DO + t * C::QT, tmem + slot_dp(t));
      mma_commit_w(&sdp_full[t]);
    }
    long long tw[5] = {0, 0, 0, 0, 0};               // wait dS, wait Q, wait dQ drained, wait dO, total
    const long long tbeg = tick<TL>();
    for (int n = 0; n < N; ++n) {
      const int x = n & 1;
      const int st = n % C::NQ;
      long long w0 = tick<TL>();
      mbar_wait(&ds_full[x], (n >> 1) & 1);
      tw[0] += tick<TL>() - w0;
      tc_fence_after();
      load_base();
      const uint32_t sds = base + C::OFF_DS + x * 16384;
      mma_dv(tmem + slot_s(x), base + C::OFF_DO + st * C::QT, n > 0);
      if (PAIR) mma_commit_mc_w(&do_empty[st], kMask);   // released in every CTA of the cluster (each loads into all)
      else mma_commit_w(&do_empty[st]);
      mma_dq(base + C::OFF_K, sds, tmem + slot_dp(x));
      mma_commit_w(&dq_full[x]);
      mma_dk(sds, tmem + slot_s(x), base + C::OFF_Q + st * C::QT, n > 0);
      if (PAIR) mma_commit_mc_w(&q_empty[st], kMask);
      else mma_commit_w(&q_empty[st]);
      if (n + 2 < N) {
        const int st2 = (n + 2) % C::NQ;
        const uint32_t ph2 = ((n + 2) / C::NQ) & 1;
        long long w1 = tick<TL>();
        mbar_wait(&q_full[st2], ph2);
        tw[1] += tick<TL>() - w1;
        tc_fence_after();
        mma_sp(base + C::OFF_K, base + C::OFF_Q + st2 * C::QT, tmem + slot_s(x));   // after dV(n) read P^T
        w1 = tick<TL>();
        mbar_wait(&dq_empty[x], (n >> 1) & 1);                                        // dQ^T(n) drained
        tw[2] += tick<TL>() - w1;
        w1 = tick<TL>();
        mbar_wait(&do_full[st2], ph2);
        tw[3] += tick<TL>() - w1;
        tc_fence_after();
        mma_sp(base + C::OFF_V, base + C::OFF_DO + st2 * C::QT, tmem + slot_dp(x));
        mma_commit_w(&sdp_full[x]);
      }
    }
    mma_commit_w(dkv_full);
    tw[4] = tick<TL>() - tbeg;
    if (TL && a.dbg && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0)
      for (int i = 0; i < 5; ++i) a.dbg[i] = tw[i];
  } else if (warp < kSoftmaxWarps) {
    // ------------------------------------------------ softmax-gradient warpgroups: WG x owns slot x
    regs_inc<kRegsSoftmax>();
    const int x = warp >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;                   // key row of the tile
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const long long key = (long long)jb * 128 + r;
    const float sl2 = a.scale_log2;
    const uint32_t tS = tmem + (x ? C::TM_S1 : C::TM_S0) + lane_off;
    const uint32_t tP = tmem + (x ? C::TM_DP1 : C::TM_DP0) + lane_off;
    const uint32_t dsbase = smem_u32(smem + C::OFF_DS + x * 16384);
    auto load_stat = [&](int n) -> float {            // threads 0-63: -lse*log2e of query r, 64-127: delta
      const int h = tile_h(n);
      const long long q = (long long)tile_qt(n) * 64 + (r & 63);
      if (q >= a.S) return 0.f;
      return r < 64 ? a.lse[(long long)h * a.ld_lse + q] * -1.4426950408889634f : a.delta[q * a.ld_delta + h];
    };
    float stat_next = x < N ? load_stat(x) : 0.f;
    long long te[2] = {0, 0};                         // wait S/dP, E
    for (int n = x; n < N; n += 2) {
      const int qt = tile_qt(n);
      const long long q0 = (long long)qt * 64;
      const int par = (n >> 1) & 1;
      float* s_lse2 = stats + ((x * 2 + par) * 2 + 0) * 64;
      float* s_delta = stats + ((x * 2 + par) * 2 + 1) * 64;
      (r < 64 ? s_lse2 : s_delta)[r & 63] = stat_next;
      if (n + 2 < N) stat_next = load_stat(n + 2);
      const long long e0 = tick<TL>();
      if (quad == 0) mbar_wait(&sdp_full[x], (n >> 1) & 1);
      named_bar_sync(1 + x, kWg);
      const long long e1 = tick<TL>();
      te[0] += e1 - e0;
      tc_fence_after();
      // the diagonal tile pair, and (PAIR, odd CTA) the pair's common tiles that lie entirely below its keys
      const bool need_mask = (a.causal && (qt >> 1) <= jb) || q0 + 64 > a.S || (long long)jb * 128 + 128 > a.S;
      const long long qmin = key >= a.S ? a.S : (a.causal ? key : 0);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int col0 = c * 32;
        uint32_t rs[32], rp[32];
        tmem_ld32(tS + col0, rs);
        tmem_ld32(tP + col0, rp);
        const float4* l4 = reinterpret_cast<const float4*>(s_lse2 + col0);
        const float4* d4 = reinterpret_cast<const float4*>(s_delta + col0);
        float4 lx[8], dl[8];
#pragma unroll
        for (int i4 = 0; i4 < 8; ++i4) lx[i4] = l4[i4];
        tmem_wait_ld();
#pragma unroll
        for (int i4 = 0; i4 < 8; ++i4) dl[i4] = d4[i4];
        const uint64_t sl2x2 = f2_pack(sl2, sl2);
        uint64_t pp[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float4 xx = lx[j >> 1];
          const uint64_t nl = (j & 1) ? f2_pack(xx.z, xx.w) : f2_pack(xx.x, xx.y);
          const uint64_t t = f2_fma(f2_pack(__uint_as_float(rs[2 * j]), __uint_as_float(rs[2 * j + 1])), sl2x2, nl);
          float t0, t1;
          f2_unpack(t, t0, t1);
          pp[j] = f2_pack(ex2b(t0), ex2b(t1));
        }
        if (need_mask) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float p0, p1;
            f2_unpack(pp[j], p0, p1);
            const long long qa = q0 + col0 + 2 * j;
            p0 = (qa >= qmin && qa < a.S) ? p0 : 0.f;
            p1 = (qa + 1 >= qmin && qa + 1 < a.S) ? p1 : 0.f;
            pp[j] = f2_pack(p0, p1);
          }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float4 y = dl[j >> 1];
          const uint64_t dlt = (j & 1) ? f2_pack(y.z, y.w) : f2_pack(y.x, y.y);
          const uint64_t ds = f2_mul(pp[j], f2_sub(f2_pack(__uint_as_float(rp[2 * j]), __uint_as_float(rp[2 * j + 1])), dlt));
          float d0, d1, p0, p1;
          f2_unpack(ds, d0, d1);
          f2_unpack(pp[j], p0, p1);
          rp[j] = pack_bf16(d0, d1);
          rs[j] = pack_bf16(p0, p1);
        }
        // P^T (bf16 pairs) into the S^T columns already read: queries [col0, col0+32) -> cols 16 c, or (kDkTs)
        // cols 32 c with dS^T (the dK MMA's A operand) next to it in cols 32 c + 16
        if constexpr (kDkTs) {
          tmem_st16(tS + c * 32, *reinterpret_cast<uint32_t(*)[16]>(rs));
          tmem_st16(tS + c * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(rp));
          if (c == 0) tmem_wait_st();   // the stores' source registers stay reserved until the wait (else: spills)
        } else {
          tmem_st16(tS + c * 16, *reinterpret_cast<uint32_t(*)[16]>(rs));
        }
#pragma unroll
        for (int v8 = 0; v8 < 4; ++v8)
          st_shared_v4(dsbase + sw128_offset(r, col0 + v8 * 8), rp[4 * v8], rp[4 * v8 + 1], rp[4 * v8 + 2], rp[4 * v8 + 3]);
      }
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&ds_full[x]);
      te[1] += tick<TL>() - e1;
    }
    if (TL && a.dbg && blockIdx.x == 0 && blockIdx.y == 0 && quad == 0 && lane == 0) {
      a.dbg[5 + 2 * x] = te[0];
      a.dbg[6 + 2 * x] = te[1];
    }
    // ---- dK / dV epilogue (TMEM lane = key row): warpgroup 0 writes dV, warpgroup 1 dK
    mbar_wait(dkv_full, 0);
    tc_fence_after();
    const long long ldacc = (long long)a.nkv * D;
    const int which = x;
    const uint32_t tcol = which ? C::TM_DK : C::TM_DV;
    const float sc = which ? a.scale : 1.f;
    float* acc = (which ? a.dk_acc : a.dv_acc);
    const bool ob = which ? (a.nkseg || a.dk_bf16) : (a.nvseg || a.dv_bf16);
#pragma unroll 1
    for (int c = 0; c < D; c += 32) {
      uint32_t rr[32];
      tmem_ld32(tmem + tcol + lane_off + c, rr);
      tmem_wait_ld();
      if (key >= a.S || N == 0) continue;
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(rr[i]) * sc;
      float4* accp = acc ? reinterpret_cast<float4*>(acc + key * ldacc + (long long)g * D + c) : nullptr;
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
        if (which && a.rope.hi) rope_rotate<16>(v, a.rope.hi, a.rope.lo, D, a.rope.pos0 + key, c, -1.f);
        uint4* dst = reinterpret_cast<uint4*>(kv_out_row(a, which, key) + (long long)g * D + c);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_uint4(pack_bf16(v[8 * i + 0], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                              pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
      }
    }
  } else if (warp < kSoftmaxWarps + 4) {
    // ------------------------------------------------ dQ drain (warps 8-11): TMEM lane = head dim
    regs_inc<kRegsDrain>();
    const int quad = warp & 3;                        // dims [32 quad, 32 quad + 32) = this warp's box
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    uint8_t* const box = smem + C::OFF_STG + quad * 8192;
    const uint32_t bbase = smem_u32(box);
    long long td[1] = {0};
    int* sem_prev = nullptr;                          // deterministic dQ: released one step late (below)
    for (int n = 0; n < N; ++n) {
      const int x = n & 1;
      const int h = tile_h(n);
      const int q0 = tile_qt(n) * 64;
      int* const sem = DET ? a.dq_sem + ((long long)h * nT64 + q0 / 64) * 4 + quad : nullptr;
      // Deterministic dQ: key tile jb adds after key tiles 0..jb-1 (every earlier key tile contributes to
      // every query tile this CTA visits); the release of step n waits for its reduce to COMPLETE, which is
      // done one step later (wait_group 1) so the drain never idles on its own reduce.
      auto issue = [&](auto&& do_reduce) {
        if (sem) sem_wait_eq(sem, jb);
        do_reduce();
        bulk_commit();
        if (sem_prev) {
          bulk_wait1();
          fence_proxy_async_global();
          st_release_gpu(sem_prev, jb + 1);
        }
        sem_prev = sem;
      };
      const long long d0 = tick<TL>();
      if (lane == 0) mbar_wait(&dq_full[x], (n >> 1) & 1);
      __syncwarp();
      td[0] += tick<TL>() - d0;
      tc_fence_after();
      uint32_t rq[2][32];
      const uint32_t tq = tmem + (x ? C::TM_DP1 : C::TM_DP0) + lane_off;
      tmem_ld32(tq, rq[0]);
      tmem_ld32(tq + 32, rq[1]);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&dq_empty[x]);
      if (lane == 0) bulk_wait_read0();               // this warp's previous box has been read by its reduce
      __syncwarp();
      if (a.dq_dim_major) {
        // dim-major accumulator: row lane (dim) of two 32-token boxes, 16-byte chunks, 128B swizzle
#pragma unroll
        for (int bx = 0; bx < 2; ++bx)
#pragma unroll
          for (int j = 0; j < 8; ++j)
            st_shared_v4(bbase + bx * 4096 + lane * 128 + ((j ^ (lane & 7)) << 4),
                         __float_as_uint(__uint_as_float(rq[bx][4 * j + 0]) * a.scale),
                         __float_as_uint(__uint_as_float(rq[bx][4 * j + 1]) * a.scale),
                         __float_as_uint(__uint_as_float(rq[bx][4 * j + 2]) * a.scale),
                         __float_as_uint(__uint_as_float(rq[bx][4 * j + 3]) * a.scale));
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0)
          issue([&] {
            tma_reduce_add_2d(&tmdQ, box, q0, h * D + quad * 32);
            tma_reduce_add_2d(&tmdQ, box + 4096, q0 + 32, h * D + quad * 32);
          });
        continue;
      }
      // row q (query), column lane (dim): 128B-swizzled rows of 32 fp32
#pragma unroll
      for (int q = 0; q < 64; ++q)
        st_shared_f32(bbase + q * 128 + ((((uint32_t)lane >> 2) ^ ((uint32_t)q & 7)) << 4) + (lane & 3) * 4,
                      __uint_as_float(rq[q >> 5][q & 31]) * a.scale);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) issue([&] { tma_reduce_add_2d(&tmdQ, box, h * D + quad * 32, q0); });
    }
    if (lane == 0) {
      bulk_wait0();
      if (sem_prev) {
        fence_proxy_async_global();
        st_release_gpu(sem_prev, jb + 1);
      }
    }
    if (TL && a.dbg && blockIdx.x == 0 && blockIdx.y == 0 && quad == 0 && lane == 0) {
      a.dbg[9] = td[0];
      a.dbg[10] = N;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
  if (PAIR) cluster_sync();                // no CTA leaves while its peer may still multicast into it or signal it
}

// d = 128: the 64-query ping-pong kernel. Under the 1000 W power cap it runs at lower SM clocks than
// the 128-query kernel (busier tensor pipe), yet with the dim-major dQ accumulator and last-to-first
// query order it is ahead at every length measured: attn bwd per step 375 -> 340 ms at 128K, 5940 ->
// 5618 ms at 512K, 24184 -> 24066 ms at 1M (profiles/r01_ab_bwd_q64_dimmajor_512k_1m.txt). Before those
// two changes it lost at 512K (6005 vs 6091 ms). UPIPE_BWD_Q64=0 selects the 128-query kernel.
// The CTA-pair variant of the 64-query kernel (Q / dO multicast within the pair), default: half the L2 -> SM
// operand traffic lowers the energy per tile, so the power-capped clock rises (A/B at 128K on one box: attn
// bwd 350.3 -> 342.7 ms per step at 1477-1485 -> 1507 MHz). UPIPE_BWD_PAIR=0 selects the single-CTA launch.
// A cta_group::2 variant (128-query tiles over CTA pairs, pair MMAs for all five products, dQ over both CTAs' keys
// with dS exchanged over DSMEM) passed kernel parity but ran at half this kernel's rate (530-570 TFLOP/s at 32K-128K,
// profiles/r02_ab_bwd_cta2.txt): in our probes pair MMAs issued back to back took ~106-166 cycles per K16 instruction
// (profiles/r02_micro_pair.txt) and its softmax could not overlap the MMAs. Source: commit 4d629cc; retired.
bool bwd_pair() {
  static const bool on = [] {
    const char* v = getenv("UPIPE_BWD_PAIR");
    return !(v && v[0] == '0');
  }();
  return on;
}

bool use_q64(const AttnBwdProblem& p) {
  static const int q64_env = [] {
    const char* v = getenv("UPIPE_BWD_Q64");
    return v ? (v[0] == '1' ? 1 : 0) : -1;
  }();
  if (p.d != 128) return false;
  return q64_env != 0;
}

}  // namespace

bool attn_bwd_dq_dim_major(const AttnBwdProblem& p) {
  static const bool off = [] {
    const char* v = getenv("UPIPE_DQ_DIM_MAJOR");
    return v && v[0] == '0';
  }();
  return !off && use_q64(p);
}

bool attn_bwd_dq_dim_major_supported(const AttnBwdProblem& p) { return use_q64(p); }

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
  a.dq_acc = p.dq_acc;
  a.lse = p.lse;
  a.delta = p.delta;
  a.dk_acc = p.dk_acc;
  a.dv_acc = p.dv_acc;
  a.dk_bf16 = reinterpret_cast<__nv_bfloat16*>(p.dk_bf16);
  a.dv_bf16 = reinterpret_cast<__nv_bfloat16*>(p.dv_bf16);
  a.nkseg = p.dk_seg.n;
  a.nvseg = p.dv_seg.n;
  const int64_t seg_rows = p.dk_seg.n ? p.dk_seg.rows : p.dv_seg.rows;
  a.kvseg_rows = seg_rows > 0 ? seg_rows : 1;
  for (int i = 0; i < kMaxSeg; ++i) {
    a.dkseg[i] = reinterpret_cast<__nv_bfloat16*>(p.dk_seg.p[i]);
    a.dvseg[i] = reinterpret_cast<__nv_bfloat16*>(p.dv_seg.p[i]);
  }
  for (const SegPtrs* sp : {&p.dk_seg, &p.dv_seg})
    if (sp->n && (sp->rows != seg_rows || sp->rows <= 0 || sp->n > kMaxSeg || (p.S + sp->rows - 1) / sp->rows > sp->n)) {
      snprintf(err, errlen, "attn_bwd: segmented dK/dV need equal segment rows covering S");
      return cudaErrorInvalidValue;
    }
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
  a.rope = p.rope;
  a.dq_dim_major = 0;
  a.dq_sem = p.dq_sem;
  // UPIPE_BWD_TIMELINE=1: per-role cycle breakdown of CTA (0,0), printed to stderr after the launch
  static long long* dbg_dev = nullptr;
  const char* tlenv = getenv("UPIPE_BWD_TIMELINE");
  a.dbg = nullptr;
  if (tlenv && tlenv[0] == '1') {
    if (!dbg_dev) cudaMalloc(&dbg_dev, 16 * sizeof(long long));
    cudaMemsetAsync(dbg_dev, 0, 16 * sizeof(long long), stream);
    a.dbg = dbg_dev;
  }
  const int nT = (int)((p.S + 127) / 128);
  dim3 grid(nT, p.nkv);
  cudaError_t e;
  if (use_q64(p)) {
    if (p.dq_dim_major && p.ld_dqt < p.S) {
      snprintf(err, errlen, "attn_bwd: dim-major dq_acc needs ld_dqt >= S");
      return cudaErrorInvalidValue;
    }
    a.dq_dim_major = p.dq_dim_major;
    CUtensorMap tq64, tdo64, tdq64;
    if (!make_tmap_3d(&tq64, p.q, p.d, p.nq, p.S, p.d, p.ldq, 64, 1, 64, err, errlen)) return cudaErrorInvalidValue;
    if (!make_tmap_3d(&tdo64, p.dout, p.d, p.nq, p.S, p.d, p.ldo_grad, 64, 1, 64, err, errlen))
      return cudaErrorInvalidValue;
    if (p.dq_dim_major) {
      if (!make_tmap_2d_f32(&tdq64, p.dq_acc, p.S, (uint64_t)p.nq * p.d, p.ld_dqt, 32, 32, err, errlen))
        return cudaErrorInvalidValue;
    } else if (!make_tmap_2d_f32(&tdq64, p.dq_acc, (uint64_t)p.nq * p.d, p.S, (uint64_t)p.nq * p.d, 32, 64, err,
                                 errlen)) {
      return cudaErrorInvalidValue;
    }
    const cudaError_t attr = set_smem_attr((const void*)attn_bwd_q64_kernel<false>, Q64Cfg::SMEM) == cudaSuccess &&
                                     set_smem_attr((const void*)attn_bwd_q64_kernel<false, false, true>, Q64Cfg::SMEM) ==
                                         cudaSuccess
                                 ? set_smem_attr((const void*)attn_bwd_q64_kernel<false, true>, Q64Cfg::SMEM)
                                 : cudaErrorInvalidValue;
    if (attr != cudaSuccess) { snprintf(err, errlen, "attn_bwd_q64 attr: %s", cudaGetErrorString(attr)); return attr; }
    const cudaError_t attr2 = set_smem_attr((const void*)attn_bwd_q64_kernel<true>, Q64Cfg::SMEM);
    if (attr2 != cudaSuccess) { snprintf(err, errlen, "attn_bwd_q64 attr: %s", cudaGetErrorString(attr2)); return attr2; }
    if (a.dbg) attn_bwd_q64_kernel<true><<<grid, kThreads, Q64Cfg::SMEM, stream>>>(tq64, tk, tv, tdo64, tdq64, a);
    else if (a.dq_sem) attn_bwd_q64_kernel<false, true><<<grid, kThreads, Q64Cfg::SMEM, stream>>>(tq64, tk, tv, tdo64, tdq64, a);
    else if (bwd_pair()) {
      // CTA pairs (clusters of 2 along the key tiles; an odd tile count gets one key tile past the end, fully
      // masked and written nowhere)
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      cfg.gridDim = dim3((unsigned)((nT + kBwdCluster - 1) / kBwdCluster * kBwdCluster), (unsigned)p.nkv);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = Q64Cfg::SMEM;
      cfg.stream = stream;
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = kBwdCluster;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      CUtensorMap tq32, tdo32;                 // quads: one quarter (32 query rows of one 64-dim chunk) per CTA
      if (kBwdCluster == 4 &&
          (!make_tmap_3d(&tq32, p.q, p.d, p.nq, p.S, p.d, p.ldq, 64, 1, 32, err, errlen) ||
           !make_tmap_3d(&tdo32, p.dout, p.d, p.nq, p.S, p.d, p.ldo_grad, 64, 1, 32, err, errlen)))
        return cudaErrorInvalidValue;
      cudaLaunchKernelEx(&cfg, attn_bwd_q64_kernel<false, false, true>, kBwdCluster == 4 ? tq32 : tq64, tk, tv,
                         kBwdCluster == 4 ? tdo32 : tdo64, tdq64, a);
    } else attn_bwd_q64_kernel<false><<<grid, kThreads, Q64Cfg::SMEM, stream>>>(tq64, tk, tv, tdo64, tdq64, a);
    count_launches(1);
    e = cudaGetLastError();
    if (e != cudaSuccess) snprintf(err, errlen, "attn_bwd_q64 launch: %s", cudaGetErrorString(e));
    if (a.dbg) {
      long long h[16];
      cudaMemcpyAsync(h, a.dbg, sizeof h, cudaMemcpyDeviceToHost, stream);
      cudaStreamSynchronize(stream);
      fprintf(stderr,
              "[attn_bwd_q64 timeline CTA(0,0) N=%lld 64-query tiles, cycles] mma: wait_dS %lld wait_Q %lld "
              "wait_dQdrain %lld wait_dO %lld total %lld | WG0: wait_SdP %lld E %lld | WG1: wait_SdP %lld E %lld | "
              "drain: wait_dQ %lld\n",
              h[10], h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9]);
    }
    return e;
  }
  if (p.d == 128) {
    const cudaError_t attr = set_smem_attr((const void*)attn_bwd_kernel<128, false>, BwdCfg<128>::SMEM) == cudaSuccess
                                 ? set_smem_attr((const void*)attn_bwd_kernel<128, false, true>, BwdCfg<128>::SMEM)
                                 : cudaErrorInvalidValue;
    if (attr != cudaSuccess) { snprintf(err, errlen, "attn_bwd attr: %s", cudaGetErrorString(attr)); return attr; }
    const cudaError_t attr2 = set_smem_attr((const void*)attn_bwd_kernel<128, true>, BwdCfg<128>::SMEM);
    if (attr2 != cudaSuccess) { snprintf(err, errlen, "attn_bwd attr: %s", cudaGetErrorString(attr2)); return attr2; }
    if (a.dbg) attn_bwd_kernel<128, true><<<grid, kThreads, BwdCfg<128>::SMEM, stream>>>(tq, tk, tv, tdo, tdq, a);
    else if (a.dq_sem) attn_bwd_kernel<128, false, true><<<grid, kThreads, BwdCfg<128>::SMEM, stream>>>(tq, tk, tv, tdo, tdq, a);
    else attn_bwd_kernel<128, false><<<grid, kThreads, BwdCfg<128>::SMEM, stream>>>(tq, tk, tv, tdo, tdq, a);
    count_launches(1);
  } else {
    const cudaError_t attr = set_smem_attr((const void*)attn_bwd_kernel<64, false>, BwdCfg<64>::SMEM) == cudaSuccess
                                 ? set_smem_attr((const void*)attn_bwd_kernel<64, false, true>, BwdCfg<64>::SMEM)
                                 : cudaErrorInvalidValue;
    if (attr != cudaSuccess) { snprintf(err, errlen, "attn_bwd attr: %s", cudaGetErrorString(attr)); return attr; }
    if (a.dq_sem) attn_bwd_kernel<64, false, true><<<grid, kThreads, BwdCfg<64>::SMEM, stream>>>(tq, tk, tv, tdo, tdq, a);
    else attn_bwd_kernel<64, false><<<grid, kThreads, BwdCfg<64>::SMEM, stream>>>(tq, tk, tv, tdo, tdq, a);
    count_launches(1);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) snprintf(err, errlen, "attn_bwd launch: %s", cudaGetErrorString(e));
  if (a.dbg) {
    long long h[16];
    cudaMemcpyAsync(h, a.dbg, sizeof h, cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    fprintf(stderr,
            "[attn_bwd timeline CTA(0,0) N=%lld cycles] softmax: bar %lld wait_sdp %lld E %lld (wait_dsempty %lld) | "
            "drain: wait_dq %lld drain %lld | mma: wait_ds %lld issue_dV_dQ %lld wait_q %lld wait_dqempty %lld wait_do %lld | "
            "E: ld %lld math %lld store %lld wait_st %lld\n",
            h[10], h[0], h[1], h[2], h[11], h[3], h[4], h[5], h[6], h[7], h[8], h[9], h[12], h[13], h[14], h[15]);
  }
  return e;
}

}  // namespace upipe
