// Causal GQA flash-attention forward for sm_100a.
//
// One CTA owns two consecutive 128-row query tiles (A, B) of one local head and
// streams the KV tiles of the head's KV group through shared memory (TMA, 128B
// swizzle). Warp roles (384 threads; setmaxnreg: softmax 200 registers, others 56):
//   warps 0-3  softmax for tile A  (thread = one query row: the 32x32b TMEM load
//              gives each thread a whole S row, so row max / row sum are
//              thread-local and need no shuffles)
//   warps 4-7  softmax for tile B
//   warp 8     TMA producer (Q once, then K and V per KV tile)
//   warp 9     MMA issuer: S = Q K^T into TMEM, O += P V with P (bf16) from shared memory
//   warps 10-11 idle (complete the third warpgroup for setmaxnreg)
// TMEM (512 columns): S_A | S_B | O_A | O_B (d = 128). P (bf16) goes to shared memory, so S(it+1) of
// a tile is issued as soon as its softmax has read S(it) into registers and only PV(it) waits for the
// softmax; the tensor core alternates between the tiles' S and PV work (ping-pong).
// Online softmax in the exp2 domain with the log2(e)/sqrt(d) scale folded into
// one FFMA; O is rescaled only when the running max grows by more than 8 (2^8
// headroom in fp32/bf16), which is exact: l and O always share the reference max.
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace upipe {
namespace {

using namespace dev;

struct FwdArgs {
  __nv_bfloat16* o;
  float* o32;        // non-null: O written in fp32 here instead (ring-hybrid partials, merged by LSE)
  float* lse;
  long long S, ldo, ldo32, ld_lse;
  int nq, nkv, causal, n_pairs;
  int pair_heads;    // PAIR launch with clusters of two query heads of one KV group (same query tiles) instead of
                     // two adjacent query-tile pairs of one head
  float scale_log2;  // log2(e) / sqrt(d)
  long long* dbg;    // UPIPE_FWD_TIMELINE=1: per-role cycle totals of CTA (0, 0)
  __nv_bfloat16* oseg[kMaxSeg];   // N2 (noseg > 0): row q of O -> oseg[q / oseg_rows] + (q % oseg_rows) * ldo
  long long oseg_rows;
  int noseg;
};

// Cycle counters of the per-role timeline; compiled out unless the timeline variant is launched.
template <bool TL>
__device__ __forceinline__ long long tick() { if constexpr (TL) return clock64(); else return 0; }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

#ifndef UPIPE_FWD_POLY_EVERY
// exp pairs j with j % N == N - 1 use the FMA-pipe polynomial (0: none). Under the power cap at 128K
// (profiles/r02_ab_fwd_poly*.txt): N = 8 114.5 ms of attn fwd per bench step, 4: 117.0, all MUFU 120.8, 3: 121.5,
// 2: 134.5 (round 1 chose 4 from short 32K runs)
#define UPIPE_FWD_POLY_EVERY 8
#endif

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

template <int D>
struct FwdCfg {
  static constexpr int TILE = 128;
  static constexpr int QBYTES = TILE * D * 2;       // one 128 x D bf16 tile
  static constexpr int PBYTES = TILE * TILE * 2;    // one 128 x 128 bf16 P tile
  // K single-buffered (K(it+1) has the whole previous iteration to land: S is issued early), V
  // double-buffered (PV(it) is the late consumer and V(it+1) is needed right after it)
  static constexpr int V_STAGES = 2;
  static constexpr int OFF_QA = 0;
  static constexpr int OFF_QB = QBYTES;
  static constexpr int OFF_K = 2 * QBYTES;
  static constexpr int OFF_V = OFF_K + QBYTES;
  static constexpr int OFF_PA = OFF_V + V_STAGES * QBYTES;   // P_A, P_B: bf16, K-major 128B-swizzled (A of PV)
  static constexpr int OFF_PB = OFF_PA + PBYTES;
  static constexpr int OFF_BAR = OFF_PB + PBYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr uint32_t TM_SA = 0, TM_SB = 128, TM_OA = 256, TM_OB = 256 + D;
  static_assert(SMEM <= 232448, "shared memory");
};

// PAIR (UPIPE_FWD_PAIR): clusters of two CTAs on adjacent query-tile pairs of one head stream the same KV
// tiles (the longer pair's range; the shorter one's extra tiles are fully masked for its tile B), each CTA
// loading one 64-dimension half of every K / V tile with a TMA multicast to both: half the L2 -> SM K/V traffic.
template <int D, bool TL, bool PAIR = false>
__global__ void __launch_bounds__(384, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const FwdArgs a) {
  using C = FwdCfg<D>;
  constexpr int NCH = D / 64;  // 64-wide column chunks of a head
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = bars + 2;
  uint64_t* v_full = bars + 3;                    // [V_STAGES]
  uint64_t* v_empty = bars + 5;                   // [V_STAGES]
  uint64_t* s_full = bars + 7;                    // [2] tile A/B: S(it) in TMEM
  uint64_t* s_free = bars + 9;                    // [2] the softmax has read S(it) into registers
  uint64_t* p_full = bars + 11;                   // [2] P(it) in smem and O rescaled
  uint64_t* o_full = bars + 13;                   // [2] PV(it) done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int warp = warp_id(), lane = lane_id();
  const int pair = a.n_pairs - 1 - blockIdx.x;    // longest (causal) work first (PAIR: -1 = padding CTA)
  const int head = blockIdx.y;
  const int kvh = head / (a.nq / a.nkv);
  const int qt0 = 2 * pair;                       // query tile index of A (B = qt0 + 1)
  const int ntiles_kv = (int)((a.S + 127) / 128);
  const uint32_t crank = PAIR ? cluster_ctarank() : 0;
  const int qt_long = PAIR && !a.pair_heads ? 2 * (a.n_pairs - 1 - (int)(blockIdx.x & ~1u)) : qt0;   // the cluster's longer pair
  const int nA = a.causal ? min(qt0 + 1, ntiles_kv) : ntiles_kv;
  const int nB = a.causal ? min(qt_long + 2, ntiles_kv) : ntiles_kv;   // PAIR: the KV stream both CTAs share

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    mbar_init(k_full, 1); mbar_init(k_empty, PAIR ? 2 : 1);   // PAIR: released by both CTAs
    for (int s = 0; s < C::V_STAGES; ++s) {
      mbar_init(&v_full[s], 1); mbar_init(&v_empty[s], PAIR ? 2 : 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1); mbar_init(&s_free[t], 128); mbar_init(&p_full[t], 128); mbar_init(&o_full[t], 1);
    }
    fence_barrier_init();
    tmem_slot[1] = smem_u32(smem);
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();                      // the peer's barriers exist before any multicast lands in them
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 8) regs_dec<56>();      // warpgroup 2 (TMA, MMA, 2 idle warps) gives registers to softmax
  if (warp == 8) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      mbar_arrive_expect_tx(q_full, 2 * C::QBYTES);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        tma_load_3d(smem + C::OFF_QA + c * 16384, &tmQ, q_full, c * 64, head, qt0 * 128);
        tma_load_3d(smem + C::OFF_QB + c * 16384, &tmQ, q_full, c * 64, head, qt0 * 128 + 128);
      }
      for (int it = 0; it < nB; ++it) {
        mbar_wait(k_empty, (it & 1) ^ 1);
        mbar_arrive_expect_tx(k_full, C::QBYTES);
        if (PAIR) {                                 // this CTA's 64-dimension half to both CTAs
          tma_load_3d_mc(smem + C::OFF_K + crank * 16384, &tmK, k_full, crank * 64, kvh, it * 128, 0x3);
        } else {
#pragma unroll
          for (int c = 0; c < NCH; ++c)
            tma_load_3d(smem + C::OFF_K + c * 16384, &tmK, k_full, c * 64, kvh, it * 128);
        }
        const int sv = it % C::V_STAGES;
        mbar_wait(&v_empty[sv], ((it / C::V_STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&v_full[sv], C::QBYTES);
        if (PAIR) {
          tma_load_3d_mc(smem + C::OFF_V + sv * C::QBYTES + crank * 16384, &tmV, &v_full[sv], crank * 64, kvh, it * 128,
                         0x3);
        } else {
#pragma unroll
          for (int c = 0; c < NCH; ++c)
            tma_load_3d(smem + C::OFF_V + sv * C::QBYTES + c * 16384, &tmV, &v_full[sv], c * 64, kvh, it * 128);
        }
      }
    }
  } else if (warp == 9) {
    {
      // ------------------------------------------------ MMA issuer (whole warp; elect.sync inside the MMA asm)
      constexpr uint32_t idS = idesc_bf16(128, 128, false, false);  // Q (K-major) x K (K-major)
      constexpr uint32_t idO = idesc_bf16(128, D, false, true);     // P (smem, K-major) x V (MN-major)
      // smem base re-read (volatile) per KV tile: descriptors are formed next to each MMA
      // instead of being hoisted into registers (see mma_ss_w in sm100.cuh)
      uint32_t base = ld_volatile_shared_u32(tmem_slot + 1);
      auto issue_S = [&](uint32_t sq, uint32_t sk, uint32_t tm) {
        const uint64_t dq = desc_sw128(sq, 16, 1024), dk = desc_sw128(sk, 16, 1024);
#pragma unroll
        for (int i = 0; i < 4 * NCH; ++i) {
          const uint32_t off = ((i >> 2) * 16384 + (i & 3) * 32) >> 4;
          mma_ss_w(tm, dq + off, dk + off, idS, i != 0);
        }
      };
      // O += P V: A = P in smem (K-major over keys), B = V (MN-major)
      auto issue_PV = [&](uint32_t sp, uint32_t sv, uint32_t tm, bool acc) {
        const uint64_t dp = desc_sw128(sp, 16, 1024), dv = desc_sw128(sv, 16384, 1024);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          mma_ss_w(tm, dp + (((ks >> 2) * 16384 + (ks & 3) * 32) >> 4), dv + (((ks >> 2) * 8192 + (ks & 3) * 2048) >> 4),
                   idO, (acc || ks) ? 1u : 0u);
      };
      long long tw[4] = {0, 0, 0, 0};   // wait s_free (A+B), wait p_full A, wait p_full B, wait K/V
      const long long t_begin = tick<TL>();
      mbar_wait(q_full, 0);
      mbar_wait(k_full, 0);
      tc_fence_after();
      issue_S(base + C::OFF_QA, base + C::OFF_K, tmem + C::TM_SA);
      mma_commit_w(&s_full[0]);
      issue_S(base + C::OFF_QB, base + C::OFF_K, tmem + C::TM_SB);
      mma_commit_w(&s_full[1]);
      if (PAIR) mma_commit_mc_w(k_empty, 0x3);   // K(0) consumed once both S MMAs complete (both CTAs)
      else mma_commit_w(k_empty);
      // Per KV tile: S(it+1) of each tile is issued as soon as its softmax has read S(it) (P lives in
      // smem, so the S columns are free), then PV(it) once P(it) is written. The softmax of a tile
      // therefore never waits for its own PV + S round trip, only for the tensor core's queue.
      for (int it = 0; it < nB; ++it) {
        base = ld_volatile_shared_u32(tmem_slot + 1);
        const bool more = it + 1 < nB;
        long long w0 = tick<TL>();
        if (more) mbar_wait(k_full, (it + 1) & 1);
        tw[3] += tick<TL>() - w0;
        w0 = tick<TL>();
        if (it + 1 < nA) {
          mbar_wait(&s_free[0], it & 1);
          tc_fence_after();
          issue_S(base + C::OFF_QA, base + C::OFF_K, tmem + C::TM_SA);
          mma_commit_w(&s_full[0]);
        }
        if (more) {
          mbar_wait(&s_free[1], it & 1);
          tc_fence_after();
          issue_S(base + C::OFF_QB, base + C::OFF_K, tmem + C::TM_SB);
          mma_commit_w(&s_full[1]);
          if (PAIR) mma_commit_mc_w(k_empty, 0x3);
          else mma_commit_w(k_empty);
        }
        tw[0] += tick<TL>() - w0;
        w0 = tick<TL>();
        const int sv = it % C::V_STAGES;
        mbar_wait(&v_full[sv], (it / C::V_STAGES) & 1);
        tw[3] += tick<TL>() - w0;
        if (it < nA) {
          w0 = tick<TL>();
          mbar_wait(&p_full[0], it & 1);
          tw[1] += tick<TL>() - w0;
          tc_fence_after();
          issue_PV(base + C::OFF_PA, base + C::OFF_V + sv * C::QBYTES, tmem + C::TM_OA, it > 0);
          mma_commit_w(&o_full[0]);
        }
        w0 = tick<TL>();
        mbar_wait(&p_full[1], it & 1);
        tw[2] += tick<TL>() - w0;
        tc_fence_after();
        issue_PV(base + C::OFF_PB, base + C::OFF_V + sv * C::QBYTES, tmem + C::TM_OB, it > 0);
        mma_commit_w(&o_full[1]);
        if (PAIR) mma_commit_mc_w(&v_empty[sv], 0x3);
        else mma_commit_w(&v_empty[sv]);
      }
      if (TL && a.dbg && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0) {
        for (int i = 0; i < 4; ++i) a.dbg[i] = tw[i];
        a.dbg[4] = tick<TL>() - t_begin;
        a.dbg[5] = nB;
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------ softmax warpgroups
    regs_inc<200>();
    const int wg = warp >> 2;                       // 0: tile A, 1: tile B
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const int qt = qt0 + wg;
    const long long q = (long long)qt * 128 + row;  // global query token
    const int n = wg ? nB : nA;
    const uint32_t tS = tmem + (wg ? C::TM_SB : C::TM_SA) + ((uint32_t)(quad * 32) << 16);
    const uint32_t tO = tmem + (wg ? C::TM_OB : C::TM_OA) + ((uint32_t)(quad * 32) << 16);
    const float sl2 = a.scale_log2;
    const uint32_t sP = smem_u32(smem + (wg ? C::OFF_PB : C::OFF_PA));
    float m_ref = -INFINITY, l_run = 0.f;
    long long ts[5] = {0, 0, 0, 0, 0};   // wait S, TMEM load, max+exp+sum, O wait+rescale, P store+arrive
    for (int it = 0; it < n; ++it) {
      const long long e0 = tick<TL>();
      mbar_wait(&s_full[wg], it & 1);
      tc_fence_after();
      const long long e1 = tick<TL>();
      ts[0] += e1 - e0;
      // raw scores (scale folded below): the four 32-column loads are in flight together
      uint32_t sr[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(sr + c * 32));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&s_free[wg]);                     // S(it) is in registers: the MMA warp may issue S(it+1)
      float* s = reinterpret_cast<float*>(sr);
      const long long e2 = tick<TL>();
      ts[1] += e2 - e1;
      const long long key0 = (long long)it * 128;
      const bool edge = a.causal ? (it >= qt) : (key0 + 128 > a.S);   // PAIR: it > qt is fully masked
      if (edge) {
#pragma unroll
        for (int i = 0; i < 128; ++i) {
          const long long key = key0 + i;
          if ((a.causal && key > q) || key >= a.S) s[i] = -INFINITY;
        }
      }
      // row max with 3-input FMNMX3, four independent chains
      float mq[4] = {fmaxf(s[0], s[1]), fmaxf(s[2], s[3]), fmaxf(s[4], s[5]), fmaxf(s[6], s[7])};
#pragma unroll
      for (int i = 8; i < 128; i += 8)
#pragma unroll
        for (int u = 0; u < 4; ++u) mq[u] = fmax3(mq[u], s[i + 2 * u], s[i + 2 * u + 1]);
      float mx = fmax3(mq[0], mq[1], fmaxf(mq[2], mq[3]));
      mx *= sl2;                                       // log2(e)/sqrt(d) > 0: max commutes with the scale
      // lazy rescale: keep the old reference max unless the row max grew by > 8 (log2 units)
      bool rescale = false;
      float alpha = 1.f;
      if (mx > m_ref + 8.f) {
        alpha = ex2(m_ref - mx);                      // 0 when m_ref = -inf
        rescale = it > 0;
        m_ref = mx;
      }
      // p = 2^(s*c - m) on fp32 pairs (FFMA2): pairs j with j % UPIPE_FWD_POLY_EVERY == N - 1 as the
      // polynomial on the FMA pipe, the rest on MUFU (XU also packs P to bf16); row sum with FADD2.
      const uint64_t sl2x2 = f2_pack(sl2, sl2), nm2 = f2_pack(-m_ref, -m_ref);
      uint64_t acc2[4] = {0, 0, 0, 0};
      uint32_t pk[4];
      const long long eo = tick<TL>();
      if (it > 0) {
        mbar_wait(&o_full[wg], (it - 1) & 1);         // PV(it-1) done: P buffer free, O may be rescaled
        tc_fence_after();
      }
      ts[3] += tick<TL>() - eo;                     // (reported as "O": waiting for PV(it-1))
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const uint64_t t = f2_fma(f2_pack(s[2 * j], s[2 * j + 1]), sl2x2, nm2);
        uint64_t e;
        if (UPIPE_FWD_POLY_EVERY > 0 && (j % (UPIPE_FWD_POLY_EVERY > 0 ? UPIPE_FWD_POLY_EVERY : 1)) == UPIPE_FWD_POLY_EVERY - 1) {
          e = ex2_fma2(t);
        } else {
          float t0, t1;
          f2_unpack(t, t0, t1);
          e = f2_pack(ex2(t0), ex2(t1));
        }
        acc2[j & 3] = f2_add(acc2[j & 3], e);
        // P (bf16 pairs) -> smem row `row` (K-major, 128B swizzle: keys [64 kc, 64 kc + 64) in chunk kc),
        // 16 bytes at a time
        float e0, e1;
        f2_unpack(e, e0, e1);
        pk[j & 3] = pack_bf16(e0, e1);
        if ((j & 3) == 3) {
          const int g8 = j >> 2;                       // 8-key group: keys [8 g8, 8 g8 + 8)
          st_shared_v4(sP + (g8 >> 3) * 16384 + sw128_offset(row, (g8 & 7) * 8), pk[0], pk[1], pk[2], pk[3]);
        }
      }
      float s1, s2;
      f2_unpack(f2_add(f2_add(acc2[0], acc2[1]), f2_add(acc2[2], acc2[3])), s1, s2);
      const float sum = s1 + s2;
      l_run = l_run * alpha + sum;
      const long long e3 = tick<TL>();
      ts[2] += e3 - e2;
      // tcgen05.ld/st are warp-collective (.sync.aligned): the rescale decision is per row, so the
      // warp rescales if any of its rows needs it (alpha = 1 for the others). A per-thread branch
      // here diverges the warp and hangs once rows' maxima grow at different tiles.
      if (__any_sync(0xffffffffu, rescale)) {
        if (!rescale) alpha = 1.f;
#pragma unroll
        for (int c = 0; c < D / 16; ++c) {
          uint32_t r[16];
          tmem_ld16(tO + c * 16, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
          tmem_st16(tO + c * 16, r);
        }
        tmem_wait_st();
      }
      const long long e4 = tick<TL>();
      ts[4] += e4 - e3;
      fence_proxy_async_smem();                     // P writes visible to the tensor core (async proxy)
      tc_fence_before();
      mbar_arrive(&p_full[wg]);
      ts[4] += tick<TL>() - e4;
    }
    if (TL && a.dbg && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0 && quad == 0)
      for (int i = 0; i < 5; ++i) a.dbg[6 + wg * 5 + i] = ts[i];
    // ---- epilogue: O / l -> bf16, lse
    if (n > 0) {                                    // PAIR padding CTA: tile A has no key tiles
      mbar_wait(&o_full[wg], (n - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / l_run;
      const bool valid = q >= 0 && q < a.S;
      __nv_bfloat16* orow = (a.noseg ? a.oseg[valid ? q / a.oseg_rows : 0] + (q % a.oseg_rows) * a.ldo : a.o + q * a.ldo) +
                            (long long)head * D;   // N2: straight into the owner rank's O receive block
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tO + c * 32, r);
        tmem_wait_ld();
        if (valid && a.o32) {
          float4* dst = reinterpret_cast<float4*>(a.o32 + q * a.ldo32 + (long long)head * D + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            dst[i] = make_float4(__uint_as_float(r[4 * i + 0]) * inv, __uint_as_float(r[4 * i + 1]) * inv,
                                 __uint_as_float(r[4 * i + 2]) * inv, __uint_as_float(r[4 * i + 3]) * inv);
        } else if (valid) {
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(pack_bf16(__uint_as_float(r[8 * i + 0]) * inv, __uint_as_float(r[8 * i + 1]) * inv),
                                pack_bf16(__uint_as_float(r[8 * i + 2]) * inv, __uint_as_float(r[8 * i + 3]) * inv),
                                pack_bf16(__uint_as_float(r[8 * i + 4]) * inv, __uint_as_float(r[8 * i + 5]) * inv),
                                pack_bf16(__uint_as_float(r[8 * i + 6]) * inv, __uint_as_float(r[8 * i + 7]) * inv));
        }
      }
      if (valid) a.lse[(long long)head * a.ld_lse + q] = (m_ref + __log2f(l_run)) * 0.69314718055994531f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
  if (PAIR) cluster_sync();                      // no CTA leaves while its peer may still multicast into it
}

}  // namespace

cudaError_t attn_fwd_run(const AttnFwdProblem& p, cudaStream_t stream, char* err, size_t errlen) {
  if (p.S <= 0 || p.nq <= 0) return cudaSuccess;
  if ((p.d != 64 && p.d != 128) || p.nkv <= 0 || p.nq % p.nkv) {
    snprintf(err, errlen, "attn_fwd: unsupported head_dim %d or head counts %d/%d", p.d, p.nq, p.nkv);
    return cudaErrorInvalidValue;
  }
  CUtensorMap tq, tk, tv;
  // 3-D views {d, heads, S}: head stride d elements, token stride ld
  if (!make_tmap_3d(&tq, p.q, p.d, p.nq, p.S, p.d, p.ldq, 64, 1, 128, err, errlen)) return cudaErrorInvalidValue;
  if (!make_tmap_3d(&tk, p.k, p.d, p.nkv, p.S, p.d, p.ldkv, 64, 1, 128, err, errlen)) return cudaErrorInvalidValue;
  if (!make_tmap_3d(&tv, p.v, p.d, p.nkv, p.S, p.d, p.ldkv, 64, 1, 128, err, errlen)) return cudaErrorInvalidValue;
  FwdArgs a;
  a.o = reinterpret_cast<__nv_bfloat16*>(p.o);
  a.noseg = p.o_seg.n;
  a.oseg_rows = p.o_seg.rows > 0 ? p.o_seg.rows : 1;
  for (int i = 0; i < kMaxSeg; ++i) a.oseg[i] = reinterpret_cast<__nv_bfloat16*>(p.o_seg.p[i]);
  if (a.noseg && (p.o32 || p.o_seg.rows <= 0 || p.o_seg.n > kMaxSeg || (p.S + p.o_seg.rows - 1) / p.o_seg.rows > p.o_seg.n)) {
    snprintf(err, errlen, "attn_fwd: segmented O needs bf16 output and segments covering S");
    return cudaErrorInvalidValue;
  }
  a.o32 = p.o32;
  a.lse = p.lse;
  a.S = p.S;
  a.ldo = p.ldo;
  a.ldo32 = p.ldo32;
  a.ld_lse = p.ld_lse;
  a.nq = p.nq;
  a.nkv = p.nkv;
  a.causal = p.causal;
  const int ntiles = (int)((p.S + 127) / 128);
  a.n_pairs = (ntiles + 1) / 2;
  a.scale_log2 = 1.4426950408889634f / sqrtf((float)p.d);
  dim3 grid(a.n_pairs, p.nq);
  // UPIPE_FWD_TIMELINE=1: per-role cycle breakdown of CTA (0,0), printed to stderr after the launch
  static long long* dbg_dev = nullptr;
  const char* tlenv = getenv("UPIPE_FWD_TIMELINE");
  a.dbg = nullptr;
  if (tlenv && tlenv[0] == '1') {
    if (!dbg_dev) cudaMalloc(&dbg_dev, 32 * sizeof(long long));
    cudaMemsetAsync(dbg_dev, 0, 32 * sizeof(long long), stream);
    a.dbg = dbg_dev;
  }
  cudaError_t e;
  auto go = [&](auto kern, int smem) -> cudaError_t {
    cudaError_t at = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (at != cudaSuccess) { snprintf(err, errlen, "attn_fwd attr: %s", cudaGetErrorString(at)); return at; }
    kern<<<grid, 384, smem, stream>>>(tq, tk, tv, a);
    count_launches(1);
    return cudaSuccess;
  };
  // PAIR: clusters of two CTAs (an odd pair count gets one padding CTA, fully masked, storing nothing)
  auto go_pair = [&](auto kern, int smem) -> cudaError_t {
    cudaError_t at = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (at != cudaSuccess) { snprintf(err, errlen, "attn_fwd attr: %s", cudaGetErrorString(at)); return at; }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute la[1];
    cfg.gridDim = a.pair_heads ? dim3((unsigned)a.n_pairs, (unsigned)p.nq) : dim3((unsigned)((a.n_pairs + 1) & ~1), (unsigned)p.nq);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    la[0].id = cudaLaunchAttributeClusterDimension;
    la[0].val.clusterDim.x = a.pair_heads ? 1 : 2;
    la[0].val.clusterDim.y = a.pair_heads ? 2 : 1;
    la[0].val.clusterDim.z = 1;
    cfg.attrs = la;
    cfg.numAttrs = 1;
    const cudaError_t le = cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, a);
    count_launches(1);
    return le;
  };
  // UPIPE_FWD_PAIR=1 / 0 forces the CTA-pair launch on / off. Default: pairs when the launch has >= 4 query heads
  // (grids of >= 4 x 512 CTAs at 128K) (A/B at 128K on one box, profiles/r02_ab_fwd_pair.txt: nq/nkv 8/2 1235 -> 1248
  // TFLOP/s, attn fwd 117.1 -> 116.4 ms per bench step; nq/nkv 1/1 1328 -> 1113 TFLOP/s, so not there)
  static const int pair_env = [] {
    const char* v = getenv("UPIPE_FWD_PAIR");
    return v ? (v[0] == '1' ? 1 : v[0] == '2' ? 2 : 0) : -1;
  }();
  const int G = p.nq / p.nkv;
  // UPIPE_FWD_PAIR=2: clusters of two query heads of one KV group (needs an even group size)
  a.pair_heads = pair_env == 2 && G % 2 == 0 ? 1 : 0;
  const bool use_pair = pair_env < 0 ? p.nq >= 4 : (pair_env == 1 || a.pair_heads);
  if (p.d == 128 && !a.dbg && use_pair) e = go_pair(attn_fwd_kernel<128, false, true>, FwdCfg<128>::SMEM);
  else if (p.d == 128) e = a.dbg ? go(attn_fwd_kernel<128, true>, FwdCfg<128>::SMEM) : go(attn_fwd_kernel<128, false>, FwdCfg<128>::SMEM);
  else e = go(attn_fwd_kernel<64, false>, FwdCfg<64>::SMEM);
  if (e != cudaSuccess) return e;
  e = cudaGetLastError();
  if (e != cudaSuccess) snprintf(err, errlen, "attn_fwd launch: %s", cudaGetErrorString(e));
  if (a.dbg) {
    long long h[32];
    cudaMemcpyAsync(h, a.dbg, sizeof h, cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    fprintf(stderr,
            "[attn_fwd timeline CTA(0,0) nB=%lld total %lld cycles] mma: wait_pA %lld wait_pB %lld wait_K %lld wait_V %lld | "
            "softmax A: wait_S %lld ld %lld math %lld O %lld store %lld | B: wait_S %lld ld %lld math %lld O %lld store %lld\n",
            h[5], h[4], h[0], h[1], h[2], h[3], h[6], h[7], h[8], h[9], h[10], h[11], h[12], h[13], h[14], h[15]);
  }
  return e;
}

}  // namespace upipe
