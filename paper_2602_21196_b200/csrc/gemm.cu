// tcgen05 GEMM for the UPipe projections.
//
// Persistent CTAs (one per SM) walk 128 x BN output tiles: warp 0 issues TMA loads of 64-wide
// granules into a STAGES-deep shared-memory ring (128B swizzle), warp 1 issues
// tcgen05.mma (M=128, N=BN, K=16) into a TMEM accumulator, warps 2..5 drain TMEM
// with tcgen05.ld (one accumulator row per thread; two accumulators so the epilogue
// of one tile overlaps the next tile's main loop) and run the epilogue
// (bf16 store into the all-to-all send layout, fp32 store, or fp32 accumulate).
// The per-stage head gather of the UPipe schedule is folded into the TMA
// coordinates (see OperandMap in kernels.h), so no pack kernel runs before the
// all-to-all: the projection epilogue writes the send buffer directly.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace upipe {
namespace {

using namespace dev;

struct DevOpMap {
  int o_base, o_len, o_istride, o_kstride;
  int k_base, k_len, k_kstride, k_istride;
};
struct DevOut {
  float* f32;
  __nv_bfloat16* bf16;
  long long ld_f32, ld_bf16;
  long long r_base, m_len, r_mstride, r_nstride;
  long long c_base, n_len, c_nstride, c_mstride;
  int epi;
  RopeRef rope;
};
constexpr int kMaxParts = 3;
struct DevDot {              // RowDot (kernels.h): fused delta of the dO projection, part 0
  const __nv_bfloat16* o;    // null: off
  long long ld_o, col0, col_stride, dst_stride;
  float* dst[kMaxSeg];
  int ld_dst, d;
};
// N2 direct-to-peer bf16 stores of part 0: one 2-D map per destination segment ({col, row}, 64 x 32 boxes)
struct SegMaps {
  CUtensorMap m[kMaxSeg];
};
struct GemmArgs {
  int M, N, K;
  float alpha;
  int nparts, kind;          // kind: 0 single / K-concatenation, 1 M-concatenation (see GemmGroup)
  long long* dbg;            // UPIPE_GEMM_TIMELINE=1: wait/issue cycle totals of CTA 0 (else null)
  int dbg_mode;              // UPIPE_GEMM_TIMELINE=2: no TMA loads (MMA-only rate); 3: no MMAs (TMA-only rate)
  int a_box_g, b_box_g;      // 64-row granules per TMA box (K-major operands: one box per operand tile)
  int c_tma;                 // 1: part 0's fp32 store / accumulate goes through shared memory and TMA
                             //    (bulk tensor store / reduce-add into L2) instead of per-thread global RMW
  int kcum[kMaxParts + 1];   // K-concat: first K index of each part (multiples of BK)
  int mcum[kMaxParts + 1];   // M-concat: first row of each part (multiples of BM)
  int ncum[kMaxParts + 1];   // N-concat: first column of each part (multiples of BN)
  DevOpMap a[kMaxParts], b[kMaxParts];
  DevOut c[kMaxParts];
  DevDot dot;
  __nv_bfloat16* segp[kMaxSeg];   // N2: part 0's bf16 output segment bases (nsegp > 0), see OutMap::seg
  int nsegp;
  int ksplit;                     // split-K: each output tile is computed by ksplit units over K / ksplit and
                                  // ADDED (atomically) into the zero-initialised output (fp32 store epilogues)
};

// fp32 atomic add of 4 consecutive floats (split-K epilogue without a TMA map)
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int GRANULE_BYTES = 64 * 64 * 2;  // one TMA box: 64 x 64 bf16
#ifndef UPIPE_GEMM_RING_KB
#define UPIPE_GEMM_RING_KB 192
#endif
constexpr int RING_BYTES = UPIPE_GEMM_RING_KB * 1024;

template <int BN, bool PAIR = false>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * BK * 2;   // PAIR: this CTA's half of the B tile
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = RING_BYTES / STAGE_BYTES;
  static constexpr int STG = STAGES * STAGE_BYTES;          // two 16 KB epilogue staging boxes (128 rows x 32 fp32)
  static constexpr int SMEM = STG + 32768 + 1024 + 256;
  static_assert(SMEM <= 232448, "shared memory");
};

template <int BN, bool A_MN, bool B_MN, int CL, bool PAIR>
__global__ void __launch_bounds__(192, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB0,
                const __grid_constant__ CUtensorMap tmB1, const __grid_constant__ CUtensorMap tmB2,
                const __grid_constant__ CUtensorMap tmC, const __grid_constant__ SegMaps tmSeg, const GemmArgs g) {
  // Grouped forms (GemmGroup): K-concatenation sums the products of up to three (A, B) pairs
  // into one accumulator (one epilogue pass); M-concatenation stacks up to three A operands
  // (own output maps) against one B. The part of a k-block / tile selects the tensor maps.
  // Persistent: work unit u = (m-block, n-block), N fastest (CTAs running at the same time share
  // the A row block through L2). Two TMEM accumulators: the epilogue of tile i overlaps the main
  // loop of tile i+1.
  // MC (2-CTA clusters): the two CTAs of a cluster take the two 128-row tiles of one 256-row
  // unit with the same n-block; each loads half of the shared B tile and multicasts it to both,
  // so per SM the ring carries A (16 KB) + B/2 (BN*64 B) per k-block instead of A + B. Each
  // CTA's MMA commit frees the stage in both CTAs (empty barriers count 2 arrivals).
  // PAIR (cta_group::2, CL = 2): the two CTAs of a cluster run one M = 256 MMA per k-step; each loads
  // its 128 rows of A and its half of B (no multicast) into its own ring, both loads completing on
  // the leader's full barrier; the leader issues the MMAs, its commits free the stage in both CTAs and
  // mark both CTAs' accumulators full; both epilogues release the accumulator to the leader. Per SM
  // the ring carries A + B/2 per k-block and the tensor pipe works on 128 x BN of a 256 x BN tile.
  // PAIR with CL = 4: two pairs (ranks 0,1 and 2,3) on four consecutive m-blocks of one n-block share
  // the B tile: CTA r loads a quarter of B (its pair-half q = r & 1, quarter p = r >> 1) and multicasts it
  // to itself and CTA r ^ 2 (same half in the other pair); every stage is then written by both pairs,
  // so each pair leader's commit frees it in all four CTAs (empty barriers count 2 arrivals).
  static_assert(!PAIR || CL == 2 || CL == 4, "CTA pairs: clusters of 2 or 4");
  constexpr bool P4 = PAIR && CL == 4;
  // BN = 512 (PAIR only): each CTA owns a 128 x 512 output (the whole TMEM, one accumulator, so the
  // epilogue is not overlapped) computed as two N = 256 pair MMAs per k-step; per SM the ring carries
  // A + 256 B rows per k-block for twice the FLOPs of BN = 256 (L2->SM delivery is the GEMM's limit).
  constexpr bool WIDE = BN > 256;
  static_assert(!WIDE || (PAIR && CL == 2 && BN == 512), "BN = 512 needs CTA pairs");
  constexpr int NMMA = WIDE ? BN / 256 : 1, MMA_N = BN / NMMA;
  constexpr int NACC = WIDE ? 1 : 2;                 // TMEM accumulators (512 columns in total)
  using C = Cfg<BN, PAIR>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STG + 32768);
  uint64_t* empty = full + C::STAGES;
  uint64_t* acc_full = empty + C::STAGES;   // [2]
  uint64_t* acc_empty = acc_full + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const int ntn = (g.N + BN - 1) / BN;
  const int ntm = (g.M + BM - 1) / BM;
  constexpr bool MC = CL > 1;
  // cluster rank r: m-sub-block ms = r & 1 (CL >= 2), n-sub-block ns = r >> 1 (CL == 4)
  const int crank = MC ? (int)cluster_ctarank() : 0;
  const int ms = crank & 1, ns = CL == 4 ? crank >> 1 : 0;
  const int unit0 = blockIdx.x / CL, nunit_step = gridDim.x / CL;
  const int ntn_u = CL == 4 && !P4 ? ntn / 2 : ntn;              // n-units (CL = 4: pairs of n-blocks)
  const int nunits0 = ntn_u * (P4 ? (ntm + 3) / 4 : (MC ? (ntm + 1) / 2 : ntm));
  const int nunits = nunits0 * g.ksplit;          // split-K: unit u = split u / nunits0 of tile-unit u % nunits0
  const int nk = (g.K + BK - 1) / BK;
  auto tile_m = [&](int u) {
    u %= nunits0;
    return P4 ? (u / ntn_u) * 4 + crank : (MC ? (u / ntn_u) * 2 + ms : u / ntn_u);
  };
  auto tile_n = [&](int u) { u %= nunits0; return CL == 4 && !P4 ? (u % ntn_u) * 2 + ns : u % ntn_u; };
  auto kb_begin = [&](int u) { return (int)((long long)(u / nunits0) * nk / g.ksplit); };
  auto kb_end = [&](int u) { return (int)((long long)(u / nunits0 + 1) * nk / g.ksplit); };
  const uint32_t leader = crank & ~1u;                            // PAIR: rank of this CTA's pair leader
  // multicast masks: A to the CTAs sharing this m-block (CL = 4), B to those sharing this n-block;
  // an MMA commit frees the stage in every CTA that writes into this CTA's ring
  const uint16_t maskA = CL == 4 ? (uint16_t)((1u << crank) | (1u << (crank ^ 2))) : 0;
  const uint16_t maskB = CL == 4 ? (uint16_t)((1u << crank) | (1u << (crank ^ 1))) : 0x3;
  const uint16_t maskE = CL == 4 ? (uint16_t)(maskA | maskB) : 0x3;

  auto mapA = [&](int p) { return p == 0 ? &tmA0 : (p == 1 ? &tmA1 : &tmA2); };
  auto mapB = [&](int p) { return p == 0 ? &tmB0 : (p == 1 ? &tmB1 : &tmB2); };
  auto mpart = [&](int m0) {            // M-concat part of a tile
    int p = 0;
    if (g.kind == 1)
      while (p + 1 < g.nparts && m0 >= g.mcum[p + 1]) ++p;
    return p;
  };
  auto npart = [&](int n0) {            // N-concat part of a tile
    int p = 0;
    if (g.kind == 2)
      while (p + 1 < g.nparts && n0 >= g.ncum[p + 1]) ++p;
    return p;
  };
  if (warp == 0 && lane == 0) {
    for (int p = 0; p < g.nparts; ++p) {
      tma_prefetch(mapA(p));
      tma_prefetch(mapB(p));
    }
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], P4 ? 2 : (PAIR ? 1 : (CL == 4 ? 3 : (MC ? 2 : 1))));
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], PAIR ? 256 : 128);   // PAIR: both CTAs' epilogues release the leader's accumulator
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (PAIR) tmem_alloc_pair<NACC * BN>(tmem_slot);
    else tmem_alloc<NACC * BN>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  if (MC) cluster_sync();                  // peer barriers initialised before any multicast arrives
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      long long tl_prod = 0;
      int stage = 0;
      uint32_t phase = 0;
      // TMA coordinates: the i-dependent parts of map_outer / map_k are formed once per tile (and
      // operand part); the k-dependent parts advance incrementally (k / k_len, k % k_len) so the
      // single producer thread does no integer division per k-block.
      constexpr int GA = BM / 64, GB = BN / 64;       // A / B granules (64 rows each)
      constexpr int GB0 = P4 ? GB / 4 : (MC ? GB / 2 : GB);   // B granules this CTA loads (MC: half, P4: quarter)
      constexpr int GA0 = CL == 4 && !P4 ? GA / 2 : GA;       // A granules this CTA loads (CL = 4: its half)
      static_assert(!P4 || GB0 >= 1, "P4 needs BN = 256");
      for (int u = unit0; u < nunits; u += nunit_step) {
        const int mt = tile_m(u);
        const bool valid = mt < ntm;           // MC: the odd last m-block pairs with an empty tile
        const int m0 = mt * BM, n0 = tile_n(u) * BN;
        const int pm = mpart(m0), pn = npart(n0);
        const int ml0 = m0 - (g.kind == 1 ? g.mcum[pm] : 0);
        const int nl0 = n0 - (g.kind == 2 ? g.ncum[pn] : 0);
        const int cb0 = P4 ? ms * (GB / 2) + ns * GB0 : (MC ? ms * GB0 : 0);   // first B granule (tile rows / 64)
        const int cbd = P4 ? ns * GB0 : (PAIR ? 0 : cb0);                        // its granule in this CTA's ring
        const int ca0 = CL == 4 && !P4 ? ns * GA0 : 0;
        int pk = -1, pa = 0, pb = 0;
        int a_out[GA0], a_kb[GA0], b_out[GB0], b_kb[GB0], b_pt[GB0];
        int ka_len = 1, kb_len = 1, kqa_o = 0, kqa_k = 0, kqb_o = 0, kqb_k = 0;
        int kra = 0, krb = 0, kqa = 0, kqb = 0;
        const int kb0 = kb_begin(u), kb1 = kb_end(u);
        for (int kb = kb0; kb < kb1; ++kb) {
          const long long w0 = g.dbg ? clock64() : 0;
          mbar_wait(&empty[stage], phase ^ 1);
          if (g.dbg) tl_prod += clock64() - w0;
          uint8_t* sa = ring + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + C::A_BYTES;
          int npk = pk < 0 ? 0 : pk;
          if (g.kind == 0)
            while (npk + 1 < g.nparts && kb * BK >= g.kcum[npk + 1]) ++npk;
          if (npk != pk) {                     // new tile or new K part: per-(tile, part) constants
            pk = npk;
            pa = g.kind == 1 ? pm : (g.kind == 2 ? 0 : pk);
            pb = g.kind == 1 ? 0 : (g.kind == 2 ? pn : pk);
            const DevOpMap& am = g.a[pa];
            const DevOpMap& bm = g.b[pb];
#pragma unroll
            for (int c = 0; c < GA0; ++c) {
              const int ii = ml0 + (ca0 + c) * 64;
              a_out[c] = am.o_base + (ii / am.o_len) * am.o_istride + ii % am.o_len;
              a_kb[c] = am.k_base + (ii / am.o_len) * am.k_istride;
            }
#pragma unroll
            for (int c = 0; c < GB0; ++c) {
              // WIDE: granule c of this CTA = half ms of MMA (c / 2)'s 256 B rows
              const int ig = (WIDE ? (c >> 1) * (GB / NMMA) + ms * 2 + (c & 1) : cb0 + c) * 64;
              // N-concat: a tile may span parts; each 64-row granule takes its own part's B operand
              const int pg = g.kind == 2 ? npart(n0 + ig) : pb;
              const DevOpMap& bg = g.b[pg];
              const int ii = (g.kind == 2 ? n0 + ig - g.ncum[pg] : nl0 + ig);
              b_pt[c] = pg;
              b_out[c] = bg.o_base + (ii / bg.o_len) * bg.o_istride + ii % bg.o_len;
              b_kb[c] = bg.k_base + (ii / bg.o_len) * bg.k_istride;
            }
            ka_len = am.k_len; kqa_o = am.o_kstride; kqa_k = am.k_kstride;
            kb_len = bm.k_len; kqb_o = bm.o_kstride; kqb_k = bm.k_kstride;
            // k within the part (K-concat offsets are multiples of BK; split-K units start mid-part)
            const int kl = kb * BK - (g.kind == 1 ? 0 : g.kcum[pk]);
            kqa = kl / ka_len; kra = kl % ka_len;
            kqb = kl / kb_len; krb = kl % kb_len;
          }
          const CUtensorMap* tA = mapA(pa);
          const CUtensorMap* tB = mapB(pb);   // N-concat: per granule (below)
          if (g.dbg_mode == 2) {                // timeline experiment: MMA-only
            mbar_arrive(&full[stage]);
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
          const uint32_t full_leader = PAIR ? mapa_shared(&full[stage], leader) : 0;
          if (!PAIR) {
            mbar_arrive_expect_tx(&full[stage], (valid ? C::A_BYTES : 0) + C::B_BYTES);
          } else if (crank == leader) {         // the pair leader expects both CTAs' bytes
            const bool valid1 = tile_m(u) + 1 < ntm;
            mbar_arrive_expect_tx(&full[stage], ((valid ? 1 : 0) + (valid1 ? 1 : 0)) * C::A_BYTES + 2 * C::B_BYTES);
          }
          if (valid) {
#pragma unroll
            for (int c = 0; c < GA0; ++c) {
              if (c % g.a_box_g) continue;       // covered by the previous (multi-granule) box
              const int oc = a_out[c] + kqa * kqa_o, kc = a_kb[c] + kqa * kqa_k + kra;
              uint8_t* dst = sa + (ca0 + c) * GRANULE_BYTES;
              if (PAIR) {
                if (A_MN) tma_load_2d_pair(dst, tA, full_leader, oc, kc);
                else      tma_load_2d_pair(dst, tA, full_leader, kc, oc);
              } else if (CL == 4) {
                if (A_MN) tma_load_2d_mc(dst, tA, &full[stage], oc, kc, maskA);
                else      tma_load_2d_mc(dst, tA, &full[stage], kc, oc, maskA);
              } else {
                if (A_MN) tma_load_2d(dst, tA, &full[stage], oc, kc);
                else      tma_load_2d(dst, tA, &full[stage], kc, oc);
              }
            }
          }
#pragma unroll
          for (int c = 0; c < GB0; ++c) {
            if (c % g.b_box_g) continue;
            if (g.kind == 2) tB = mapB(b_pt[c]);
            const int oc = b_out[c] + kqb * kqb_o, kc = b_kb[c] + kqb * kqb_k + krb;
            uint8_t* dst = sb + (cbd + c) * GRANULE_BYTES;
            if (P4) {                           // to both pairs; each copy completes on its pair leader's barrier
              const uint16_t mk = (uint16_t)((1u << crank) | (1u << (crank ^ 2)));
              if (B_MN) tma_load_2d_pair_mc(dst, tB, &full[stage], oc, kc, mk);
              else      tma_load_2d_pair_mc(dst, tB, &full[stage], kc, oc, mk);
            } else if (PAIR) {
              if (B_MN) tma_load_2d_pair(dst, tB, full_leader, oc, kc);
              else      tma_load_2d_pair(dst, tB, full_leader, kc, oc);
            } else if (MC) {
              if (B_MN) tma_load_2d_mc(dst, tB, &full[stage], oc, kc, maskB);
              else      tma_load_2d_mc(dst, tB, &full[stage], kc, oc, maskB);
            } else {
              if (B_MN) tma_load_2d(dst, tB, &full[stage], oc, kc);
              else      tma_load_2d(dst, tB, &full[stage], kc, oc);
            }
          }
          if ((kra += BK) >= ka_len) { kra = 0; ++kqa; }
          if ((krb += BK) >= kb_len) { krb = 0; ++kqb; }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
      if (g.dbg && blockIdx.x == 0) g.dbg[0] = tl_prod;
    }
  } else if (warp == 1) {
    if (!PAIR || crank == leader) {
      // ---------------- MMA issuer (whole warp; elect.sync inside the MMA asm, see mma_ss_w)
      constexpr uint32_t idesc = idesc_bf16(PAIR ? 2 * BM : BM, MMA_N, A_MN, B_MN);
      long long tl_full = 0, tl_acc = 0;
      const long long t_start = clock64();
      int stage = 0;
      uint32_t phase = 0;
      int i = 0;
      for (int u = unit0; u < nunits; u += nunit_step, ++i) {
        const int ab = i % NACC;
        const long long a0 = g.dbg ? clock64() : 0;
        mbar_wait(&acc_empty[ab], ((i / NACC) & 1) ^ 1);   // the epilogue has drained this accumulator
        if (g.dbg) tl_acc += clock64() - a0;
        tc_fence_after();
        const uint32_t acc = tmem + ab * BN;
        const int kb0 = kb_begin(u), kb1 = kb_end(u);
        for (int kb = kb0; kb < kb1; ++kb) {
          const long long w0 = g.dbg ? clock64() : 0;
          mbar_wait(&full[stage], phase);
          if (g.dbg) tl_full += clock64() - w0;
          tc_fence_after();
          const uint32_t sa = smem_u32(ring + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t da = A_MN ? desc_sw128(sa + kk * 2048, GRANULE_BYTES, 1024) : desc_sw128(sa + kk * 32, 16, 1024);
            const uint64_t db = B_MN ? desc_sw128(sb + kk * 2048, GRANULE_BYTES, 1024) : desc_sw128(sb + kk * 32, 16, 1024);
            if (g.dbg_mode == 3) continue;
            if (PAIR) {
#pragma unroll
              for (int j = 0; j < NMMA; ++j)             // MMA j: TMEM columns [256 j, 256 j + 256), B sub-tile j
                mma_ss_pair_w(acc + j * MMA_N, da, db + ((j * (MMA_N / 2) * BK * 2) >> 4), idesc, (kb != kb0 || kk != 0));
            } else {
              mma_ss_w(acc, da, db, idesc, (kb != kb0 || kk != 0));
            }
          }
          if (PAIR) mma_commit_pair_w(&empty[stage], P4 ? 0xF : 0x3);  // frees the stage where this pair's data lives
          else if (MC) mma_commit_mc_w(&empty[stage], maskE);   // frees the stage in every CTA writing into ours
          else mma_commit_w(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if (PAIR) mma_commit_pair_w(&acc_full[ab], (uint16_t)(0x3u << leader));
        else mma_commit_w(&acc_full[ab]);
      }
      if (g.dbg && blockIdx.x == 0 && lane == 0) {
        g.dbg[1] = tl_full;
        g.dbg[2] = tl_acc;
        g.dbg[3] = clock64() - t_start;
        g.dbg[4] = i;
      }
    }
  } else {
    // ---------------- epilogue warps 2..5: TMEM lane quadrant = warp % 4
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    int i = 0;
    for (int u = unit0; u < nunits; u += nunit_step, ++i) {
      const int ab = i % NACC;
      const int m0 = tile_m(u) * BM, n0 = tile_n(u) * BN;
      const int pc = g.kind == 2 ? npart(n0) : mpart(m0);
      const DevOut& oc_ = g.c[pc];
      const bool seg_out = pc == 0 || g.kind == 2;    // part 0's output map (N-concat: one segmented output)
      const int m = m0 + row;
      const int ml = m - (g.kind == 1 ? g.mcum[pc] : 0);
      mbar_wait(&acc_full[ab], (i / NACC) & 1);
      tc_fence_after();
      const bool mvalid = m < g.M;
      const long long mseg = mvalid ? ml / oc_.m_len : 0, min_ = mvalid ? ml % oc_.m_len : 0;
      if (g.c_tma == 2 && seg_out) {
        // bf16 store through shared memory: each warp stages its 32 rows x 64 columns (128B swizzle,
        // two 4 KB slots) and issues one TMA store per box into the output's 3-D view {col, row, segment}
        // (full-line writes instead of 32 rows x 16 bytes per store instruction). N2: one 2-D map per
        // destination segment (a peer's receive block). RowDot: delta of each head from the rounded values.
        float dot_acc = 0.f;
#pragma unroll 1
        for (int c64 = 0; c64 < BN / 64; ++c64) {
          const int n = n0 + c64 * 64;
          if (n >= g.N) break;                          // uniform across the CTA
          uint32_t r[64];
          tmem_ld32(tmem + ab * BN + ((uint32_t)(quad * 32) << 16) + c64 * 64, *reinterpret_cast<uint32_t(*)[32]>(r));
          tmem_ld32(tmem + ab * BN + ((uint32_t)(quad * 32) << 16) + c64 * 64 + 32,
                    *reinterpret_cast<uint32_t(*)[32]>(r + 32));
          tmem_wait_ld();
          float v[64];
#pragma unroll
          for (int q = 0; q < 64; ++q) v[q] = __uint_as_float(r[q]) * g.alpha;
          const RopeRef& rp = g.kind == 2 ? g.c[npart(n)].rope : oc_.rope;   // N-concat: the box's own part
          if (rp.hi) {
            rope_rotate<16>(v, rp.hi, rp.lo, rp.d, rp.pos0 + m, n % rp.d, 1.f);
            rope_rotate<16>(v + 32, rp.hi, rp.lo, rp.d, rp.pos0 + m, (n + 32) % rp.d, 1.f);
          }
          if (g.dot.o) {
            const long long seg = n / oc_.n_len, nin = n % oc_.n_len;
            if (mvalid) {
              const uint4* orow = reinterpret_cast<const uint4*>(g.dot.o + (long long)ml * g.dot.ld_o + g.dot.col0 +
                                                                 seg * g.dot.col_stride + nin);
#pragma unroll
              for (int j = 0; j < 8; ++j) dot_acc += dot8_rounded(v + 8 * j, orow[j]);
            }
            if ((nin + 64) % g.dot.d == 0) {              // the head's last 64 columns
              float* dd = g.dot.dst_stride ? g.dot.dst[0] + seg * g.dot.dst_stride : g.dot.dst[seg];
              if (mvalid) dd[(long long)ml * g.dot.ld_dst + nin / g.dot.d] = dot_acc;
              dot_acc = 0.f;
            }
          }
          const uint32_t slot = smem_u32(smem + C::STG + quad * 8192 + (c64 & 1) * 4096);
          if (lane == 0) bulk_wait_read1();             // the store that last used this slot has read it
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            st_shared_v4(slot + lane * 128 + ((j ^ (lane & 7)) << 4), pack_bf16(v[8 * j + 0], v[8 * j + 1]),
                         pack_bf16(v[8 * j + 2], v[8 * j + 3]), pack_bf16(v[8 * j + 4], v[8 * j + 5]),
                         pack_bf16(v[8 * j + 6], v[8 * j + 7]));
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const long long seg = n / oc_.n_len, nin = n % oc_.n_len;
            if (g.nsegp) tma_store_2d(&tmSeg.m[seg], smem + C::STG + quad * 8192 + (c64 & 1) * 4096, (int)nin, m0 + quad * 32);
            else tma_store_3d(&tmC, smem + C::STG + quad * 8192 + (c64 & 1) * 4096, (int)nin, m0 + quad * 32, (int)seg);
            bulk_commit();
          }
        }
        tc_fence_before();
        if (PAIR && crank != leader) mbar_arrive_cluster(mapa_shared(&acc_empty[ab], leader));
        else mbar_arrive(&acc_empty[ab]);
        continue;
      }
      float dot_acc = 0.f;
#pragma unroll 1
      for (int c32 = 0; c32 < BN / 32; ++c32) {
        uint32_t r[32];
        tmem_ld32(tmem + ab * BN + ((uint32_t)(quad * 32) << 16) + c32 * 32, r);
        tmem_wait_ld();
        const int n = n0 + c32 * 32;
        if (n >= g.N) continue;                 // uniform across the CTA
        if (g.c_tma == 1 && pc == 0 && (oc_.epi == (int)Epi::kStoreF32 || oc_.epi == (int)Epi::kAccF32)) {
          // fp32 tile column box -> swizzled staging slot -> one TMA store / reduce-add by warp 2 lane 0
          // (L2 performs the accumulation: no global read by the SM, no per-thread RMW latency)
          const bool issuer = warp == 2 && lane == 0;
          uint8_t* slot = smem + C::STG + (c32 & 1) * 16384;
          if (issuer) bulk_wait_read1();      // the op that last used this slot has read it
          named_bar_sync(1, 128);
          const uint32_t sb = smem_u32(slot) + row * 128;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            st_shared_v4(sb + ((j ^ (row & 7)) << 4), __float_as_uint(__uint_as_float(r[4 * j + 0]) * g.alpha),
                         __float_as_uint(__uint_as_float(r[4 * j + 1]) * g.alpha),
                         __float_as_uint(__uint_as_float(r[4 * j + 2]) * g.alpha),
                         __float_as_uint(__uint_as_float(r[4 * j + 3]) * g.alpha));
          fence_proxy_async_smem();
          named_bar_sync(1, 128);
          if (issuer) {
            if (oc_.epi == (int)Epi::kAccF32 || g.ksplit > 1) tma_reduce_add_2d(&tmC, slot, n, m0);
            else tma_store_2d(&tmC, slot, n, m0);
            bulk_commit();
          }
          continue;
        }
        if (!mvalid) continue;
        const long long nseg = n / oc_.n_len, nin = n % oc_.n_len;
        const long long orow = oc_.r_base + mseg * oc_.r_mstride + min_ + nseg * oc_.r_nstride;
        const long long ocol = oc_.c_base + nseg * oc_.c_nstride + nin + mseg * oc_.c_mstride;
        float v[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(r[q]) * g.alpha;
        if (oc_.epi == (int)Epi::kStoreBF16) {
          // RoPE on the projected Q/K (row m = token pos0 + m, columns n.. = head dims n % d..)
          const RopeRef& rp = g.kind == 2 ? g.c[npart(n)].rope : oc_.rope;
          if (rp.hi) rope_rotate<16>(v, rp.hi, rp.lo, rp.d, rp.pos0 + m, n % rp.d, 1.f);
          if (pc == 0 && g.dot.o) {                       // fused row-dot (see the TMA path)
            const uint4* orw = reinterpret_cast<const uint4*>(g.dot.o + (long long)ml * g.dot.ld_o + g.dot.col0 +
                                                              nseg * g.dot.col_stride + nin);
#pragma unroll
            for (int j = 0; j < 4; ++j) dot_acc += dot8_rounded(v + 8 * j, orw[j]);
            if ((nin + 32) % g.dot.d == 0) {
              float* dd = g.dot.dst_stride ? g.dot.dst[0] + nseg * g.dot.dst_stride : g.dot.dst[nseg];
              dd[(long long)ml * g.dot.ld_dst + nin / g.dot.d] = dot_acc;
              dot_acc = 0.f;
            }
          }
          uint4* dst = reinterpret_cast<uint4*>(seg_out && g.nsegp ? g.segp[nseg] + (long long)ml * oc_.ld_bf16 + nin
                                                                     : oc_.bf16 + orow * oc_.ld_bf16 + ocol);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            dst[q] = make_uint4(pack_bf16(v[8 * q + 0], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                                pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
        } else if (g.ksplit > 1) {                     // split-K: atomic adds into the zeroed output
          float* dst = oc_.f32 + orow * oc_.ld_f32 + ocol;
#pragma unroll
          for (int q = 0; q < 8; ++q) red_add_v4(dst + 4 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
          float4* dst = reinterpret_cast<float4*>(oc_.f32 + orow * oc_.ld_f32 + ocol);
          if (oc_.epi != (int)Epi::kStoreF32) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 o = dst[q];
              v[4 * q + 0] += o.x; v[4 * q + 1] += o.y; v[4 * q + 2] += o.z; v[4 * q + 3] += o.w;
            }
          }
          if (oc_.epi == (int)Epi::kAccF32ToBF16) {
            uint4* d2 = reinterpret_cast<uint4*>(oc_.bf16 + orow * oc_.ld_bf16 + ocol);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              d2[q] = make_uint4(pack_bf16(v[8 * q + 0], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                                 pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          }
        }
      }
      tc_fence_before();
      if (PAIR && crank != leader) mbar_arrive_cluster(mapa_shared(&acc_empty[ab], leader));
      else mbar_arrive(&acc_empty[ab]);
    }
    if ((g.c_tma == 1 && warp == 2 && lane == 0) || (g.c_tma == 2 && lane == 0)) bulk_wait0();   // staged boxes written
  }
  tc_fence_before();
  __syncthreads();
  if (MC) cluster_sync();                  // no CTA leaves while its peer may still signal its barriers
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_pair<NACC * BN>(tmem);
    else tmem_dealloc<NACC * BN>(tmem);
  }
}

DevOpMap to_dev(const OperandMap& m) {
  return DevOpMap{(int)m.o_base, (int)m.o_len, (int)m.o_istride, (int)m.o_kstride,
                  (int)m.k_base, (int)m.k_len, (int)m.k_kstride, (int)m.k_istride};
}

template <int BN, bool A_MN, bool B_MN, int CL, bool PAIR>
cudaError_t launch(const CUtensorMap* ta, const CUtensorMap* tb, const CUtensorMap* tc, const SegMaps& sm,
                   const GemmArgs& args, cudaStream_t s) {
  using C = Cfg<BN, PAIR>;
  auto kern = gemm_kernel<BN, A_MN, B_MN, CL, PAIR>;
  const cudaError_t attr = set_smem_attr((const void*)kern, C::SMEM);
  if (attr != cudaSuccess) return attr;
  int dev = 0, num_sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  const int ntn = (args.N + BN - 1) / BN, ntm = (args.M + BM - 1) / BM;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  const int units = PAIR && CL == 4 ? ntn * ((ntm + 3) / 4)
                                    : (CL == 4 ? ntn / 2 : ntn) * (CL > 1 ? (ntm + 1) / 2 : ntm);
  if (CL > 1) {
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  // persistent grid: no more clusters than can be co-resident (clusters must fit inside a GPC, so
  // this can be below num_sms / CL; a second partial wave would double the tail)
  // cached per (kernel, device): occupancy is a property of the device the launch goes to
  static std::mutex mc_mu;
  static std::map<int, int> mc_by_dev;
  int max_clusters = 0;
  {
    std::lock_guard<std::mutex> lk(mc_mu);
    auto it = mc_by_dev.find(dev);
    if (it != mc_by_dev.end()) {
      max_clusters = it->second;
    } else {
      if (CL == 1) {
        max_clusters = num_sms;
      } else {
        int n = 0;
        cudaLaunchConfig_t q = cfg;
        q.gridDim = dim3(CL * (num_sms / CL));
        if (cudaOccupancyMaxActiveClusters(&n, kern, &q) != cudaSuccess || n <= 0) n = num_sms / CL;
        max_clusters = n;
      }
      mc_by_dev[dev] = max_clusters;
    }
  }
  // split-K (args.ksplit == 0: allowed, the outputs are zeroed fp32): a long-K GEMM with fewer tile-units than
  // co-resident clusters (the weight gradients: M x N = 1536 x 4096 over K = S_l) splits K so every cluster
  // works; the first split count whose waves fill >= 90 % of the clusters, K-blocks per split >= 64
  GemmArgs a = args;
  if (a.ksplit == 0) {
    const int nkb = (a.K + BK - 1) / BK;
    int best = 1;
    double best_util = 0.0;
    for (int sk = 1; sk <= 16 && nkb / sk >= 64; ++sk) {
      const long long u = (long long)units * sk;
      const double util = (double)u / ((double)((u + max_clusters - 1) / max_clusters) * max_clusters);
      if (util > best_util + 1e-9) { best_util = util; best = sk; }
      if (util >= 0.9) break;
    }
    a.ksplit = best;
  }
  const int units_all = units * a.ksplit;
  const int clusters = units_all < max_clusters ? units_all : max_clusters;
  cfg.gridDim = dim3(CL * clusters);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta[0], ta[1], ta[2], tb[0], tb[1], tb[2], *tc, sm, a);
  count_launches(1);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int BN, int CL, bool PAIR = false>
cudaError_t dispatch_cl(bool amn, bool bmn, const CUtensorMap* ta, const CUtensorMap* tb, const CUtensorMap* tc,
                        const SegMaps& sm, const GemmArgs& a, cudaStream_t s) {
  if (!amn && !bmn) return launch<BN, false, false, CL, PAIR>(ta, tb, tc, sm, a, s);
  if (!amn && bmn) return launch<BN, false, true, CL, PAIR>(ta, tb, tc, sm, a, s);
  if (amn && !bmn) return launch<BN, true, false, CL, PAIR>(ta, tb, tc, sm, a, s);
  return launch<BN, true, true, CL, PAIR>(ta, tb, tc, sm, a, s);
}

template <int BN>
cudaError_t dispatch_major(bool amn, bool bmn, int cl, const CUtensorMap* ta, const CUtensorMap* tb,
                           const CUtensorMap* tc, const SegMaps& sm, const GemmArgs& a, cudaStream_t s) {
  if constexpr (BN == 512) {
    return dispatch_cl<BN, 2, true>(amn, bmn, ta, tb, tc, sm, a, s);
  } else if constexpr (BN >= 128) {
    if (cl == -2) return dispatch_cl<BN, 2, true>(amn, bmn, ta, tb, tc, sm, a, s);
    if constexpr (BN == 256)
      if (cl == -4) return dispatch_cl<BN, 4, true>(amn, bmn, ta, tb, tc, sm, a, s);
    if (cl == 4) return dispatch_cl<BN, 4>(amn, bmn, ta, tb, tc, sm, a, s);
    if (cl == 2) return dispatch_cl<BN, 2>(amn, bmn, ta, tb, tc, sm, a, s);
    return dispatch_cl<BN, 1>(amn, bmn, ta, tb, tc, sm, a, s);
  } else {
    return dispatch_cl<BN, 1>(amn, bmn, ta, tb, tc, sm, a, s);
  }
}

bool seg_ok(int64_t len) { return len % 64 == 0 && len > 0; }

DevOut to_dev(const OutMap& c) {
  return DevOut{reinterpret_cast<float*>(c.out_f32), reinterpret_cast<__nv_bfloat16*>(c.out_bf16), c.ld_f32, c.ld_bf16,
                c.r_base, c.m_len, c.r_mstride, c.r_nstride, c.c_base, c.n_len, c.c_nstride, c.c_mstride, (int)c.epi,
                c.rope};
}

}  // namespace

cudaError_t gemm_run_group(const GemmProblem* parts, int n, GemmGroup kind, cudaStream_t stream, char* err,
                           size_t errlen) {
  if (n < 1 || n > kMaxParts) {
    snprintf(err, errlen, "gemm: %d parts (1..%d)", n, kMaxParts);
    return cudaErrorInvalidValue;
  }
  GemmProblem pp[kMaxParts];
  for (int i = 0; i < n; ++i) pp[i] = parts[i];
  int ncum[kMaxParts + 1] = {0, 0, 0, 0};
  if (kind == GemmGroup::kNConcat) {
    // [B_0; B_1; ...] against one A: part 0 carries the whole output, the parts' n_len-column segments in
    // order (bf16 stores); the other parts contribute their B operand and their epilogue options (RoPE)
    GemmProblem& q = pp[0];
    q.c.seg = SegPtrs{};
    int64_t ncols = 0;
    for (int i = 0; i < n; ++i) {
      const GemmProblem& pi = parts[i];
      const int64_t nlen = pi.c.n_len < pi.N ? pi.c.n_len : pi.N;
      if (pi.M != q.M || pi.K != q.K || pi.a.ptr != q.a.ptr || pi.b.mn_major != q.b.mn_major ||
          pi.c.epi != Epi::kStoreBF16 || nlen != (q.c.n_len < parts[0].N ? q.c.n_len : parts[0].N) ||
          pi.c.ld_bf16 != q.c.ld_bf16 || pi.N % nlen) {
        snprintf(err, errlen, "gemm N-concat: parts need equal M, K, A, segment width and bf16 stores");
        return cudaErrorInvalidValue;
      }
      for (int64_t j = 0; j < pi.N / nlen; ++j) {
        if (q.c.seg.n >= kMaxSeg) {
          snprintf(err, errlen, "gemm N-concat: more than %d output segments", kMaxSeg);
          return cudaErrorInvalidValue;
        }
        q.c.seg.p[q.c.seg.n++] = pi.c.seg.n ? pi.c.seg.p[j]
                                            : static_cast<char*>(pi.c.out_bf16) + (size_t)(j * pi.c.r_nstride * pi.c.ld_bf16) * 2;
      }
      ncols += pi.N;
      ncum[i + 1] = (int)ncols;
    }
    for (int i = n + 1; i <= kMaxParts; ++i) ncum[i] = (int)ncols;
    q.N = ncols;
    q.c.out_bf16 = nullptr;
    q.c.r_nstride = 0;
    for (int i = 1; i < n; ++i) pp[i].N = ncols;      // the shared tile grid (B maps keep their own extents)
  }
  parts = pp;
  const GemmProblem& p0 = parts[0];
  int64_t M = p0.M, K = p0.K;
  for (int i = 1; i < n; ++i) {
    const GemmProblem& pi = parts[i];
    if (kind == GemmGroup::kNConcat) continue;         // checked above
    if (pi.N != p0.N || pi.a.mn_major != p0.a.mn_major || pi.b.mn_major != p0.b.mn_major) {
      snprintf(err, errlen, "gemm group: parts differ in N or operand majorness");
      return cudaErrorInvalidValue;
    }
    if (kind == GemmGroup::kKConcat) {
      if (pi.M != p0.M || p0.K % BK || parts[i - 1].K % BK) {
        snprintf(err, errlen, "gemm K-concat: parts need equal M and K multiples of %d", BK);
        return cudaErrorInvalidValue;
      }
      K += pi.K;
    } else {
      if (pi.K != p0.K || parts[i - 1].M % BM) {
        snprintf(err, errlen, "gemm M-concat: parts need equal K and M multiples of %d", BM);
        return cudaErrorInvalidValue;
      }
      M += pi.M;
    }
  }
  if (M <= 0 || p0.N <= 0 || K <= 0) return cudaSuccess;
  if (p0.N % 64) {
    snprintf(err, errlen, "gemm: N=%lld not a multiple of 64", (long long)p0.N);
    return cudaErrorInvalidValue;
  }
  // Tile width: the widest of 256/128/64 that stays inside one B-outer and one output segment.
  int bn = 256;
  auto bn_ok = [&](int w) {
    if (p0.N % w) return false;
    if (kind == GemmGroup::kNConcat) {       // tiles may span parts (per-granule B maps, segmented output)
      for (int i = 0; i < n; ++i)
        if (ncum[i] % 64 || parts[i].b.o_len % 64 || parts[i].c.n_len % 64) return false;
      return true;
    }
    for (int i = 0; i < n; ++i)
      if ((parts[i].b.o_len % w) || (parts[i].c.n_len % w)) return false;
    return true;
  };
  while (bn > 64 && !bn_ok(bn)) bn >>= 1;
  GemmArgs args;
  args.M = (int)M;
  args.N = (int)p0.N;
  args.K = (int)K;
  args.alpha = p0.alpha;
  args.nparts = n;
  static long long* dbg_dev = nullptr;
  static const int tl_env = [] {
    const char* e = getenv("UPIPE_GEMM_TIMELINE");
    return e ? atoi(e) : 0;
  }();
  args.dbg = nullptr;
  args.dbg_mode = tl_env;
  if (tl_env) {
    if (!dbg_dev) cudaMalloc(&dbg_dev, 8 * sizeof(long long));
    cudaMemsetAsync(dbg_dev, 0, 8 * sizeof(long long), stream);
    args.dbg = dbg_dev;
  }
  args.kind = kind == GemmGroup::kMConcat ? 1 : (kind == GemmGroup::kNConcat ? 2 : 0);
  for (int i = 0; i <= kMaxParts; ++i) args.ncum[i] = ncum[i];
  // split-K allowed when every part stores fp32 into an output the caller zeroed (OutMap::zeroed)
  bool splittable = true;
  for (int i = 0; i < n; ++i) splittable = splittable && parts[i].c.epi == Epi::kStoreF32 && parts[i].c.zeroed;
  static const int splitk_env = [] {
    const char* e = getenv("UPIPE_GEMM_SPLITK");
    return e ? atoi(e) : 1;
  }();
  args.ksplit = splittable && splitk_env ? 0 : 1;
  // Clusters with operand multicast (UPIPE_GEMM_MC caps the cluster size: 1, 2 or 4; default 4):
  // 2 CTAs share B (two m-blocks, same n-block); 4 CTAs (2 x 2) also share A. Needs BN >= 128 (B, A
  // split into 64-row halves), two or more m-blocks, and for 4 an even number of n-blocks.
  static const int mc_env = [] {
    const char* e = getenv("UPIPE_GEMM_MC");
    return e ? atoi(e) : 4;
  }();
  // UPIPE_GEMM_PAIR=1 (default): CTA pairs (cta_group::2, M = 256 per MMA) instead of multicast clusters
  static const int pair_env = [] {
    const char* e = getenv("UPIPE_GEMM_PAIR");
    return e ? atoi(e) : 1;
  }();
  const int ntn_all = (int)(p0.N / bn);
  int cl = 1;
  if (bn >= 128 && M > BM && mc_env >= 2) cl = (mc_env >= 4 && ntn_all % 2 == 0) ? 4 : 2;
  // UPIPE_GEMM_PAIR=2: two pairs per cluster sharing B by multicast (BN = 256, four or more m-blocks)
  const bool pair = cl > 1 && pair_env;
  // UPIPE_GEMM_WIDE=1 (default): 128 x 512 tiles per CTA (two N = 256 pair MMAs) where N allows
  static const int wide_env = [] {
    const char* e = getenv("UPIPE_GEMM_WIDE");
    return e ? atoi(e) : 1;
  }();
  // ... and only with store epilogues: an fp32 read-modify-write epilogue (dX accumulation) is too long
  // to leave un-overlapped (measured: dX 17.4 -> 21.1 ms per step at 128K with BN = 512)
  bool store_epi = true;
  for (int i = 0; i < n; ++i)
    store_epi = store_epi && (parts[i].c.epi == Epi::kStoreBF16 || parts[i].c.epi == Epi::kStoreF32);
  // ... and only with K long enough to amortise the 128 x 512 tile's un-overlapped epilogue (~9K cycles
  // against 1K per k-block; measured 131072 x 4096 x 1024: 1044 TFLOP/s wide vs cuBLAS 1258)
  // ... and (UPIPE_GEMM_WIDE_DOT=0) not with the fused row-dot, whose epilogue also reads O (A/B)
  static const int wide_dot_env = [] {
    const char* e = getenv("UPIPE_GEMM_WIDE_DOT");
    return e ? atoi(e) : 1;
  }();
  const bool dot_ok = wide_dot_env || !parts[0].c.dot.o;
  if (pair && wide_env && pair_env == 1 && bn == 256 && store_epi && bn_ok(512) && K >= 2048 && dot_ok) bn = 512;
  const bool pair4 = pair && pair_env >= 2 && bn == 256 && M > 3 * BM;
  if (pair) cl = pair4 ? 4 : 2;
  const bool mc = cl > 1;
  // TMA box rows: a K-major operand tile (rows x 64 k) goes in one box when its rows never cross an
  // operand segment (fewer, larger TMA requests); MN-major tiles stay 64 x 64 granules (128B swizzle
  // caps the inner box at 64 elements).
  auto box_g = [&](bool is_a, int rows) {
    int gr = rows / 64;
    if (!is_a && kind == GemmGroup::kNConcat)   // a multi-granule B box must not cross a part boundary
      for (int i = 0; i < n; ++i)
        if (ncum[i] % rows) return 1;
    for (int i = 0; i < n; ++i) {
      const OperandMap& m = is_a ? parts[i].a : parts[i].b;
      if (m.mn_major || (m.o_len < (1 << 30) && m.o_len % rows)) return 1;
    }
    return gr;
  };
  const int a_g = box_g(true, cl == 4 && !pair ? BM / 2 : BM),
            b_g = box_g(false, bn == 512 ? 128 : (pair4 ? bn / 4 : (mc ? bn / 2 : bn)));
  args.a_box_g = a_g;
  args.b_box_g = b_g;
  CUtensorMap ta[kMaxParts], tb[kMaxParts];
  int64_t kc = 0, mrow = 0;
  for (int i = 0; i < kMaxParts; ++i) {
    const GemmProblem& pi = parts[i < n ? i : 0];
    if (i < n) {
      for (const OperandMap* m : {&pi.a, &pi.b}) {
        if (!seg_ok(m->o_len) || !seg_ok(m->k_len)) {
          snprintf(err, errlen, "gemm: operand segment lengths must be multiples of 64");
          return cudaErrorInvalidValue;
        }
      }
      if (!seg_ok(pi.c.n_len) || pi.c.m_len <= 0) {
        snprintf(err, errlen, "gemm: output segment lengths invalid");
        return cudaErrorInvalidValue;
      }
    }
    if (!make_tmap_2d(&ta[i], pi.a.ptr, pi.a.inner, pi.a.outer, pi.a.ld, 64, 64 * a_g, err, errlen)) return cudaErrorInvalidValue;
    if (!make_tmap_2d(&tb[i], pi.b.ptr, pi.b.inner, pi.b.outer, pi.b.ld, 64, 64 * b_g, err, errlen)) return cudaErrorInvalidValue;
    args.a[i] = to_dev(pi.a);
    args.b[i] = to_dev(pi.b);
    args.c[i] = to_dev(pi.c);
    args.kcum[i] = (int)kc;
    args.mcum[i] = (int)mrow;
    if (i < n) {
      kc += pi.K;
      mrow += pi.M;
    }
  }
  args.kcum[kMaxParts] = (int)kc;
  args.mcum[kMaxParts] = (int)mrow;
  // TMA epilogue for part 0's fp32 store / accumulate when its output map is a plain row-major matrix
  // (the dX accumulator, dWo): UPIPE_GEMM_TMA_EPI=0 disables it
  static const int tma_epi_env = [] {
    const char* e = getenv("UPIPE_GEMM_TMA_EPI");
    return e ? atoi(e) : 1;
  }();
  CUtensorMap tc = ta[0];
  args.c_tma = 0;
  {
    const OutMap& c0 = p0.c;
    const bool plain = c0.r_base == 0 && c0.c_base == 0 && c0.m_len >= M && c0.n_len >= p0.N && c0.r_mstride == 0 &&
                       c0.r_nstride == 0 && c0.c_nstride == 0 && c0.c_mstride == 0;
    if (tma_epi_env && kind == GemmGroup::kKConcat && (c0.epi == Epi::kStoreF32 || c0.epi == Epi::kAccF32) && plain &&
        c0.out_f32 && (reinterpret_cast<uintptr_t>(c0.out_f32) & 15) == 0 && c0.ld_f32 % 4 == 0 && p0.alpha == 1.0f) {
      if (!make_tmap_2d_f32(&tc, c0.out_f32, (uint64_t)p0.N, (uint64_t)M, (uint64_t)c0.ld_f32, 32, 128, err, errlen))
        return cudaErrorInvalidValue;
      args.c_tma = 1;
    }
    // bf16 stores (projections into the a2a send layout, the output projection): 3-D view {col within
    // the segment, row, segment} so boxes clip at the segment's last row (ragged S_l)
    static const int tma_bf16_env = [] {
      const char* e = getenv("UPIPE_GEMM_TMA_BF16");
      return e ? atoi(e) : 1;
    }();
    const bool seg_rows_ok = c0.r_mstride == 0 && c0.m_len >= M && c0.r_base == 0 && c0.c_base == 0 &&
                             c0.c_nstride == 0 && c0.c_mstride == 0;
    const int64_t nlen = c0.n_len < p0.N ? c0.n_len : p0.N;
    const int64_t nseg = (p0.N + nlen - 1) / nlen;
    const bool segd = c0.seg.n > 0;           // N2: per-segment destinations (peers' receive blocks)
    if (tma_epi_env && tma_bf16_env && !args.c_tma && kind != GemmGroup::kMConcat && c0.epi == Epi::kStoreBF16 &&
        seg_rows_ok && (segd || (c0.out_bf16 && (reinterpret_cast<uintptr_t>(c0.out_bf16) & 15) == 0)) &&
        c0.ld_bf16 % 8 == 0 && nlen % 64 == 0 && (segd || nseg == 1 || c0.r_nstride >= M)) {
      if (!segd) {
        const int64_t s2 = nseg > 1 ? c0.r_nstride * c0.ld_bf16 : (int64_t)M * c0.ld_bf16;
        if (!make_tmap_3d(&tc, c0.out_bf16, (uint64_t)nlen, (uint64_t)M, (uint64_t)nseg, (uint64_t)c0.ld_bf16,
                          (uint64_t)s2, 64, 32, 1, err, errlen))
          return cudaErrorInvalidValue;
      }
      args.c_tma = 2;
    }
  }
  // N2 direct-to-peer segments and the fused row-dot (part 0 of a single GEMM)
  SegMaps sm;
  std::memset(&sm, 0, sizeof sm);
  args.nsegp = 0;
  std::memset(&args.segp, 0, sizeof args.segp);
  std::memset(&args.dot, 0, sizeof args.dot);
  {
    const OutMap& c0 = p0.c;
    if (c0.seg.n > 0) {
      const int64_t nlen = c0.n_len < p0.N ? c0.n_len : p0.N;
      if ((n != 1 && kind != GemmGroup::kNConcat) || c0.epi != Epi::kStoreBF16 || c0.seg.n > kMaxSeg ||
          c0.seg.n * nlen < p0.N ||
          c0.r_mstride != 0 || c0.m_len < M || c0.r_base != 0 || c0.c_base != 0 || c0.c_nstride != 0 ||
          c0.c_mstride != 0 || c0.ld_bf16 % 8) {
        snprintf(err, errlen, "gemm: segmented (direct-to-peer) output needs a single bf16-store GEMM with "
                              "plain segments covering N (%d segments of %lld columns, N = %lld)",
                 c0.seg.n, (long long)nlen, (long long)p0.N);
        return cudaErrorInvalidValue;
      }
      for (int q = 0; q < c0.seg.n; ++q) {
        if (!c0.seg.p[q] || (reinterpret_cast<uintptr_t>(c0.seg.p[q]) & 15)) {
          snprintf(err, errlen, "gemm: segment %d destination null or not 16-byte aligned", q);
          return cudaErrorInvalidValue;
        }
        args.segp[q] = reinterpret_cast<__nv_bfloat16*>(c0.seg.p[q]);
        if (args.c_tma == 2 &&
            !make_tmap_2d(&sm.m[q], c0.seg.p[q], (uint64_t)nlen, (uint64_t)M, (uint64_t)c0.ld_bf16, 64, 32, err, errlen))
          return cudaErrorInvalidValue;
      }
      args.nsegp = c0.seg.n;
    }
    if (c0.dot.o) {
      const RowDot& r = c0.dot;
      const int w = args.c_tma == 2 ? 64 : 32;          // the epilogue's column chunk
      if (n != 1 || c0.epi != Epi::kStoreBF16 || r.d <= 0 || r.d % w || bn % r.d || c0.n_len % r.d ||
          (reinterpret_cast<uintptr_t>(r.o) & 15) || r.ld_o % 8 || r.col0 % 8 || r.col_stride % 8 || p0.alpha != 1.0f) {
        snprintf(err, errlen, "gemm: fused row-dot needs a single bf16-store GEMM with head-aligned tiles "
                              "(d = %d, BN = %d) and 16-byte aligned O columns", r.d, bn);
        return cudaErrorInvalidValue;
      }
      args.dot.o = reinterpret_cast<const __nv_bfloat16*>(r.o);
      args.dot.ld_o = r.ld_o;
      args.dot.col0 = r.col0;
      args.dot.col_stride = r.col_stride;
      args.dot.dst_stride = r.dst_stride;
      for (int q = 0; q < kMaxSeg; ++q) args.dot.dst[q] = r.dst[q];
      args.dot.ld_dst = r.ld_dst;
      args.dot.d = r.d;
    }
  }
  cudaError_t e;
  const int clk = pair4 ? -4 : (pair ? -2 : cl);
  if (bn == 512) e = dispatch_major<512>(p0.a.mn_major, p0.b.mn_major, clk, ta, tb, &tc, sm, args, stream);
  else if (bn == 256) e = dispatch_major<256>(p0.a.mn_major, p0.b.mn_major, clk, ta, tb, &tc, sm, args, stream);
  else if (bn == 128) e = dispatch_major<128>(p0.a.mn_major, p0.b.mn_major, clk, ta, tb, &tc, sm, args, stream);
  else e = dispatch_major<64>(p0.a.mn_major, p0.b.mn_major, 1, ta, tb, &tc, sm, args, stream);
  if (e != cudaSuccess) snprintf(err, errlen, "gemm launch: %s", cudaGetErrorString(e));
  if (args.dbg) {
    long long h[8];
    cudaMemcpyAsync(h, args.dbg, sizeof h, cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    fprintf(stderr, "[gemm timeline CTA 0] M=%d N=%d K=%d BN=%d mc=%d tiles=%lld: producer wait_empty %lld | mma wait_full %lld "
            "wait_acc_empty %lld total %lld cycles\n", args.M, args.N, args.K, bn, cl, h[4], h[0], h[1], h[2], h[3]);
  }
  return e;
}

cudaError_t gemm_run(const GemmProblem& p, cudaStream_t stream, char* err, size_t errlen) {
  return gemm_run_group(&p, 1, GemmGroup::kKConcat, stream, err, errlen);
}

}  // namespace upipe
