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
};
constexpr int kMaxParts = 3;
struct GemmArgs {
  int M, N, K;
  float alpha;
  int nparts, kind;          // kind: 0 single / K-concatenation, 1 M-concatenation (see GemmGroup)
  int kcum[kMaxParts + 1];   // K-concat: first K index of each part (multiples of BK)
  int mcum[kMaxParts + 1];   // M-concat: first row of each part (multiples of BM)
  DevOpMap a[kMaxParts], b[kMaxParts];
  DevOut c[kMaxParts];
};

__device__ __forceinline__ int map_outer(const DevOpMap& m, int i, int k) {
  return m.o_base + (i / m.o_len) * m.o_istride + i % m.o_len + (k / m.k_len) * m.o_kstride;
}
__device__ __forceinline__ int map_k(const DevOpMap& m, int i, int k) {
  return m.k_base + (k / m.k_len) * m.k_kstride + k % m.k_len + (i / m.o_len) * m.k_istride;
}

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int GRANULE_BYTES = 64 * 64 * 2;  // one TMA box: 64 x 64 bf16
constexpr int RING_BYTES = 192 * 1024;

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = RING_BYTES / STAGE_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(192, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB0,
                const __grid_constant__ CUtensorMap tmB1, const __grid_constant__ CUtensorMap tmB2, const GemmArgs g) {
  // Grouped forms (GemmGroup): K-concatenation sums the products of up to three (A, B) pairs
  // into one accumulator (one epilogue pass); M-concatenation stacks up to three A operands
  // (own output maps) against one B. The part of a k-block / tile selects the tensor maps.
  // Persistent: CTA b processes tiles b, b + gridDim.x, ... (N fastest, so CTAs running at the
  // same time share the A row block through L2). Two TMEM accumulators: the epilogue of tile i
  // overlaps the main loop of tile i+1.
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* acc_full = empty + C::STAGES;   // [2]
  uint64_t* acc_empty = acc_full + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const int ntn = (g.N + BN - 1) / BN;
  const int ntiles = ntn * ((g.M + BM - 1) / BM);
  const int nk = (g.K + BK - 1) / BK;

  auto mapA = [&](int p) { return p == 0 ? &tmA0 : (p == 1 ? &tmA1 : &tmA2); };
  auto mapB = [&](int p) { return p == 0 ? &tmB0 : (p == 1 ? &tmB1 : &tmB2); };
  auto mpart = [&](int m0) {            // M-concat part of a tile
    int p = 0;
    if (g.kind == 1)
      while (p + 1 < g.nparts && m0 >= g.mcum[p + 1]) ++p;
    return p;
  };
  if (warp == 0 && lane == 0) {
    for (int p = 0; p < g.nparts; ++p) {
      tma_prefetch(mapA(p));
      tma_prefetch(mapB(p));
    }
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<2 * BN>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int m0 = (t / ntn) * BM, n0 = (t % ntn) * BN;
        const int pm = mpart(m0);
        const int ml0 = m0 - (g.kind == 1 ? g.mcum[pm] : 0);
        int pk = 0;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = ring + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + C::A_BYTES;
          if (g.kind == 0)
            while (pk + 1 < g.nparts && kb * BK >= g.kcum[pk + 1]) ++pk;
          const int k0 = kb * BK - (g.kind == 0 ? g.kcum[pk] : 0);
          const int pa = g.kind == 1 ? pm : pk, pb = g.kind == 1 ? 0 : pk;
          const CUtensorMap* tA = mapA(pa);
          const CUtensorMap* tB = mapB(pb);
          const DevOpMap& am = g.a[pa];
          const DevOpMap& bm = g.b[pb];
          mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
#pragma unroll
          for (int c = 0; c < BM / 64; ++c) {
            const int i = ml0 + c * 64;
            const int oc = map_outer(am, i, k0), kc = map_k(am, i, k0);
            if (A_MN) tma_load_2d(sa + c * GRANULE_BYTES, tA, &full[stage], oc, kc);
            else      tma_load_2d(sa + c * GRANULE_BYTES, tA, &full[stage], kc, oc);
          }
#pragma unroll
          for (int c = 0; c < BN / 64; ++c) {
            const int i = n0 + c * 64;
            const int oc = map_outer(bm, i, k0), kc = map_k(bm, i, k0);
            if (B_MN) tma_load_2d(sb + c * GRANULE_BYTES, tB, &full[stage], oc, kc);
            else      tma_load_2d(sb + c * GRANULE_BYTES, tB, &full[stage], kc, oc);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    {
      // ---------------- MMA issuer (whole warp; elect.sync inside the MMA asm, see mma_ss_w)
      constexpr uint32_t idesc = idesc_bf16(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int i = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int ab = i & 1;
        mbar_wait(&acc_empty[ab], ((i >> 1) & 1) ^ 1);     // the epilogue has drained this accumulator
        tc_fence_after();
        const uint32_t acc = tmem + ab * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(ring + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t da = A_MN ? desc_sw128(sa + kk * 2048, GRANULE_BYTES, 1024) : desc_sw128(sa + kk * 32, 16, 1024);
            const uint64_t db = B_MN ? desc_sw128(sb + kk * 2048, GRANULE_BYTES, 1024) : desc_sw128(sb + kk * 32, 16, 1024);
            mma_ss_w(acc, da, db, idesc, (kb | kk) != 0);
          }
          mma_commit_w(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit_w(&acc_full[ab]);
      }
    }
  } else {
    // ---------------- epilogue warps 2..5: TMEM lane quadrant = warp % 4
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    int i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int ab = i & 1;
      const int m0 = (t / ntn) * BM, n0 = (t % ntn) * BN;
      const int pc = mpart(m0);
      const DevOut& oc_ = g.c[pc];
      const int m = m0 + row;
      const int ml = m - (g.kind == 1 ? g.mcum[pc] : 0);
      mbar_wait(&acc_full[ab], (i >> 1) & 1);
      tc_fence_after();
      const bool mvalid = m < g.M;
      const long long mseg = mvalid ? ml / oc_.m_len : 0, min_ = mvalid ? ml % oc_.m_len : 0;
#pragma unroll 1
      for (int c32 = 0; c32 < BN / 32; ++c32) {
        uint32_t r[32];
        tmem_ld32(tmem + ab * BN + ((uint32_t)(quad * 32) << 16) + c32 * 32, r);
        tmem_wait_ld();
        const int n = n0 + c32 * 32;
        if (!mvalid || n >= g.N) continue;
        const long long nseg = n / oc_.n_len, nin = n % oc_.n_len;
        const long long orow = oc_.r_base + mseg * oc_.r_mstride + min_ + nseg * oc_.r_nstride;
        const long long ocol = oc_.c_base + nseg * oc_.c_nstride + nin + mseg * oc_.c_mstride;
        float v[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(r[q]) * g.alpha;
        if (oc_.epi == (int)Epi::kStoreBF16) {
          uint4* dst = reinterpret_cast<uint4*>(oc_.bf16 + orow * oc_.ld_bf16 + ocol);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            dst[q] = make_uint4(pack_bf16(v[8 * q + 0], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                                pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
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
      mbar_arrive(&acc_empty[ab]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<2 * BN>(tmem);
  }
}

DevOpMap to_dev(const OperandMap& m) {
  return DevOpMap{(int)m.o_base, (int)m.o_len, (int)m.o_istride, (int)m.o_kstride,
                  (int)m.k_base, (int)m.k_len, (int)m.k_kstride, (int)m.k_istride};
}

template <int BN, bool A_MN, bool B_MN>
cudaError_t launch(const CUtensorMap* ta, const CUtensorMap* tb, const GemmArgs& args, cudaStream_t s) {
  using C = Cfg<BN>;
  auto kern = gemm_kernel<BN, A_MN, B_MN>;
  static const cudaError_t attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (attr != cudaSuccess) return attr;
  static const int num_sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const int ntiles = ((args.N + BN - 1) / BN) * ((args.M + BM - 1) / BM);
  dim3 grid(ntiles < num_sms ? ntiles : num_sms);
  kern<<<grid, 192, C::SMEM, s>>>(ta[0], ta[1], ta[2], tb[0], tb[1], tb[2], args);
  count_launches(1);
  return cudaGetLastError();
}

template <int BN>
cudaError_t dispatch_major(bool amn, bool bmn, const CUtensorMap* ta, const CUtensorMap* tb, const GemmArgs& a,
                           cudaStream_t s) {
  if (!amn && !bmn) return launch<BN, false, false>(ta, tb, a, s);
  if (!amn && bmn) return launch<BN, false, true>(ta, tb, a, s);
  if (amn && !bmn) return launch<BN, true, false>(ta, tb, a, s);
  return launch<BN, true, true>(ta, tb, a, s);
}

bool seg_ok(int64_t len) { return len % 64 == 0 && len > 0; }

DevOut to_dev(const OutMap& c) {
  return DevOut{reinterpret_cast<float*>(c.out_f32), reinterpret_cast<__nv_bfloat16*>(c.out_bf16), c.ld_f32, c.ld_bf16,
                c.r_base, c.m_len, c.r_mstride, c.r_nstride, c.c_base, c.n_len, c.c_nstride, c.c_mstride, (int)c.epi};
}

}  // namespace

cudaError_t gemm_run_group(const GemmProblem* parts, int n, GemmGroup kind, cudaStream_t stream, char* err,
                           size_t errlen) {
  if (n < 1 || n > kMaxParts) {
    snprintf(err, errlen, "gemm: %d parts (1..%d)", n, kMaxParts);
    return cudaErrorInvalidValue;
  }
  const GemmProblem& p0 = parts[0];
  int64_t M = p0.M, K = p0.K;
  for (int i = 1; i < n; ++i) {
    const GemmProblem& pi = parts[i];
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
  args.kind = kind == GemmGroup::kMConcat ? 1 : 0;
  CUtensorMap ta[kMaxParts], tb[kMaxParts];
  int64_t kc = 0, mc = 0;
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
    if (!make_tmap_2d(&ta[i], pi.a.ptr, pi.a.inner, pi.a.outer, pi.a.ld, 64, 64, err, errlen)) return cudaErrorInvalidValue;
    if (!make_tmap_2d(&tb[i], pi.b.ptr, pi.b.inner, pi.b.outer, pi.b.ld, 64, 64, err, errlen)) return cudaErrorInvalidValue;
    args.a[i] = to_dev(pi.a);
    args.b[i] = to_dev(pi.b);
    args.c[i] = to_dev(pi.c);
    args.kcum[i] = (int)kc;
    args.mcum[i] = (int)mc;
    if (i < n) {
      kc += pi.K;
      mc += pi.M;
    }
  }
  args.kcum[kMaxParts] = (int)kc;
  args.mcum[kMaxParts] = (int)mc;
  cudaError_t e;
  if (bn == 256) e = dispatch_major<256>(p0.a.mn_major, p0.b.mn_major, ta, tb, args, stream);
  else if (bn == 128) e = dispatch_major<128>(p0.a.mn_major, p0.b.mn_major, ta, tb, args, stream);
  else e = dispatch_major<64>(p0.a.mn_major, p0.b.mn_major, ta, tb, args, stream);
  if (e != cudaSuccess) snprintf(err, errlen, "gemm launch: %s", cudaGetErrorString(e));
  return e;
}

cudaError_t gemm_run(const GemmProblem& p, cudaStream_t stream, char* err, size_t errlen) {
  return gemm_run_group(&p, 1, GemmGroup::kKConcat, stream, err, errlen);
}

}  // namespace upipe
