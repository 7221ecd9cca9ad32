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
struct GemmArgs {
  int M, N, K;
  float alpha;
  DevOpMap a, b;
  DevOut c;
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
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const GemmArgs g) {
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

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
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
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = ring + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + C::A_BYTES;
          const int k0 = kb * BK;
          mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
#pragma unroll
          for (int c = 0; c < BM / 64; ++c) {
            const int i = m0 + c * 64;
            const int oc = map_outer(g.a, i, k0), kc = map_k(g.a, i, k0);
            if (A_MN) tma_load_2d(sa + c * GRANULE_BYTES, &tmA, &full[stage], oc, kc);
            else      tma_load_2d(sa + c * GRANULE_BYTES, &tmA, &full[stage], kc, oc);
          }
#pragma unroll
          for (int c = 0; c < BN / 64; ++c) {
            const int i = n0 + c * 64;
            const int oc = map_outer(g.b, i, k0), kc = map_k(g.b, i, k0);
            if (B_MN) tma_load_2d(sb + c * GRANULE_BYTES, &tmB, &full[stage], oc, kc);
            else      tma_load_2d(sb + c * GRANULE_BYTES, &tmB, &full[stage], kc, oc);
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
      const int m = m0 + row;
      mbar_wait(&acc_full[ab], (i >> 1) & 1);
      tc_fence_after();
      const bool mvalid = m < g.M;
      const long long mseg = mvalid ? m / g.c.m_len : 0, min_ = mvalid ? m % g.c.m_len : 0;
#pragma unroll 1
      for (int c32 = 0; c32 < BN / 32; ++c32) {
        uint32_t r[32];
        tmem_ld32(tmem + ab * BN + ((uint32_t)(quad * 32) << 16) + c32 * 32, r);
        tmem_wait_ld();
        const int n = n0 + c32 * 32;
        if (!mvalid || n >= g.N) continue;
        const long long nseg = n / g.c.n_len, nin = n % g.c.n_len;
        const long long orow = g.c.r_base + mseg * g.c.r_mstride + min_ + nseg * g.c.r_nstride;
        const long long ocol = g.c.c_base + nseg * g.c.c_nstride + nin + mseg * g.c.c_mstride;
        float v[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(r[q]) * g.alpha;
        if (g.c.epi == (int)Epi::kStoreBF16) {
          uint4* dst = reinterpret_cast<uint4*>(g.c.bf16 + orow * g.c.ld_bf16 + ocol);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            dst[q] = make_uint4(pack_bf16(v[8 * q + 0], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                                pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
        } else {
          float4* dst = reinterpret_cast<float4*>(g.c.f32 + orow * g.c.ld_f32 + ocol);
          if (g.c.epi != (int)Epi::kStoreF32) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 o = dst[q];
              v[4 * q + 0] += o.x; v[4 * q + 1] += o.y; v[4 * q + 2] += o.z; v[4 * q + 3] += o.w;
            }
          }
          if (g.c.epi == (int)Epi::kAccF32ToBF16) {
            uint4* d2 = reinterpret_cast<uint4*>(g.c.bf16 + orow * g.c.ld_bf16 + ocol);
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
cudaError_t launch(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& args, cudaStream_t s) {
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
  kern<<<grid, 192, C::SMEM, s>>>(ta, tb, args);
  count_launches(1);
  return cudaGetLastError();
}

template <int BN>
cudaError_t dispatch_major(bool amn, bool bmn, const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a,
                           cudaStream_t s) {
  if (!amn && !bmn) return launch<BN, false, false>(ta, tb, a, s);
  if (!amn && bmn) return launch<BN, false, true>(ta, tb, a, s);
  if (amn && !bmn) return launch<BN, true, false>(ta, tb, a, s);
  return launch<BN, true, true>(ta, tb, a, s);
}

bool seg_ok(int64_t len) { return len % 64 == 0 && len > 0; }

}  // namespace

cudaError_t gemm_run(const GemmProblem& p, cudaStream_t stream, char* err, size_t errlen) {
  if (p.M <= 0 || p.N <= 0 || p.K <= 0) return cudaSuccess;
  if (p.N % 64) {
    snprintf(err, errlen, "gemm: N=%lld not a multiple of 64", (long long)p.N);
    return cudaErrorInvalidValue;
  }
  for (const OperandMap* m : {&p.a, &p.b}) {
    if (!seg_ok(m->o_len) || !seg_ok(m->k_len)) {
      snprintf(err, errlen, "gemm: operand segment lengths must be multiples of 64");
      return cudaErrorInvalidValue;
    }
  }
  if (!seg_ok(p.c.n_len) || p.c.m_len <= 0) {
    snprintf(err, errlen, "gemm: output segment lengths invalid");
    return cudaErrorInvalidValue;
  }
  // Tile width: the widest of 256/128/64 that stays inside one B-outer and one output segment.
  int bn = 256;
  while (bn > 64 && ((p.b.o_len % bn) || (p.c.n_len % bn) || (p.N % bn))) bn >>= 1;
  CUtensorMap ta, tb;
  if (!make_tmap_2d(&ta, p.a.ptr, p.a.inner, p.a.outer, p.a.ld, 64, 64, err, errlen)) return cudaErrorInvalidValue;
  if (!make_tmap_2d(&tb, p.b.ptr, p.b.inner, p.b.outer, p.b.ld, 64, 64, err, errlen)) return cudaErrorInvalidValue;
  GemmArgs args;
  args.M = (int)p.M;
  args.N = (int)p.N;
  args.K = (int)p.K;
  args.alpha = p.alpha;
  args.a = to_dev(p.a);
  args.b = to_dev(p.b);
  args.c = DevOut{reinterpret_cast<float*>(p.c.out_f32), reinterpret_cast<__nv_bfloat16*>(p.c.out_bf16),
                  p.c.ld_f32, p.c.ld_bf16, p.c.r_base, p.c.m_len, p.c.r_mstride, p.c.r_nstride,
                  p.c.c_base, p.c.n_len, p.c.c_nstride, p.c.c_mstride, (int)p.c.epi};
  cudaError_t e;
  if (bn == 256) e = dispatch_major<256>(p.a.mn_major, p.b.mn_major, ta, tb, args, stream);
  else if (bn == 128) e = dispatch_major<128>(p.a.mn_major, p.b.mn_major, ta, tb, args, stream);
  else e = dispatch_major<64>(p.a.mn_major, p.b.mn_major, ta, tb, args, stream);
  if (e != cudaSuccess) snprintf(err, errlen, "gemm launch: %s", cudaGetErrorString(e));
  return e;
}

}  // namespace upipe
