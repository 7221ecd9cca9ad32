// Microbenchmark + layout probe for tcgen05.mma.cta_group::2 (CTA pairs) on B200, for the attention backward's
// operand shapes: cycles per K = 16 MMA step for M = 256 (128 rows per CTA) with N = 64 / 128 (SS and TS), and
// M = 128 (64 rows per CTA), against cta_group::1 M = 128, N = 64 / 128; and the TMEM placement of the M = 128
// pair accumulator (which lanes / columns of which CTA hold D[m][n]).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2602_21196_b200/csrc micro_pair.cu -o micro_pair
#include <cstdio>
#include <cstdlib>
#include "sm100.cuh"
using namespace upipe::dev;

__device__ __forceinline__ void mma_ts_pair_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_pair1_w(uint64_t* bar) {   // arrive on this CTA's barrier only
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)1)
      : "memory");
}

// mode: 0 pair M256 N64 SS, 1 pair M256 N128 SS, 2 pair M128 N64 SS, 3 pair M256 N128 TS, 4 pair M256 N256 SS,
//       5 pair M128 N128 SS
__global__ void __launch_bounds__(128, 1) pair_rate(long long* out, int iters, int mode, int nacc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = warp_id();
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) tmem_alloc_pair<512>(&slot);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tm = slot;
  const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
  const uint32_t crank = cluster_ctarank();
  if (warp == 0 && crank == 0) {
    const uint32_t M = (mode == 2 || mode == 5) ? 128 : 256;
    const uint32_t N = (mode == 0 || mode == 2) ? 64 : mode == 4 ? 256 : 128;
    const uint32_t id = idesc_bf16(M, N, false, false);
    const uint64_t da = desc_sw128(sa, 16, 1024), db = desc_sw128(sb, 16, 1024);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t off = ((k >> 2) * 16384 + (k & 3) * 32) >> 4;
        const uint32_t dst = tm + (k % nacc) * (N > 64 ? 128 : 64);   // nacc independent accumulators, interleaved
        if (mode == 3) mma_ts_pair_w(dst, tm + 256 + k * 8, db + off, id, (it | k) >= nacc);
        else mma_ss_pair_w(dst, da + off, db + off, id, (it | k) >= nacc);
      }
    }
    mma_commit_pair1_w(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (lane_id() == 0) out[blockIdx.x / 2] = t1 - t0;
  }
  if (threadIdx.x == 0) {
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    out[1024 + blockIdx.x] = sm;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc_pair<512>(tm);
}


__device__ __forceinline__ void mma_pair_plain(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_pair_mask(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  const uint32_t z = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(z)
      : "memory");
}
// variant 1: elect outside, plain asm; 2: the same with the disable-output-lane mask operand; M256 N128 SS
__global__ void __launch_bounds__(128, 1) pair_variant(long long* out, int iters, int variant) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = warp_id();
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) tmem_alloc_pair<512>(&slot);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tm = slot;
  const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
  const uint32_t crank = cluster_ctarank();
  if (warp == 0 && crank == 0) {
    const uint32_t id = idesc_bf16(256, 128, false, false);
    const uint64_t da = desc_sw128(sa, 16, 1024), db = desc_sw128(sb, 16, 1024);
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t off = ((k >> 2) * 16384 + (k & 3) * 32) >> 4;
          if (variant == 1) mma_pair_plain(tm, da + off, db + off, id, (it | k) != 0);
          else mma_pair_mask(tm, da + off, db + off, id, (it | k) != 0);
        }
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   ::"r"(smem_u32(&bar)), "h"((uint16_t)1) : "memory");
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (lane_id() == 0) out[blockIdx.x / 2] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc_pair<512>(tm);
}

// cta_group::1 reference rates (mode 0: N64, 1: N128), launched in the same 2-CTA clusters
__global__ void __launch_bounds__(128, 1) single_rate(long long* out, int iters, int mode, int nacc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = warp_id();
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
  if (warp == 0) {
    const uint32_t id = idesc_bf16(128, mode == 0 ? 64 : 128, false, false);
    const uint64_t da = desc_sw128(sa, 16, 1024), db = desc_sw128(sb, 16, 1024);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t off = ((k >> 2) * 16384 + (k & 3) * 32) >> 4;
        mma_ss_w(tm + (k % nacc) * 128, da + off, db + off, id, (it | k) >= nacc);
      }
    }
    if (elect_one()) mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (lane_id() == 0 && (blockIdx.x & 1) == 0) out[blockIdx.x / 2] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

// Layout probe: one pair MMA (M = 128 or 256, N = 64, K = 16) with A[m][0] = m, A[m][1] = 1 and B[n][0] = 1000,
// B[n][1] = n, so D[m][n] = 1000 m + n. CTA c holds A rows [c M/2, (c+1) M/2) and B rows [32 c, 32 c + 32) (the
// cta_group::2 operand split). TMEM is pre-filled with -1; out[c][lane][col] for 128 lanes x 128 columns.
__global__ void __launch_bounds__(128, 1) pair_probe(float* out, int M) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = warp_id(), lane = lane_id();
  const uint32_t crank = cluster_ctarank();
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  __syncthreads();
  __nv_bfloat16* A = reinterpret_cast<__nv_bfloat16*>(smem);
  __nv_bfloat16* B = reinterpret_cast<__nv_bfloat16*>(smem + 32768);
  const int mrows = M / 2;
  if (threadIdx.x < mrows) {
    const int r = threadIdx.x, m = crank * mrows + r;
    A[sw128_offset(r, 0) / 2] = __float2bfloat16((float)m);
    A[sw128_offset(r, 1) / 2] = __float2bfloat16(1.f);
  }
  if (threadIdx.x < 32) {
    const int j = threadIdx.x, n = crank * 32 + j;
    B[sw128_offset(j, 0) / 2] = __float2bfloat16(1000.f);
    B[sw128_offset(j, 1) / 2] = __float2bfloat16((float)n);
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc_pair<512>(&slot);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  {
    uint32_t neg[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) neg[i] = __float_as_uint(-1.f);
    for (int c = 0; c < 128; c += 16) tmem_st16(tm + ((uint32_t)(warp * 32) << 16) + c, neg);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 0 && crank == 0) {
    const uint32_t id = idesc_bf16(M, 64, false, false);
    mma_ss_pair_w(tm, desc_sw128(smem_u32(A), 16, 1024), desc_sw128(smem_u32(B), 16, 1024), id, 0);
    mma_commit_pair_w(&bar, 0x3);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < 128; c += 32) {
    uint32_t r[32];
    tmem_ld32(tm + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i)
      out[((size_t)crank * 128 + warp * 32 + lane) * 128 + c + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc_pair<512>(tm);
}

template <class K, class... Args>
static cudaError_t launch2(K kern, int grid, int smem, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchKernelEx(&cfg, kern, args...);
  return cudaDeviceSynchronize();
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  long long* d;
  cudaMalloc(&d, 2048 * sizeof(long long));
  const int smem = getenv("SMEM_KB") ? atoi(getenv("SMEM_KB")) * 1024 : 65536 + 1024;
  const int iters = 4096;
  auto report = [&](const char* name, double per_sm_flop_per_mma, double floor) {
    long long h[74];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 74; ++i) avg += h[i];
    avg /= 74.0 * iters * 8;
    printf("%-34s %.1f cycles per K16 MMA (per-SM compute floor %.0f), %.0f flop/clk/SM\n", name, avg, floor,
           per_sm_flop_per_mma / avg);
  };
  char nm[96];
  for (int nacc : {1, 2, 4})
  for (int mode = 0; mode < 2; ++mode) {
    cudaError_t e = launch2(single_rate, 148, smem, d, iters, mode, nacc);
    if (e != cudaSuccess) { printf("single %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
    const int N = mode == 0 ? 64 : 128;
    snprintf(nm, sizeof nm, "cta_group::1 M128 N%d SS acc x%d", N, nacc);
    report(nm, 2.0 * 128 * N * 16, 128.0 * N / 256);
  }
  const char* names[] = {"cta_group::2 M256 N64 SS", "cta_group::2 M256 N128 SS", "cta_group::2 M128 N64 SS",
                         "cta_group::2 M256 N128 TS", "cta_group::2 M256 N256 SS", "cta_group::2 M128 N128 SS"};
  for (int nacc : {1, 2, 4})
  for (int mode = 0; mode < 6; ++mode) {
    if (mode == 4 && nacc > 2) continue;
    cudaError_t e = launch2(pair_rate, 148, smem, d, iters, mode, nacc);
    if (e != cudaSuccess) { printf("pair %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
    const int M = (mode == 2 || mode == 5) ? 128 : 256;
    const int N = (mode == 0 || mode == 2) ? 64 : mode == 4 ? 256 : 128;
    snprintf(nm, sizeof nm, "%s acc x%d", names[mode], nacc);
    report(nm, 2.0 * (M / 2) * N * 16, (M / 2.0) * N / 256);
    if (mode == 0 && nacc == 1) {
      long long hs[148];
      cudaMemcpy(hs, d + 1024, sizeof hs, cudaMemcpyDeviceToHost);
      int same_tpc = 0;
      for (int i = 0; i < 74; ++i) same_tpc += (hs[2 * i] >> 1) == (hs[2 * i + 1] >> 1);
      printf("  cluster SM ids: %lld,%lld %lld,%lld %lld,%lld %lld,%lld ... pairs on one TPC (smid>>1 equal): %d / 74\n",
             hs[0], hs[1], hs[2], hs[3], hs[4], hs[5], hs[6], hs[7], same_tpc);
    }
  }
  for (int variant : {1, 2}) {
    cudaError_t e = launch2(pair_variant, 148, smem, d, iters, variant);
    if (e != cudaSuccess) { printf("variant %d: %s\n", variant, cudaGetErrorString(e)); return 1; }
    report(variant == 1 ? "pair M256 N128 SS, elect outside" : "pair M256 N128 SS, with lane mask", 2.0 * 128 * 128 * 16, 64);
  }
  float* dout;
  cudaMalloc(&dout, 2 * 128 * 128 * sizeof(float));
  static float h[2 * 128 * 128];
  for (int M : {128}) {
    cudaError_t e = launch2(pair_probe, 2, smem, dout, M);
    if (e != cudaSuccess) { printf("probe M%d: %s\n", M, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, dout, sizeof h, cudaMemcpyDeviceToHost);
    printf("probe M=%d N=64 (value = 1000 m + n; -1 = untouched):\n", M);
    for (int c = 0; c < 2; ++c) {
      for (int lane : {0, 1, 15, 16, 31, 32, 33, 63, 64, 65, 95, 96, 127}) {
        printf("  cta %d lane %3d:", c, lane);
        for (int col : {0, 1, 2, 31, 32, 33, 63, 64, 127}) {
          const float v = h[(c * 128 + lane) * 128 + col];
          if (v < 0) printf("  [c%d] -", col);
          else printf("  [c%d] m%d,n%d", col, (int)v / 1000, (int)v % 1000);
        }
        printf("\n");
      }
    }
  }
  return 0;
}
