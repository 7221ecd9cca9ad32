// Microbenchmark: tcgen05.mma kind::f16 cycles per instruction (K = 16) on B200, one CTA per SM,
// for the operand forms the attention kernels use, optionally with other warps streaming
// STS.128 into shared memory (the softmax / dQ-staging traffic of the backward kernel).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2602_21196_b200/csrc micro_mma.cu -o micro_mma
#include <cstdio>
#include "sm100.cuh"
using namespace upipe::dev;

// mode 0: SS M128 N128, both K-major      mode 1: SS M128 N256
// mode 2: TS M128 N128 (A from TMEM)      mode 3: SS M128 N128, B MN-major (dK/dQ form)
// mode 4: SS N128 alternating two accumulators (TMEM cols 0 / 128)   mode 5: TS N128 alternating
// mode 6: SS N64 alternating two accumulators
// mode 7: SS N128, K-loop fully unrolled (descriptor offsets are immediates)
// mode 8: as 7 but issued by the whole warp with elect.sync inside the asm (no compiler ELECT loop)
// mode 9: as 8 with N = 64 (half query tiles of the backward)
// sts_warps: warps 1..sts_warps store 16 B per lane per instruction into a separate smem region
__global__ void __launch_bounds__(384, 1) mma_rate(long long* out, int iters, int mode, int sts_warps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ int stop;
  const int warp = warp_id();
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); stop = 0; }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 65536);
  if (warp == 0 && mode == 12) {
    // mode 12: the 64-query backward's per-tile MMA sequence, back to back (no waits): dV += P^T dO (4 x TS N128,
    // B MN-major), dQ^T = K^T dS (8 x SS N64, both MN-major), dK += dS^T Q (4 x SS N128, B MN-major), S (8 x SS N64),
    // dP (8 x SS N64); TMEM as in the kernel (S 0 | dP 64 | dV 256 | dK 384); "cycles/MMA" = cycles per tile / 32
    const uint32_t id_sp = idesc_bf16(128, 64, false, false), id_kmn = idesc_bf16(128, 128, false, true),
                   id_dq = idesc_bf16(128, 64, true, true);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint64_t db_do = desc_sw128(sb, 8192, 1024), da_k = desc_sw128(sa, 16384, 1024), db_ds = desc_sw128(sb, 8192, 1024);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) mma_ts_w(tm + 256, tm + ks * 8, db_do + ks * (2048 >> 4), id_kmn, 1);
#pragma unroll
      for (int i = 0; i < 8; ++i) mma_ss_w(tm + 64, da_k + i * (2048 >> 4), db_ds + i * (2048 >> 4), id_dq, i != 0);
      const uint64_t da_ds = desc_sw128(sa, 16, 1024), db_q = desc_sw128(sb, 8192, 1024);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) mma_ss_w(tm + 384, da_ds + ((ks * 32) >> 4), db_q + ks * (2048 >> 4), id_kmn, 1);
      const uint64_t da = desc_sw128(sa, 16, 1024), db = desc_sw128(sb, 16, 1024);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        mma_ss_w(tm, da + (((i >> 2) * 16384 + (i & 3) * 32) >> 4), db + (((i >> 2) * 8192 + (i & 3) * 32) >> 4), id_sp, i != 0);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        mma_ss_w(tm + 64, da + (((i >> 2) * 16384 + (i & 3) * 32) >> 4), db + (((i >> 2) * 8192 + (i & 3) * 32) >> 4), id_sp, i != 0);
    }
    if (elect_one()) mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (lane_id() == 0) out[blockIdx.x] = (t1 - t0) / 4;   // report per 8 MMAs: the harness divides by iters * 8
    if (lane_id() == 0) stop = 1;
  } else if (warp == 0 && (mode == 10 || mode == 11)) {
    // mode 10: TS N128 warp-issued, unrolled (A from TMEM columns 256+, D at column 0; the dV / dK form);
    // mode 11: TS N128 with B MN-major (exactly the backward's dV: B = dO MN-major)
    const uint32_t id = idesc_bf16(128, 128, false, mode == 11);
    const uint64_t db = mode == 11 ? desc_sw128(sb, 8192, 1024) : desc_sw128(sb, 16, 1024);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t off = mode == 11 ? (k * 2048) >> 4 : ((k >> 2) * 16384 + (k & 3) * 32) >> 4;
        mma_ts_w(tm, tm + 256 + k * 8, db + off, id, (it | k) != 0);
      }
    }
    if (elect_one()) mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (lane_id() == 0) out[blockIdx.x] = t1 - t0;
    if (lane_id() == 0) stop = 1;
  } else if (warp == 0 && (mode == 8 || mode == 9)) {
    const uint32_t id = idesc_bf16(128, mode == 9 ? 64 : 128, false, false);
    const uint64_t da = desc_sw128(sa, 16, 1024), db = desc_sw128(sb, 16, 1024);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t off = ((k >> 2) * 16384 + (k & 3) * 32) >> 4;
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
            "l"(da + off), "l"(db + off), "r"(id), "r"((it | k) != 0 ? 1 : 0)
            : "memory");
      }
    }
    if (elect_one()) mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (lane_id() == 0) out[blockIdx.x] = t1 - t0;
    if (lane_id() == 0) stop = 1;
  } else if (warp == 0) {
    if (lane_id() == 0) {
      const uint32_t N = mode == 1 ? 256 : mode == 6 ? 64 : 128;
      const uint32_t id = idesc_bf16(128, N, false, mode == 3);
      const bool alt = mode >= 4;
      const uint64_t da = desc_sw128(sa, 16, 1024);
      const uint64_t db = mode == 3 ? desc_sw128(sb, 16384, 1024) : desc_sw128(sb, 16, 1024);
      long long t0 = clock64();
      if (mode == 7) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t off = ((k >> 2) * 16384 + (k & 3) * 32) >> 4;
            mma_ss(tm, da + off, db + off, id, (it | k) != 0);
          }
        }
        iters = 0;
      }
      for (int it = 0; it < iters; ++it) {
#pragma unroll 1
        for (int k = 0; k < 8; ++k) {
          const uint32_t offa = ((k >> 2) * 16384 + (k & 3) * 32) >> 4;
          const uint32_t offb = mode == 3 ? k * (2048 >> 4) : offa;
          const uint32_t dst = tm + (alt ? (k & 1) * 128 : 0);
          if (mode == 2 || mode == 5)
            mma_ts(dst, tm + 256 + k * 8, db + offb, id, (it | k) > 1);
          else
            mma_ss(dst, da + offa, db + offb, id, (it | k) > 1);
        }
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      long long t1 = clock64();
      out[blockIdx.x] = t1 - t0;
      stop = 1;
    }
  } else if (mode == 12 && warp >= 1 && warp <= 8 && sts_warps > 8) {
    // mode 12 with sts_warps = 16: warps 1..8 stream tcgen05.ld 32x32b.x32 from TMEM (the softmax / drain loads of
    // the backward: ~96 KB per tile there) instead of STS
    volatile int* st = &stop;
    const uint32_t ta = tm + ((uint32_t)((warp & 3) * 32) << 16) + 448;   // a warp reads its sub-partition's lanes
    uint32_t acc = 0;
    while (!*st) {
      uint32_t r[32];
      tmem_ld32(ta, r);
      tmem_wait_ld();
      acc += r[0] ^ r[31];
    }
    if (acc == 0x12345678) stop = 2;
  } else if (warp <= sts_warps && sts_warps <= 8) {
    const uint32_t base = smem_u32(smem + 131072) + ((warp - 1) & 3) * 8192 + lane_id() * 16;
    volatile int* st = &stop;
    uint32_t v = threadIdx.x;
    while (!*st) {
#pragma unroll
      for (int j = 0; j < 16; ++j) st_shared_v4(base + (j & 15) * 512, v, v + 1, v + 2, v + j);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int smem = 131072 + 32768 + 1024;
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"SS N128 K-major", "SS N256 K-major", "TS N128", "SS N128 B MN-major",
                         "SS N128 2 accums", "TS N128 2 accums", "SS N64 2 accums", "SS N128 unrolled",
                         "SS N128 warp-issued", "SS N64 warp-issued", "TS N128 warp-issued", "TS N128 B-MN warp-issued",
                         "bwd tile sequence (x4 = cycles per 64-query tile; floor 1664)"};
  const int iters = 4096;
  for (int sts : {0, 8, 16}) {
    for (int mode = 0; mode < 13; ++mode) {
      mma_rate<<<148, 384, smem>>>(d, iters, mode, sts);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long h[148];
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148.0 * iters * 8;
      const double N = mode == 1 ? 256 : (mode == 6 || mode == 9) ? 64 : 128;
      printf("%-20s sts_warps=%d: %.1f cycles/MMA (floor %.0f), %.0f flop/clk/SM\n", names[mode], sts, avg,
             128 * N / 256, 2.0 * 128 * N * 16 / avg);
    }
  }
  return 0;
}
