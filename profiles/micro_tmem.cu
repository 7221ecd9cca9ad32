// Microbenchmark: tcgen05.ld (32x32b.x32) throughput per SM and MUFU/F2FP issue cost on B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2602_21196_b200/csrc micro_tmem.cu -o micro_tmem
#include <cstdio>
#include "sm100.cuh"
using namespace upipe::dev;

template <int WARPS>
__global__ void tmem_ld_bw(long long* out, int iters) {
  __shared__ uint32_t slot;
  if (warp_id() == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot + ((uint32_t)((warp_id() & 3) * 32) << 16);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[32];
    tmem_ld32(tm + ((i * 32 + (warp_id() >> 2) * 128) & 511), r);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 32; ++j) acc ^= r[j];
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678) out[1000] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(slot);
}

// 8 independent dependency chains per thread: ex2(ex2(...)) or cvt(cvt(...)); no other instructions
__global__ void xu_cost(long long* out, int iters, int mode) {
  float v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = threadIdx.x * 1e-4f - j * 1e-3f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (mode == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[j]));
      } else {
        uint32_t u;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(u) : "f"(v[j]));
        v[j] = __uint_as_float(u);
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += v[j];
  if (s == 1234.5f) out[1000] = 1;
}

int main() {
  long long* d;
  cudaMalloc(&d, 2000 * 8);
  long long h[148];
  const int iters = 4096;
  tmem_ld_bw<4><<<148, 128>>>(d, iters);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  printf("tmem ld 4 warps: %.1f B/clk/SM\n", 4.0 * 32 * 32 * 4 * iters / h[0]);
  tmem_ld_bw<8><<<148, 256>>>(d, iters);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  printf("tmem ld 8 warps: %.1f B/clk/SM\n", 8.0 * 32 * 32 * 4 * iters / h[0]);
  tmem_ld_bw<16><<<148, 512>>>(d, iters);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  printf("tmem ld 16 warps: %.1f B/clk/SM\n", 16.0 * 32 * 32 * 4 * iters / h[0]);
  for (int mode = 0; mode < 2; ++mode) {
    xu_cost<<<148, 512>>>(d, iters, mode);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
    printf("%s: %.2f lane-ops/clk/SM\n", mode ? "F2FP bf16x2 (cvt.rn.bf16x2.f32)" : "MUFU ex2", 512.0 * 8 * iters / h[0]);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
