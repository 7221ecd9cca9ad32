// Microbenchmark: issue cost of the elementwise instructions the attention kernels mix, per SM
// sub-partition (SMSP), 16 warps per CTA (4 per SMSP), 8 independent chains per thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 micro_pipes.cu -o micro_pipes
#include <cstdint>
#include <cstdio>

template <int MODE>
__global__ void __launch_bounds__(512, 1) pipe_cost(long long* out, int iters, float seed) {
  float v[8];
  uint64_t w[8];
  uint32_t u[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    v[j] = seed * (threadIdx.x + 1) - j * 1e-3f;
    asm("mov.b64 %0, {%1, %1};" : "=l"(w[j]) : "f"(v[j]));
    u[j] = __float_as_uint(v[j]);
  }
  const uint64_t c2 = w[0];
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(v[j]) : "f"(seed));
      if (MODE == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(w[j]) : "l"(c2));
      if (MODE == 2) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[j]));
      if (MODE == 3) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(u[j]) : "f"(__uint_as_float(u[j])));
      if (MODE == 4) asm volatile("mad.lo.u32 %0, %0, 8388608, %0;" : "+r"(u[j]));
      if (MODE == 5) asm volatile("prmt.b32 %0, %0, %0, 0x7632;" : "+r"(u[j]));
      if (MODE == 6) asm volatile("add.u32 %0, %0, 32768;" : "+r"(u[j]));
      if (MODE == 7) asm volatile("max.f32 %0, %0, %1, %0;" : "+f"(v[j]) : "f"(seed));
      if (MODE == 8) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(w[j]) : "l"(c2));
      if (MODE == 9) asm volatile("max.f32 %0, %0, %1;" : "+f"(v[j]) : "f"(seed));
      // mixes: one MUFU.EX2 with 4 FFMA2 (10: pipes overlap -> 8 cycles; serialised -> 16), with 8 FFMA (11),
      // with 4 F2FP (12)
      if (MODE == 10) {
        if (j == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[j]));
        else if (j <= 4) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(w[j]) : "l"(c2));
      }
      if (MODE == 11) {
        if (j == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[j]));
        else asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(v[j]) : "f"(seed));
      }
      if (MODE == 12) {
        if (j == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[j]));
        else if (j <= 4) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(u[j]) : "f"(__uint_as_float(u[j])));
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += v[j] + __uint_as_float(u[j]) + __uint_as_float((uint32_t)w[j]);
  if (s == 1234.5f) out[1000] = 1;
}

template <int MODE>
void run(const char* name, long long* d) {
  const int iters = 4096;
  pipe_cost<MODE><<<148, 512>>>(d, iters, 1e-7f);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  // per SMSP: 4 warps x iters x 8 instructions
  const double per = avg / (4.0 * iters * 8);
  printf("%-28s %.2f cycles per warp-instruction per SMSP (%.1f lanes/clk/SMSP)\n", name, per, 32.0 / per);
}

int main() {
  long long* d;
  cudaMalloc(&d, 2000 * sizeof(long long));
  run<0>("FFMA", d);
  run<1>("FFMA2 (f32x2)", d);
  run<8>("FADD2 (f32x2)", d);
  run<2>("MUFU.EX2", d);
  run<3>("F2FP bf16x2 pack", d);
  run<4>("IMAD", d);
  run<5>("PRMT", d);
  run<6>("IADD", d);
  run<7>("FMNMX3", d);
  run<9>("FMNMX", d);
  // for the mixes the printed number is cycles per 8-instruction group / 8
  run<10>("mix MUFU + 4 FFMA2 (/8)", d);
  run<11>("mix MUFU + 7 FFMA (/8)", d);
  run<12>("mix MUFU + 4 F2FP (/8)", d);
  return 0;
}
