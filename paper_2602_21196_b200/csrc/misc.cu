// HBM-bound helpers of the UPipe path: coalesced, 16-byte vectorised, grid sized
// in multiples of the SM count (148) with grid-stride loops.
//   rowdot      delta = rowsum(dO * O) per (token, head)      (DESIGN A13)
//   cvt         fp32 accumulator -> bf16 (scaled)             (B5 dQ post, F7/B8 finalize)
//   unpack_cols out-a2a receive [C][S_l][qpd d] -> o_saved    (F5)
//   synth_fill  device copy of the counter-based input generator (synth/__init__.py)
//   merge       ring-step combine of two attention partials by their LSE
//   qk_prep     Qwen3 per-head RMSNorm (+ RoPE) of the received Q / K rows
//   norm_bwd    its chain rule fused into the fp32 -> bf16 conversion of dQ / dK (+ d(gamma))
#include <algorithm>
#include <cstdio>

#include "kernels.h"
#include "sm100.cuh"

namespace upipe {
namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t work, int per_block) {
  int64_t b = (work + per_block - 1) / per_block;
  const int64_t cap = 148 * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

// One group of LANES = d/8 threads per (token, head); 8 bf16 per thread per tensor.
template <int LANES>
__global__ void rowdot_kernel(const __nv_bfloat16* __restrict__ dO, long long ld_do,
                              const __nv_bfloat16* __restrict__ O, long long ld_o, float* __restrict__ delta,
                              long long ld_delta, long long rows, int nheads, int d) {
  const long long groups = rows * nheads;
  const int sub = threadIdx.x % LANES;
  long long gidx = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
  const long long gstride = (long long)gridDim.x * blockDim.x / LANES;
  for (; gidx < groups; gidx += gstride) {
    const long long t = gidx / nheads;
    const int j = (int)(gidx % nheads);
    const uint4 a = *reinterpret_cast<const uint4*>(dO + t * ld_do + (long long)j * d + sub * 8);
    const uint4 b = *reinterpret_cast<const uint4*>(O + t * ld_o + (long long)j * d + sub * 8);
    float fa[8], fb[8];
    bf16x8_to_f32(a, fa);
    bf16x8_to_f32(b, fb);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s = fmaf(fa[i], fb[i], s);
#pragma unroll
    for (int off = LANES / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off, LANES);
    if (sub == 0) delta[t * ld_delta + j] = s;
  }
}

// One group of LANES = d/4 threads per (token, head), 4 fp32 per thread. Empty partials (lse = -inf)
// carry weight 0; both empty stays empty.
template <int LANES>
__global__ void merge_kernel(float* __restrict__ o_acc, const float* __restrict__ o_part, long long ld_o,
                             float* __restrict__ lse_acc, const float* __restrict__ lse_part, long long ld_lse,
                             long long rows, int nheads, int d) {
  const long long groups = rows * nheads;
  const int sub = threadIdx.x % LANES;
  long long gidx = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / LANES;
  const long long gstride = (long long)gridDim.x * blockDim.x / LANES;
  for (; gidx < groups; gidx += gstride) {
    const long long t = gidx / nheads;
    const int j = (int)(gidx % nheads);
    const float la = lse_acc[(long long)j * ld_lse + t], lb = lse_part[(long long)j * ld_lse + t];
    const float m = fmaxf(la, lb);
    const float ms = m == -INFINITY ? 0.f : m;
    const float wa = expf(la - ms), wb = expf(lb - ms);
    const float tot = wa + wb;
    const float ca = tot > 0.f ? wa / tot : 0.f, cb = tot > 0.f ? wb / tot : 0.f;
    float4* pa = reinterpret_cast<float4*>(o_acc + t * ld_o + (long long)j * d) + sub;
    const float4 b = *(reinterpret_cast<const float4*>(o_part + t * ld_o + (long long)j * d) + sub);
    const float4 a = *pa;
    *pa = make_float4(ca * a.x + cb * b.x, ca * a.y + cb * b.y, ca * a.z + cb * b.z, ca * a.w + cb * b.w);
    __syncwarp((LANES == 32) ? 0xffffffffu : (((1u << LANES) - 1u) << ((threadIdx.x & 31) / LANES * LANES)));
    if (sub == 0) lse_acc[(long long)j * ld_lse + t] = tot > 0.f ? ms + logf(tot) : -INFINITY;
  }
}

// Destination row r: dst + r * ldd, or (N2, seg.n > 0) the owner rank's receive block seg.p[r / seg.rows].
__device__ __forceinline__ __nv_bfloat16* dst_row(__nv_bfloat16* dst, const SegPtrs& seg, long long r, long long ldd) {
  if (seg.n) return reinterpret_cast<__nv_bfloat16*>(seg.p[r / seg.rows]) + (r % seg.rows) * ldd;
  return dst + r * ldd;
}

__global__ void cvt_kernel(const float* __restrict__ src, long long lds, __nv_bfloat16* __restrict__ dst,
                           long long ldd, long long rows, long long cols, float scale, RopeRef rope, SegPtrs seg) {
  const long long v8 = cols / 8;
  const long long total = rows * v8;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / v8, c = (i % v8) * 8;
    const float4 x = *reinterpret_cast<const float4*>(src + r * lds + c);
    const float4 y = *reinterpret_cast<const float4*>(src + r * lds + c + 4);
    float v[8] = {x.x * scale, x.y * scale, x.z * scale, x.w * scale, y.x * scale, y.y * scale, y.z * scale, y.w * scale};
    // row r is token rope.pos0 + r (head layout [S][heads*d]); gradients rotate back by -angle
    if (rope.hi) dev::rope_rotate<4>(v, rope.hi, rope.lo, rope.d, rope.pos0 + r, (int)(c % rope.d), -1.f);
    *reinterpret_cast<uint4*>(dst_row(dst, seg, r, ldd) + c) =
        make_uint4(dev::pack_bf16(v[0], v[1]), dev::pack_bf16(v[2], v[3]), dev::pack_bf16(v[4], v[5]),
                   dev::pack_bf16(v[6], v[7]));
  }
}

// 64 tokens x 64 dims per tile through shared memory: coalesced 256-byte reads along tokens (four
// 16-byte loads in flight per thread), 16-byte bf16 writes along dims (RoPE pairs are adjacent dims).
__global__ void cvt_dimmajor_kernel(const float* __restrict__ src, long long lds, __nv_bfloat16* __restrict__ dst,
                                    long long ldd, long long rows, long long cols, float scale, RopeRef rope,
                                    SegPtrs seg) {
  __shared__ float tile[64][65];
  const long long ntt = (rows + 63) / 64, nct = cols / 64;
  const int t = threadIdx.x;
  for (long long blk = blockIdx.x; blk < ntt * nct; blk += gridDim.x) {
    const long long t0 = (blk / nct) * 64, c0 = (blk % nct) * 64;
    {
      const int c = t >> 2, tk = (t & 3) * 16;      // dim c of the tile, tokens tk..tk+15
      const float* sp = src + (c0 + c) * lds + t0 + tk;
      if ((lds & 3) == 0 && t0 + tk + 16 <= rows) {
        float4 x[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = *reinterpret_cast<const float4*>(sp + 4 * k);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          tile[c][tk + 4 * k + 0] = x[k].x; tile[c][tk + 4 * k + 1] = x[k].y;
          tile[c][tk + 4 * k + 2] = x[k].z; tile[c][tk + 4 * k + 3] = x[k].w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) tile[c][tk + i] = (t0 + tk + i < rows) ? sp[i] : 0.f;
      }
    }
    __syncthreads();
#pragma unroll
    for (int it = t; it < 512; it += 256) {
      const int tk = it >> 3, cg = (it & 7) * 8;    // token tk, dims cg..cg+7
      if (t0 + tk < rows) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = tile[cg + i][tk] * scale;
        if (rope.hi) dev::rope_rotate<4>(v, rope.hi, rope.lo, rope.d, rope.pos0 + t0 + tk, (int)((c0 + cg) % rope.d), -1.f);
        *reinterpret_cast<uint4*>(dst_row(dst, seg, t0 + tk, ldd) + c0 + cg) =
            make_uint4(dev::pack_bf16(v[0], v[1]), dev::pack_bf16(v[2], v[3]), dev::pack_bf16(v[4], v[5]),
                       dev::pack_bf16(v[6], v[7]));
      }
    }
    __syncthreads();
  }
}

// F5 unpack: segment blockIdx.y, rows in a grid-stride loop; a thread's (row-in-block, vector) split is
// computed once, so the loop carries no 64-bit division (each row's segment is seg_v 16-byte vectors,
// contiguous in both src and dst).
__global__ void unpack_kernel(const uint4* __restrict__ src, long long rows, int seg_v,
                              __nv_bfloat16* __restrict__ dst, long long ldd, long long col_base,
                              long long col_stride) {
  const int s = blockIdx.y;
  const int nt = blockDim.x;
  const int rpb = seg_v >= nt ? 1 : nt / seg_v;           // rows per block iteration
  const int r0 = seg_v >= nt ? 0 : (int)threadIdx.x / seg_v;
  const int v0 = seg_v >= nt ? (int)threadIdx.x : (int)threadIdx.x % seg_v;
  const int vstep = seg_v >= nt ? nt : seg_v;
  if (r0 >= rpb) return;
  const uint4* sp = src + (long long)s * rows * seg_v;
  __nv_bfloat16* dp = dst + col_base + s * col_stride;
  for (long long t = (long long)blockIdx.x * rpb + r0; t < rows; t += (long long)gridDim.x * rpb)
    for (int v = v0; v < seg_v; v += vstep)
      *reinterpret_cast<uint4*>(dp + t * ldd + v * 8) = __ldcs(sp + t * seg_v + v);
}

// ---------------------------------------------------------------- Qwen3 q/k RMSNorm
// One (row, head) of d dims is handled by a group of G = d / 8 consecutive lanes, 8 dims each (16-byte
// bf16 vectors); the group reduces its sum of squares / dot products with xor-shuffles.
template <int G>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// dst[t][h] = rope(src[t][h] * rstd * gamma), rstd = 1/sqrt(mean(src^2) + eps)   (dst may alias src)
template <int G>
__global__ void qk_prep_kernel(const __nv_bfloat16* src, __nv_bfloat16* dst, long long rows, int heads, long long ld,
                               const __nv_bfloat16* __restrict__ gamma, float eps, RopeRef rope) {
  constexpr int d = G * 8;
  const int sub = threadIdx.x % G;
  float gm[8];
  bf16x8_to_f32(*reinterpret_cast<const uint4*>(gamma + sub * 8), gm);
  const long long groups = rows * heads;
  const long long gstride = (long long)gridDim.x * blockDim.x / G;
  // warp-uniform trip count (the group reductions shuffle across the whole warp); lanes past the end idle
  const long long g0 = ((long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) / G;
  for (long long gw = g0; gw < groups; gw += gstride) {
    const long long gi = gw + (threadIdx.x & 31) / G;
    const bool ok = gi < groups;
    const long long t = ok ? gi / heads : 0;
    const int h = ok ? (int)(gi % heads) : 0;
    const long long off = t * ld + (long long)h * d + sub * 8;
    float v[8];
    if (ok) {
      bf16x8_to_f32(*reinterpret_cast<const uint4*>(src + off), v);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = 0.f;
    }
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) ss = fmaf(v[i], v[i], ss);
    const float rstd = rsqrtf(group_sum<G>(ss) * (1.f / d) + eps);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = v[i] * rstd * gm[i];
    if (!ok) continue;
    if (rope.hi) dev::rope_rotate<4>(v, rope.hi, rope.lo, d, rope.pos0 + t, sub * 8, 1.f);
    *reinterpret_cast<uint4*>(dst + off) =
        make_uint4(dev::pack_bf16(v[0], v[1]), dev::pack_bf16(v[2], v[3]), dev::pack_bf16(v[4], v[5]),
                   dev::pack_bf16(v[6], v[7]));
  }
}

// Chain rule of qk_prep for one (row t, head h), fused into the fp32 -> bf16 conversion of the gradient:
//   g = rope^-1(scale * src)  (gradient w.r.t. the normalised, pre-RoPE head),  x = the pre-norm head,
//   x_hat = x rstd,  dx = rstd (g gamma - x_hat mean(g gamma x_hat)),  d(gamma) += g x_hat.
// Tiles of 64 rows x one head through shared memory; src element (t, c) at src[t * st + c] (row-major,
// DIM_MAJOR = false) or src[c * st + t] (dim-major dQ accumulator [heads d][S]).
template <int G, bool DIM_MAJOR>
__global__ void __launch_bounds__(256) norm_bwd_kernel(const float* __restrict__ src, long long st,
                                                       const __nv_bfloat16* __restrict__ x, long long ldx,
                                                       __nv_bfloat16* __restrict__ dst, long long ldd, SegPtrs seg,
                                                       long long rows, int heads, float scale,
                                                       const __nv_bfloat16* __restrict__ gamma, float eps,
                                                       RopeRef rope, float* __restrict__ dgamma,
                                                       float* __restrict__ partials) {
  constexpr int d = G * 8;
  __shared__ float tile[d][65];
  __shared__ float red[d];
  const int t = threadIdx.x;
  const int sub = t % G;                            // fixed 8-dim chunk of this thread
  for (int i = t; i < d; i += blockDim.x) red[i] = 0.f;
  float gm[8], acc[8];
  bf16x8_to_f32(*reinterpret_cast<const uint4*>(gamma + sub * 8), gm);
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
  const long long ntt = (rows + 63) / 64;
  for (long long blk = blockIdx.x; blk < ntt * heads; blk += gridDim.x) {
    const long long t0 = (blk / heads) * 64;
    const int h = (int)(blk % heads);
    __syncthreads();
    if (DIM_MAJOR) {                                // dim c of the head: 64 consecutive tokens
      for (int it = t; it < d * 16; it += blockDim.x) {
        const int c = it >> 4, tk = (it & 15) * 4;
        const float* sp = src + ((long long)h * d + c) * st + t0 + tk;
        if ((st & 3) == 0 && t0 + tk + 4 <= rows) {
          const float4 v4 = *reinterpret_cast<const float4*>(sp);
          tile[c][tk] = v4.x; tile[c][tk + 1] = v4.y; tile[c][tk + 2] = v4.z; tile[c][tk + 3] = v4.w;
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) tile[c][tk + k] = (t0 + tk + k < rows) ? sp[k] : 0.f;
        }
      }
    } else {                                        // token tk: d consecutive dims
      for (int it = t; it < 64 * (d / 4); it += blockDim.x) {
        const int tk = it / (d / 4), c = (it % (d / 4)) * 4;
        float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (t0 + tk < rows) v4 = *reinterpret_cast<const float4*>(src + (t0 + tk) * st + (long long)h * d + c);
        tile[c][tk] = v4.x; tile[c + 1][tk] = v4.y; tile[c + 2][tk] = v4.z; tile[c + 3][tk] = v4.w;
      }
    }
    __syncthreads();
    for (int it = t; it < 64 * G; it += blockDim.x) {
      const int tk = it / G;
      const long long r = t0 + tk;
      const bool ok = r < rows;                     // uniform within the G-lane group
      float g[8], xv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) g[i] = tile[sub * 8 + i][tk] * scale;
      if (rope.hi) dev::rope_rotate<4>(g, rope.hi, rope.lo, d, rope.pos0 + (ok ? r : 0), sub * 8, -1.f);
      if (ok) {
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(x + r * ldx + (long long)h * d + sub * 8), xv);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) xv[i] = 0.f;
      }
      float ss = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) ss = fmaf(xv[i], xv[i], ss);
      const float rstd = rsqrtf(group_sum<G>(ss) * (1.f / d) + eps);
      float dot = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        xv[i] *= rstd;                              // x_hat
        dot = fmaf(g[i] * gm[i], xv[i], dot);
        acc[i] = fmaf(g[i], xv[i], acc[i]);        // d(gamma): rows past the end contribute 0 (g = 0)
      }
      const float m = group_sum<G>(dot) * (1.f / d);
      float o[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = rstd * (g[i] * gm[i] - xv[i] * m);
      if (ok) {
        __nv_bfloat16* drow = seg.n ? reinterpret_cast<__nv_bfloat16*>(seg.p[r / seg.rows]) + (r % seg.rows) * ldd
                                    : dst + r * ldd;
        *reinterpret_cast<uint4*>(drow + (long long)h * d + sub * 8) =
            make_uint4(dev::pack_bf16(o[0], o[1]), dev::pack_bf16(o[2], o[3]), dev::pack_bf16(o[4], o[5]),
                       dev::pack_bf16(o[6], o[7]));
      }
    }
  }
  __syncthreads();
  if (partials) {   // deterministic: this block's d(gamma) partial in thread order, reduced in block order below
    for (int w = 0; w < (int)blockDim.x / G; ++w) {
      if (t / G == w)
#pragma unroll
        for (int i = 0; i < 8; ++i) red[sub * 8 + i] += acc[i];
      __syncthreads();
    }
    for (int i = t; i < d; i += blockDim.x) partials[(long long)blockIdx.x * d + i] = red[i];
    return;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) atomicAdd(&red[sub * 8 + i], acc[i]);
  __syncthreads();
  for (int i = t; i < d; i += blockDim.x) atomicAdd(dgamma + i, red[i]);
}

// dgamma[i] += sum over blocks b (in order) of partials[b][i]
__global__ void sum_partials_kernel(const float* __restrict__ partials, int nblocks, int d, float* __restrict__ dgamma) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int b = 0; b < nblocks; ++b) s += partials[(long long)b * d + i];
    dgamma[i] += s;
  }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

__global__ void synth_kernel(__nv_bfloat16* __restrict__ dst, long long n, uint64_t base, float step) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint64_t z = splitmix64(base + (uint64_t)i);
    const int m = (int)(z >> 56);
    dst[i] = __float2bfloat16_rn((float)(2 * m - 255) * step);   // exact: <= 8 significant bits
  }
}

}  // namespace

cudaError_t rowdot_run(const void* dO, int64_t ld_do, const void* O, int64_t ld_o, float* delta, int64_t ld_delta,
                       int64_t rows, int nheads, int d, cudaStream_t s) {
  if (rows <= 0 || nheads <= 0) return cudaSuccess;
  const int64_t groups = rows * nheads;
  if (d == 128) {
    rowdot_kernel<16><<<grid_for(groups * 16, kThreads), kThreads, 0, s>>>(
        (const __nv_bfloat16*)dO, ld_do, (const __nv_bfloat16*)O, ld_o, delta, ld_delta, rows, nheads, d);
  } else if (d == 64) {
    rowdot_kernel<8><<<grid_for(groups * 8, kThreads), kThreads, 0, s>>>(
        (const __nv_bfloat16*)dO, ld_do, (const __nv_bfloat16*)O, ld_o, delta, ld_delta, rows, nheads, d);
  } else {
    return cudaErrorInvalidValue;
  }
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t merge_partials_run(float* o_acc, const float* o_part, int64_t ld_o, float* lse_acc, const float* lse_part,
                               int64_t ld_lse, int64_t rows, int nheads, int d, cudaStream_t s) {
  if (rows <= 0 || nheads <= 0) return cudaSuccess;
  const int64_t groups = rows * nheads;
  if (d == 128) {
    merge_kernel<32><<<grid_for(groups * 32, kThreads), kThreads, 0, s>>>(o_acc, o_part, ld_o, lse_acc, lse_part,
                                                                          ld_lse, rows, nheads, d);
  } else if (d == 64) {
    merge_kernel<16><<<grid_for(groups * 16, kThreads), kThreads, 0, s>>>(o_acc, o_part, ld_o, lse_acc, lse_part,
                                                                          ld_lse, rows, nheads, d);
  } else {
    return cudaErrorInvalidValue;
  }
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t cvt_f32_bf16_run(const float* src, int64_t lds, void* dst, int64_t ldd, int64_t rows, int64_t cols,
                             float scale, cudaStream_t s, const RopeRef& inverse_rope) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if (cols % 8) return cudaErrorInvalidValue;
  cvt_kernel<<<grid_for(rows * cols / 8, kThreads), kThreads, 0, s>>>(src, lds, (__nv_bfloat16*)dst, ldd, rows,
                                                                     cols, scale, inverse_rope, SegPtrs{});
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t cvt_f32_bf16_run(const float* src, int64_t lds, void* dst, int64_t ldd, int64_t rows, int64_t cols,
                             float scale, cudaStream_t s) {
  return cvt_f32_bf16_run(src, lds, dst, ldd, rows, cols, scale, s, RopeRef{});
}

static bool seg_covers(const SegPtrs& seg, int64_t rows) {
  return seg.n > 0 && seg.n <= kMaxSeg && seg.rows > 0 && (rows + seg.rows - 1) / seg.rows <= seg.n;
}

cudaError_t cvt_f32_bf16_seg_run(const float* src, int64_t lds, const SegPtrs& dst_seg, int64_t ldd, int64_t rows,
                                 int64_t cols, float scale, cudaStream_t s, const RopeRef& inverse_rope) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if (cols % 8 || !seg_covers(dst_seg, rows)) return cudaErrorInvalidValue;
  cvt_kernel<<<grid_for(rows * cols / 8, kThreads), kThreads, 0, s>>>(src, lds, nullptr, ldd, rows, cols, scale,
                                                                     inverse_rope, dst_seg);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t cvt_dimmajor_f32_bf16_run(const float* src, int64_t lds, void* dst, int64_t ldd, int64_t rows,
                                      int64_t cols, float scale, cudaStream_t s, const RopeRef& inverse_rope,
                                      const SegPtrs* dst_seg) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if (cols % 64) return cudaErrorInvalidValue;
  if (dst_seg && dst_seg->n && !seg_covers(*dst_seg, rows)) return cudaErrorInvalidValue;
  const long long tiles = ((rows + 63) / 64) * (cols / 64);
  const int grid = (int)(tiles < 148 * 8 ? tiles : 148 * 8);
  cvt_dimmajor_kernel<<<grid, 256, 0, s>>>(src, lds, (__nv_bfloat16*)dst, ldd, rows, cols, scale, inverse_rope,
                                           dst_seg ? *dst_seg : SegPtrs{});
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t unpack_cols_run(const void* src, int64_t rows, int nseg, int seg_cols, void* dst, int64_t ldd,
                            int64_t col_base, int64_t col_stride, cudaStream_t s) {
  if (rows <= 0 || nseg <= 0) return cudaSuccess;
  if (seg_cols % 8) return cudaErrorInvalidValue;
  const int seg_v = seg_cols / 8;
  const int rpb = seg_v >= kThreads ? 1 : kThreads / seg_v;
  int64_t bx = (rows + rpb - 1) / rpb;
  const int64_t cap = std::max<int64_t>(1, 148 * 16 / nseg);
  if (bx > cap) bx = cap;
  unpack_kernel<<<dim3((unsigned)bx, (unsigned)nseg), kThreads, 0, s>>>(
      (const uint4*)src, rows, seg_v, (__nv_bfloat16*)dst, ldd, col_base, col_stride);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t qk_prep_run(const void* src, void* dst, int64_t rows, int heads, int d, int64_t ld, const void* gamma,
                        float eps, const RopeRef& rope, cudaStream_t s) {
  if (rows <= 0 || heads <= 0) return cudaSuccess;
  const int64_t threads = rows * heads * (d / 8);
  const auto* sp = static_cast<const __nv_bfloat16*>(src);
  auto* dp = static_cast<__nv_bfloat16*>(dst);
  const auto* gp = static_cast<const __nv_bfloat16*>(gamma);
  if (d == 128) qk_prep_kernel<16><<<grid_for(threads, kThreads), kThreads, 0, s>>>(sp, dp, rows, heads, ld, gp, eps, rope);
  else if (d == 64) qk_prep_kernel<8><<<grid_for(threads, kThreads), kThreads, 0, s>>>(sp, dp, rows, heads, ld, gp, eps, rope);
  else return cudaErrorInvalidValue;
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t norm_bwd_run(const float* src, int64_t st, bool dim_major, const void* x, int64_t ldx, void* dst,
                         int64_t ldd, const SegPtrs* dst_seg, int64_t rows, int heads, int d, float scale,
                         const void* gamma, float eps, const RopeRef& inverse_rope, float* dgamma, cudaStream_t s,
                         float* det_partials) {
  if (rows <= 0 || heads <= 0) return cudaSuccess;
  if (dst_seg && dst_seg->n && !seg_covers(*dst_seg, rows)) return cudaErrorInvalidValue;
  const SegPtrs seg = dst_seg ? *dst_seg : SegPtrs{};
  const long long tiles = ((rows + 63) / 64) * heads;
  const int grid = (int)(tiles < kNormBwdMaxBlocks ? tiles : kNormBwdMaxBlocks);
  const auto* xp = static_cast<const __nv_bfloat16*>(x);
  auto* dp = static_cast<__nv_bfloat16*>(dst);
  const auto* gp = static_cast<const __nv_bfloat16*>(gamma);
#define UPIPE_NORM_BWD(G, DM) \
  norm_bwd_kernel<G, DM><<<grid, 256, 0, s>>>(src, st, xp, ldx, dp, ldd, seg, rows, heads, scale, gp, eps, inverse_rope, \
                                               dgamma, det_partials)
  if (d == 128) { if (dim_major) UPIPE_NORM_BWD(16, true); else UPIPE_NORM_BWD(16, false); }
  else if (d == 64) { if (dim_major) UPIPE_NORM_BWD(8, true); else UPIPE_NORM_BWD(8, false); }
  else return cudaErrorInvalidValue;
#undef UPIPE_NORM_BWD
  count_launches(1);
  if (det_partials) {
    sum_partials_kernel<<<1, 128, 0, s>>>(det_partials, grid, d, dgamma);
    count_launches(1);
  }
  return cudaGetLastError();
}

cudaError_t synth_fill_bf16_run(void* dst, int64_t n, uint64_t seed, int tensor_id, int exponent, int64_t start,
                                cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const uint64_t base = seed * 0x9E3779B97F4A7C15ull + (uint64_t)tensor_id * 0xD1B54A32D192ED03ull + (uint64_t)start;
  const float step = ldexpf(1.0f, exponent - 8);
  synth_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>((__nv_bfloat16*)dst, n, base, step);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace upipe
