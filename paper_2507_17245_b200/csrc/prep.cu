// prep.cu — LSH / grouping pass of DistrAttention on sm_100a (one launch).
//
// Hash CTAs, one per (b*H + h, Q block) — §3.2-3.3:
//   y[k][c] = sum_r P[k][r] * Q[r][c]   fp32 fma chain, ascending r, from +0.0f (packed
//                                        fma.rn.f32x2: lane-wise identical to fmaf)
//   bit_k = y > 0 ; pattern = sum bit_k << k ; bucket = inverse-Gray(pattern)
//   perm = stable ascending order of (bucket, column) — rank by counting
//   Q̂[r][j] = Q[r][perm[j*G]] (sampling), written in the tile layout the attention
//   kernel's TMA reads: [BH][N][DR], DR = HB * d / G, hash block hb of a 128-row tile occupying
//   columns [hb*d/G, (hb+1)*d/G) and zeros elsewhere (block-diagonal stacking for block_l = 64).
// K^T CTAs, one per (b*H_kv + h, 64-key tile): K [N][d] -> K^T [d][N_pad] (bf16), the layout
//   in which per-(Q block, K tile) fusion is a sum of whole 16-byte row chunks.
//
// Bit-exactness contract with oracle/oracle.c: same fp32 operations in the same order, strict
// y > 0, LSB = projection row 0, ties broken by column index. No fast-math in this file.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"
#include "ptx.cuh"

namespace da {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxL = 128;
constexpr int kMaxD = 128;

template <typename T>
DA_DEV float load_f(const T* p);
template <>
DA_DEV float load_f<uint16_t>(const uint16_t* p) {
  return __uint_as_float(((uint32_t)*p) << 16);
}
template <>
DA_DEV float load_f<float>(const float* p) {
  return *p;
}

DA_DEV uint16_t f2bf(float x) {  // round-to-nearest-even (bf16 inputs round-trip exactly)
  return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}

DA_DEV uint32_t inverse_gray16(uint32_t p) {
  p ^= p >> 1;
  p ^= p >> 2;
  p ^= p >> 4;
  p ^= p >> 8;
  return p & 0xFFFFu;
}

// Number of 16-byte vectors per Q row.
template <typename T>
DA_DEV void hash_cta(const PrepArgs& a, int it, uint8_t* smem) {
  const int D = a.d;
  const int bh = it / a.nqb, qb = it % a.nqb;
  const int r0 = qb * a.block_l;
  const int rows = min(a.block_l, a.N - r0);
  T* q_s = reinterpret_cast<T*>(smem);                                          // [rows][D]
  float* proj_t = reinterpret_cast<float*>(smem + kMaxL * kMaxD * sizeof(T));   // [r][16]
  uint32_t* pat_s = reinterpret_cast<uint32_t*>(proj_t + kMaxL * 16);    // [4][D]
  uint32_t* key_s = pat_s + 4 * kMaxD;                                   // [D]
  uint8_t* perm_s = reinterpret_cast<uint8_t*>(key_s + kMaxD);           // [D]

  // Stage the Q block (16-byte vectors, coalesced) and the transposed projection.
  const T* qg = reinterpret_cast<const T*>(a.q) + ((size_t)bh * a.N + r0) * D;
  const int vec = 16 / sizeof(T);
  const int nvec = rows * D / vec;
  for (int i = threadIdx.x; i < nvec; i += kThreads)
    reinterpret_cast<uint4*>(q_s)[i] = reinterpret_cast<const uint4*>(qg)[i];
  for (int i = threadIdx.x; i < 16 * a.block_l; i += kThreads) {
    const int k = i / a.block_l, r = i % a.block_l;
    proj_t[r * 16 + k] = a.proj[i];
  }
  __syncthreads();

  // Projection: thread -> (column c, group of KPT consecutive projection rows).
  const int nkg = kThreads / D;  // 2 (d=128) or 4 (d=64)
  const int kpt = 16 / nkg;      // 8 or 4
  const int c = threadIdx.x % D, kg = threadIdx.x / D;
  const int k0 = kg * kpt;
  float2 y[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) y[m] = make_float2(0.0f, 0.0f);
  if (kpt == 8) {
    for (int r = 0; r < rows; ++r) {
      const float qv = load_f<T>(q_s + r * D + c);
      const float2 qq = make_float2(qv, qv);
      const float4 pa = *reinterpret_cast<const float4*>(proj_t + r * 16 + k0);
      const float4 pb = *reinterpret_cast<const float4*>(proj_t + r * 16 + k0 + 4);
      y[0] = fma2(make_float2(pa.x, pa.y), qq, y[0]);
      y[1] = fma2(make_float2(pa.z, pa.w), qq, y[1]);
      y[2] = fma2(make_float2(pb.x, pb.y), qq, y[2]);
      y[3] = fma2(make_float2(pb.z, pb.w), qq, y[3]);
    }
  } else {
    for (int r = 0; r < rows; ++r) {
      const float qv = load_f<T>(q_s + r * D + c);
      const float2 qq = make_float2(qv, qv);
      const float4 pa = *reinterpret_cast<const float4*>(proj_t + r * 16 + k0);
      y[0] = fma2(make_float2(pa.x, pa.y), qq, y[0]);
      y[1] = fma2(make_float2(pa.z, pa.w), qq, y[1]);
    }
  }
  uint32_t part = 0;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    if (2 * m < kpt) {
      part |= (y[m].x > 0.0f ? 1u : 0u) << (k0 + 2 * m);
      part |= (y[m].y > 0.0f ? 1u : 0u) << (k0 + 2 * m + 1);
    }
  }
  pat_s[kg * kMaxD + c] = part;
  __syncthreads();

  if (threadIdx.x < D) {
    uint32_t pattern = 0;
    for (int g = 0; g < nkg; ++g) pattern |= pat_s[g * kMaxD + threadIdx.x];
    const uint32_t bucket = inverse_gray16(pattern);
    key_s[threadIdx.x] = (bucket << 8) | (uint32_t)threadIdx.x;  // unique (bucket, column) key
    if (a.bucket_out) a.bucket_out[(size_t)it * D + threadIdx.x] = (uint16_t)bucket;
  }
  __syncthreads();
  if (threadIdx.x < D) {
    const uint32_t mine = key_s[threadIdx.x];
    int rank = 0;
    for (int j = 0; j < D; ++j) rank += key_s[j] < mine ? 1 : 0;
    perm_s[rank] = (uint8_t)threadIdx.x;
  }
  __syncthreads();
  if (threadIdx.x < D) {
    if (a.perm_ws) a.perm_ws[(size_t)it * D + threadIdx.x] = perm_s[threadIdx.x];
    if (a.perm_out) a.perm_out[(size_t)it * D + threadIdx.x] = perm_s[threadIdx.x];
  }
  if (!a.qhat) return;

  // Sampling: Q̂ rows of this block, 8 bf16 (16 B) per store.
  const int dg = D / a.G;
  const int half = (a.HB == 2) ? (qb & 1) : 0;
  const int cpr = a.DR / 8;  // 16-byte chunks per Q̂ row
  uint16_t* qh = a.qhat + ((size_t)bh * a.N + r0) * a.DR;
  for (int i = threadIdx.x; i < rows * cpr; i += kThreads) {
    const int r = i / cpr, ch = i % cpr;
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint16_t v2[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int col = ch * 8 + 2 * e + u;
        const int j = col - half * dg;
        v2[u] = (j >= 0 && j < dg) ? f2bf(load_f<T>(q_s + r * D + perm_s[j * a.G])) : (uint16_t)0;
      }
      w[e] = (uint32_t)v2[0] | ((uint32_t)v2[1] << 16);
    }
    *reinterpret_cast<uint4*>(qh + (size_t)r * a.DR + ch * 8) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// K [N][d] -> K^T [d][N_pad] for one (bhkv, 64-key tile). The smem tile row pitch is d+2
// elements (65 words for d=128) so that the transposed reads (8 key rows x 4 columns per warp)
// hit 16 distinct banks; global reads are 16-byte vectors, global writes 128-byte row segments.
template <typename T>
DA_DEV void kt_cta(const PrepArgs& a, int it, uint8_t* smem) {
  const int D = a.d;
  const int ntile = (a.N + 63) / 64;
  const int bhkv = it / ntile, t0 = (it % ntile) * 64;
  const int nkeys = min(64, a.N - t0);
  uint16_t* tile = reinterpret_cast<uint16_t*>(smem);  // [64][D + 2] bf16
  const int ld = D + 2;
  const T* kg = reinterpret_cast<const T*>(a.k) + ((size_t)bhkv * a.N + t0) * D;
  constexpr int VEC = 16 / sizeof(T);
  const int vpr = D / VEC;  // 16-byte vectors per K row
  for (int i = threadIdx.x; i < 64 * vpr; i += kThreads) {
    const int t = i / vpr, cv = i % vpr;
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    if (t < nkeys) {
      const uint4 x = *reinterpret_cast<const uint4*>(kg + (size_t)t * D + cv * VEC);
      if (sizeof(T) == 2) {
        w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w;
      } else {
        w[0] = (uint32_t)f2bf(__uint_as_float(x.x)) | ((uint32_t)f2bf(__uint_as_float(x.y)) << 16);
        w[1] = (uint32_t)f2bf(__uint_as_float(x.z)) | ((uint32_t)f2bf(__uint_as_float(x.w)) << 16);
      }
    }
    uint32_t* dst = reinterpret_cast<uint32_t*>(tile + t * ld + cv * VEC);
#pragma unroll
    for (int e = 0; e < VEC / 2; ++e) dst[e] = w[e];
  }
  __syncthreads();
  // Each thread writes one 16-byte chunk: 8 consecutive keys of one K^T row (8 lanes = 128 B).
  uint16_t* ktg = a.kt + (size_t)bhkv * D * a.N_pad;
  for (int i = threadIdx.x; i < D * 8; i += kThreads) {
    const int c = i / 8, ch = i % 8;
    const int t = t0 + ch * 8;
    if (t >= a.N_pad) continue;
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      w[e] = (uint32_t)tile[(ch * 8 + 2 * e) * ld + c] | ((uint32_t)tile[(ch * 8 + 2 * e + 1) * ld + c] << 16);
    *reinterpret_cast<uint4*>(ktg + (size_t)c * a.N_pad + t) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) prep_kernel(const PrepArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int bid = blockIdx.x;
  if (bid < a.n_hash_ctas)
    hash_cta<T>(a, bid, smem);
  else
    kt_cta<T>(a, bid - a.n_hash_ctas, smem);
}

__global__ void convert_kernel(const float* __restrict__ src, uint16_t* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = f2bf(src[i]);
}

}  // namespace

size_t prep_smem_bytes(int in_f32) {
  const size_t q = (size_t)kMaxL * kMaxD * (in_f32 ? 4 : 2);
  return q + kMaxL * 16 * 4 + 4 * kMaxD * 4 + kMaxD * 4 + kMaxD + 16;
}

cudaError_t launch_prep(const PrepArgs& a, cudaStream_t st) {
  const int grid = a.n_hash_ctas + a.n_kt_ctas;
  if (grid == 0) return cudaSuccess;
  const size_t smem = prep_smem_bytes(a.in_f32);
  cudaError_t e;
  if (a.in_f32) {
    e = cudaFuncSetAttribute(prep_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    prep_kernel<float><<<grid, kThreads, smem, st>>>(a);
  } else {
    e = cudaFuncSetAttribute(prep_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    prep_kernel<uint16_t><<<grid, kThreads, smem, st>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_convert_bf16(const float* src, uint16_t* dst, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int grid = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
  convert_kernel<<<grid, 256, 0, st>>>(src, dst, n);
  return cudaGetLastError();
}

}  // namespace da
