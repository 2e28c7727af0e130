// prep.cu — LSH / grouping pass of DistrAttention on sm_100a (one launch).
//
// Hash CTAs, two (b*H + h, Q block) units per CTA — §3.2-3.3:
//   y[k][c] = sum_r P[k][r] * Q[r][c]   fp32 fma chain, ascending r, from +0.0f (packed
//                                        fma.rn.f32x2: lane-wise identical to fmaf)
//   bit_k = y > 0 ; pattern = sum bit_k << k ; bucket = inverse-Gray(pattern)
//   perm = stable ascending order of (bucket, column) — rank by counting
//   -> perm workspace (fp32 forward, backward) and the optional bucket / perm exports
//   (distr_attn_hash). The bf16 forward does not launch hash CTAs: its attention CTAs hash their
//   own Q blocks (attn.cu qhat_prologue, the same arithmetic) and sample Q̂ in shared memory.
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
constexpr int kMaxL = 256;  // largest block_l (the staging below works in 128-row chunks)

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

DA_DEV int ilog2(int x) { return 31 - __clz(x); }

// Hash CTAs: two Q blocks per CTA (threads [0, 128) and [128, 256)); in each half, thread t ->
// (column pair cp = t % (D/2), projection group kg = t / (D/2)) of KPT = D/16 consecutive projection
// rows, so one 4-byte (bf16) or 8-byte (fp32) load of the column pair per row feeds KPT FFMA2
// (both columns, one projection row each); the projection (transposed to [r][16] in shared memory,
// shared by both halves) is read with 16-byte loads that are uniform across the warp. Rows are
// walked in ascending order from +0.0f (the bit-exact fma chain), the loads of 8 rows issued ahead
// of their FMAs. Q is read straight from global memory (coalesced: a warp reads 32 consecutive
// column pairs of one row).
template <typename T, int D>
DA_DEV void hash_cta(const PrepArgs& a, int cta, uint8_t* smem) {
  constexpr int NCP = D / 2, NKG = 256 / D, KPT = D / 16;
  static_assert(NCP * NKG == 128, "128 threads per Q block");
  float* proj_t = reinterpret_cast<float*>(smem);                          // [block_l][16]
  uint8_t* parts = smem + kMaxL * 16 * 4;                                  // [2][D][NKG]
  uint32_t* key_s = reinterpret_cast<uint32_t*>(parts + 2 * D * NKG);      // [2][D]
  uint8_t* perm_s = reinterpret_cast<uint8_t*>(key_s + 2 * D);             // [2][D]
  const int half = threadIdx.x >> 7, t = threadIdx.x & 127;
  const int it = 2 * cta + half;  // Q block: bh * nqb + qb
  const bool active = it < a.n_hash_ctas;
  const int lsh = ilog2(a.block_l);
  for (int i = threadIdx.x; i < 16 * a.block_l; i += kThreads) {
    const int k = i >> lsh, r = i & (a.block_l - 1);
    proj_t[r * 16 + k] = a.proj[i];
  }
  __syncthreads();
  const int bh = it / a.nqb, qb = it - bh * a.nqb;
  if (active) {
    const int r0 = qb * a.block_l;
    const int rows = min(a.block_l, a.N - r0);
    const int cp = t % NCP, kg = t / NCP, c = 2 * cp;
    const T* qg = reinterpret_cast<const T*>(a.q) + ((size_t)bh * a.N + r0) * D + c;
    float2 y[KPT];
#pragma unroll
    for (int m = 0; m < KPT; ++m) y[m] = make_float2(0.0f, 0.0f);
    auto load_pair = [&](int r) -> float2 {
      if constexpr (sizeof(T) == 2) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(qg + (size_t)r * D);
        return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
      } else {
        return *reinterpret_cast<const float2*>(qg + (size_t)r * D);
      }
    };
    auto fma_row = [&](int r, float2 qq) {
      const float* pr = proj_t + r * 16 + kg * KPT;
      float pk[KPT];
      if constexpr (KPT >= 4) {
#pragma unroll
        for (int v = 0; v < KPT / 4; ++v) {
          const float4 p4 = *reinterpret_cast<const float4*>(pr + 4 * v);
          pk[4 * v] = p4.x; pk[4 * v + 1] = p4.y; pk[4 * v + 2] = p4.z; pk[4 * v + 3] = p4.w;
        }
      } else {
        const float2 p2 = *reinterpret_cast<const float2*>(pr);
        pk[0] = p2.x; pk[1] = p2.y;
      }
#pragma unroll
      for (int m = 0; m < KPT; ++m) y[m] = fma2(make_float2(pk[m], pk[m]), qq, y[m]);
    };
    int r = 0;
    for (; r + 8 <= rows; r += 8) {
      float2 qv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) qv[j] = load_pair(r + j);
#pragma unroll
      for (int j = 0; j < 8; ++j) fma_row(r + j, qv[j]);
    }
    for (; r < rows; ++r) fma_row(r, load_pair(r));
    uint32_t pa = 0, pb = 0;
#pragma unroll
    for (int m = 0; m < KPT; ++m) {
      pa |= (y[m].x > 0.0f ? 1u : 0u) << m;
      pb |= (y[m].y > 0.0f ? 1u : 0u) << m;
    }
    parts[(half * D + c) * NKG + kg] = (uint8_t)pa;
    parts[(half * D + c + 1) * NKG + kg] = (uint8_t)pb;
  }
  __syncthreads();
  if (active && t < D) {
    uint32_t pattern = 0;
#pragma unroll
    for (int g = 0; g < NKG; ++g) pattern |= (uint32_t)parts[(half * D + t) * NKG + g] << (KPT * g);
    const uint32_t bucket = inverse_gray16(pattern);
    key_s[half * D + t] = (bucket << 8) | (uint32_t)t;  // unique (bucket, column) key
    if (a.bucket_out) a.bucket_out[(size_t)it * D + t] = (uint16_t)bucket;
  }
  __syncthreads();
  if (active && t < D) {
    const uint32_t mine = key_s[half * D + t];
    const uint4* ks = reinterpret_cast<const uint4*>(key_s + half * D);
    int rank = 0;
#pragma unroll 8
    for (int j = 0; j < D / 4; ++j) {
      const uint4 k4 = ks[j];
      rank += (k4.x < mine ? 1 : 0) + (k4.y < mine ? 1 : 0) + (k4.z < mine ? 1 : 0) + (k4.w < mine ? 1 : 0);
    }
    perm_s[half * D + rank] = (uint8_t)t;
  }
  __syncthreads();
  if (active && t < D) {
    if (a.perm_ws) a.perm_ws[(size_t)it * D + t] = perm_s[half * D + t];
    if (a.perm_out) a.perm_out[(size_t)it * D + t] = perm_s[half * D + t];
  }
}

// K [N][d] -> K^T [d][N_pad] for one (bhkv, 64-key tile).
// Staging: tile[t][*] holds key t's d values in 16-byte chunks stored at chunk index
// c8 ^ f(t), f(t) = (t & 7) ^ ((t >> 3 & 3) << 1): the 16-byte stores of a warp (2 keys x 16
// chunks) and the 2-byte column reads of a warp (8 columns x 4 key octets, 8 keys each) both hit
// distinct banks. Each thread then owns 8 consecutive keys of one column = one 16-byte chunk of
// a K^T row; a warp writes 8 rows x 64 contiguous bytes.
template <typename T, int D>
DA_DEV void kt_cta(const PrepArgs& a, int it, uint8_t* smem) {
  constexpr int CPR = D / 8;  // 16-byte chunks per key row (bf16)
  const int ntile = (a.N + 63) >> 6;
  const int bhkv = it / ntile, t0 = (it - bhkv * ntile) * 64;
  const int nkeys = min(64, a.N - t0);
  uint4* tile = reinterpret_cast<uint4*>(smem);  // [64][CPR] chunks
  const T* kg = reinterpret_cast<const T*>(a.k) + ((size_t)bhkv * a.N + t0) * D;
  constexpr int NIT = 64 * CPR / kThreads;  // 4 (d=128) or 2 (d=64): all loads in flight first
  uint4 w[NIT];
#pragma unroll
  for (int u = 0; u < NIT; ++u) {
    const int i = threadIdx.x + u * kThreads;
    const int t = i / CPR, c8 = i % CPR;
    w[u] = make_uint4(0u, 0u, 0u, 0u);
    if (t < nkeys) {
      if (sizeof(T) == 2) {
        w[u] = *reinterpret_cast<const uint4*>(kg + (size_t)t * D + c8 * 8);
      } else {
        const float4 x0 = *reinterpret_cast<const float4*>(kg + (size_t)t * D + c8 * 8);
        const float4 x1 = *reinterpret_cast<const float4*>(kg + (size_t)t * D + c8 * 8 + 4);
        w[u] = make_uint4((uint32_t)f2bf(x0.x) | ((uint32_t)f2bf(x0.y) << 16),
                          (uint32_t)f2bf(x0.z) | ((uint32_t)f2bf(x0.w) << 16),
                          (uint32_t)f2bf(x1.x) | ((uint32_t)f2bf(x1.y) << 16),
                          (uint32_t)f2bf(x1.z) | ((uint32_t)f2bf(x1.w) << 16));
      }
    }
  }
#pragma unroll
  for (int u = 0; u < NIT; ++u) {
    const int i = threadIdx.x + u * kThreads;
    const int t = i / CPR, c8 = i % CPR;
    const int f = ((t & 7) ^ (((t >> 3) & 3) << 1)) & (CPR - 1);  // d = 32: 4 chunks per key
    tile[t * CPR + (c8 ^ f)] = w[u];
  }
  __syncthreads();
  const uint16_t* te = reinterpret_cast<const uint16_t*>(tile);
  uint16_t* ktg = a.kt + (size_t)bhkv * D * a.N_pad;
  // task -> (column c, key octet k8); lane = (k8 & 3) * 8 + (c & 7)
  for (int i = threadIdx.x; i < D * 8; i += kThreads) {
    const int lane = i & 31, grp = i >> 5;
    const int c = (grp % (D / 8)) * 8 + (lane & 7);
    const int k8 = (grp / (D / 8)) * 4 + (lane >> 3);
    const int t = k8 * 8;
    if (t0 + t >= a.N_pad) continue;
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int ta = t + 2 * e, tb = ta + 1;
      const int fa = ((ta & 7) ^ (((ta >> 3) & 3) << 1)) & (CPR - 1), fb = ((tb & 7) ^ (((tb >> 3) & 3) << 1)) & (CPR - 1);
      const uint32_t lo = te[(ta * CPR + ((c >> 3) ^ fa)) * 8 + (c & 7)];
      const uint32_t hi = te[(tb * CPR + ((c >> 3) ^ fb)) * 8 + (c & 7)];
      w[e] = lo | (hi << 16);
    }
    *reinterpret_cast<uint4*>(ktg + (size_t)c * a.N_pad + t0 + t) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

template <typename T, int D>
__global__ void __launch_bounds__(kThreads) prep_kernel(const PrepArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  // Programmatic dependent launch: the attention kernel that follows may start its CTAs (and
  // their in-CTA LSH prologue, which reads only Q) while this grid runs; it waits on the grid
  // dependency before its first K^T load.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int bid = blockIdx.x, nh = (a.n_hash_ctas + 1) / 2;  // two Q blocks per hash CTA
  if (bid < nh)
    hash_cta<T, D>(a, bid, smem);
  else
    kt_cta<T, D>(a, bid - nh, smem);
}

__global__ void convert_kernel(const float* __restrict__ src, uint16_t* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = f2bf(src[i]);
}

template <typename T, int D>
size_t prep_smem_bytes(int block_l) {  // block_l = 0: no hash CTAs in this launch
  const size_t hash = block_l ? kMaxL * 16 * 4 + 2 * D * (256 / D) + 2 * D * 4 + 2 * D : 0;
  const size_t kt = 64 * D * 2;
  return std::max(hash, kt);
}

template <typename T, int D>
cudaError_t launch_prep_t(const PrepArgs& a, cudaStream_t st) {
  const int grid = (a.n_hash_ctas + 1) / 2 + a.n_kt_ctas;
  const size_t smem = prep_smem_bytes<T, D>(a.n_hash_ctas ? a.block_l : 0);
  cudaError_t e = cudaFuncSetAttribute(prep_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  prep_kernel<T, D><<<grid, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_prep(const PrepArgs& a, cudaStream_t st) {
  if (a.n_hash_ctas + a.n_kt_ctas == 0) return cudaSuccess;
  if (a.in_f32)
    return a.d == 32 ? launch_prep_t<float, 32>(a, st)
                     : a.d == 64 ? launch_prep_t<float, 64>(a, st) : launch_prep_t<float, 128>(a, st);
  return a.d == 32 ? launch_prep_t<uint16_t, 32>(a, st)
                   : a.d == 64 ? launch_prep_t<uint16_t, 64>(a, st) : launch_prep_t<uint16_t, 128>(a, st);
}

cudaError_t launch_convert_bf16(const float* src, uint16_t* dst, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int grid = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
  convert_kernel<<<grid, 256, 0, st>>>(src, dst, n);
  return cudaGetLastError();
}

}  // namespace da
