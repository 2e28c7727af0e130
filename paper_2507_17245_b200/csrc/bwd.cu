// bwd.cu — helper kernels of the DistrAttention backward (reading R18: the
// grouping of each Q block is held constant) around the fused tcgen05 kernels of bwd_fused.cu:
//
//   Ŝ = scale · Q̂ K̂ᵀ = scale · Q̃ Kᵀ   with Q̃[r][c] = Q[r][rep_j(c)] (each column replaced by its
//   group's representative, per Q block) — the same scores as Eq. 2 (distributivity), so
//   dK = scale · dŜᵀ Q̃ already holds dK̂ copied onto every group member, and dQ̃ = scale · dŜ K
//   folds onto the representatives: dQ[r][rep_j] = Σ_{c ∈ G_j} dQ̃[r][c] (zero elsewhere).
//
// Kernels: qtilde (Q̃ rows + D[r] = Σ dO∘O), lse_pad (the forward's LSE padded with +inf to whole
// 128-row tiles), fold_all (dQ from the fp32 dQ̃ workspace).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"

namespace da {
namespace {

__device__ __forceinline__ float bf2f(uint16_t x) { return __uint_as_float(((uint32_t)x) << 16); }
__device__ __forceinline__ uint16_t f2bf(float x) { return __bfloat16_as_ushort(__float2bfloat16_rn(x)); }

// One CTA per (bh, 64-row slab inside one Q block). rep map from the block's permutation.
__global__ void qtilde_kernel(const BwdArgs a) {
  __shared__ uint8_t rep_s[256];
  __shared__ uint8_t inv_s[256];
  const int bh = blockIdx.y;
  const int r0 = blockIdx.x * 64;
  const int qb = r0 / a.block_l;
  const uint8_t* perm = a.perm + ((size_t)bh * a.nqb + qb) * a.d;
  for (int i = threadIdx.x; i < a.d; i += blockDim.x) inv_s[perm[i]] = (uint8_t)i;
  __syncthreads();
  for (int c = threadIdx.x; c < a.d; c += blockDim.x) rep_s[c] = perm[(inv_s[c] / a.G) * a.G];
  __syncthreads();
  const int rows = min(64, a.N - r0);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int r = warp; r < rows; r += blockDim.x / 32) {
    const size_t row = (size_t)bh * a.N + r0 + r;
    const uint16_t* q = a.q + row * a.d;
    const uint16_t* o = a.o + row * a.d;
    const uint16_t* g = a.dout + row * a.d;
    float acc = 0.f;
    for (int c = lane; c < a.d; c += 32) {
      a.qt[row * a.d + c] = q[rep_s[c]];
      acc += bf2f(g[c]) * bf2f(o[c]);
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
    if (lane == 0) a.D[(size_t)bh * a.Dstride + r0 + r] = acc;
  }
}

int grid_for(size_t n) { return (int)std::min<size_t>((n + 255) / 256, 148 * 32); }

__global__ void lse_pad_kernel(const float* lse, float* out, int BH, int N, int N_pad) {
  const size_t total = (size_t)BH * N_pad;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t bh = i / N_pad, r = i % N_pad;
    out[i] = r < (size_t)N ? lse[bh * N + r] : __int_as_float(0x7f800000);  // +inf: P = 0 past N
  }
}

// dQ[r][rep_j] = Σ_{c in G_j} dQ̃[r][c] over whole rows (fused path); non-representatives 0.
__global__ void fold_all_kernel(const float* dqt, const uint8_t* perm, uint16_t* dq, int N, int d, int G, int nqb,
                                int block_l) {
  const int r = blockIdx.x, bh = blockIdx.y;
  const uint8_t* pm = perm + ((size_t)bh * nqb + r / block_l) * d;
  const float* src = dqt + ((size_t)bh * N + r) * d;
  uint16_t* dst = dq + ((size_t)bh * N + r) * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < d / G; j += blockDim.x) {
    float s = 0.f;
    for (int g = 0; g < G; ++g) s += src[pm[j * G + g]];
    dst[pm[j * G]] = f2bf(s);
  }
}

}  // namespace

cudaError_t launch_bwd_prologue(const BwdArgs& a, const float* lse, float* lse_pad, int N_pad, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(a.D, 0, (size_t)a.BH * N_pad * 4, st);
  if (e != cudaSuccess) return e;
  qtilde_kernel<<<dim3((a.N + 63) / 64, a.BH), 256, 0, st>>>(a);
  lse_pad_kernel<<<grid_for((size_t)a.BH * N_pad), 256, 0, st>>>(lse, lse_pad, a.BH, a.N, N_pad);
  return cudaGetLastError();
}

cudaError_t launch_fold_all(const float* dqt, const uint8_t* perm, uint16_t* dq, int BH, int N, int d, int G,
                            int nqb, int block_l, cudaStream_t st) {
  fold_all_kernel<<<dim3(N, BH), 64, 0, st>>>(dqt, perm, dq, N, d, G, nqb, block_l);
  return cudaGetLastError();
}

}  // namespace da
