// bwd.cu — helper kernels of the DistrAttention backward (reading R18: the
// grouping of each Q block is held constant) around the fused tcgen05 kernels of bwd_fused.cu:
//
//   Ŝ = scale · Q̂ K̂ᵀ = scale · Q̃ Kᵀ   with Q̃[r][c] = Q[r][rep_j(c)] (each column replaced by its
//   group's representative, per Q block) — the same scores as Eq. 2 (distributivity), so
//   dK = scale · dŜᵀ Q̃ already holds dK̂ copied onto every group member, and dQ̃ = scale · dŜ K
//   folds onto the representatives: dQ[r][rep_j] = Σ_{c ∈ G_j} dQ̃[r][c] (zero elsewhere).
//
// Kernels: qtilde (Q̃ rows + −D[r] = −Σ dO∘O), lse_pad (−log2e × the forward's LSE, padded with −inf
// to whole 128-row tiles). The fold dQ̃ -> dQ runs in the dQ̃ kernel's epilogue (bwd_fused.cu).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"

namespace da {
namespace {

__device__ __forceinline__ float bf2f(uint16_t x) { return __uint_as_float(((uint32_t)x) << 16); }
__device__ __forceinline__ uint16_t f2bf(float x) { return __bfloat16_as_ushort(__float2bfloat16_rn(x)); }

// One CTA per (bh, 64-row slab inside one Q block; block_l >= 64). The slab's Q rows are staged in
// shared memory with 16-byte loads; each thread then writes 16-byte chunks of Q̃ (8 gathered
// representatives) and the dot products D[r] = Σ dO∘O are reduced over the CPR lanes of a row.
template <int D>
__global__ void __launch_bounds__(256) qtilde_kernel(const BwdArgs a) {
  constexpr int CPR = D / 8, QP = D + 8;  // 16-byte chunks per row, staging pitch (elements)
  __shared__ __align__(16) uint16_t q_s[64 * QP];
  __shared__ uint8_t rep_s[D], inv_s[D];
  const int bh = blockIdx.y;
  const int r0 = blockIdx.x * 64;
  const int qb = r0 / a.block_l;
  const uint8_t* perm = a.perm + ((size_t)bh * a.nqb + qb) * D;
  for (int i = threadIdx.x; i < D; i += blockDim.x) inv_s[perm[i]] = (uint8_t)i;
  const int rows = min(64, a.N - r0);
  const size_t base = ((size_t)bh * a.N + r0) * D;
  for (int i = threadIdx.x; i < 64 * CPR; i += blockDim.x) {
    const int r = i / CPR, ch = i % CPR;
    float acc = 0.f;
    if (r < rows) {
      const uint4 qv = *reinterpret_cast<const uint4*>(a.q + base + (size_t)r * D + 8 * ch);
      *reinterpret_cast<uint4*>(q_s + r * QP + 8 * ch) = qv;
      const uint4 ov = *reinterpret_cast<const uint4*>(a.o + base + (size_t)r * D + 8 * ch);
      const uint4 gv = *reinterpret_cast<const uint4*>(a.dout + base + (size_t)r * D + 8 * ch);
      const uint32_t ow[4] = {ov.x, ov.y, ov.z, ov.w}, gw[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        acc += bf2f((uint16_t)(gw[e] & 0xFFFF)) * bf2f((uint16_t)(ow[e] & 0xFFFF)) +
               bf2f((uint16_t)(gw[e] >> 16)) * bf2f((uint16_t)(ow[e] >> 16));
    }
#pragma unroll
    for (int m = 1; m < CPR; m <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if (ch == 0 && r < rows) a.D[(size_t)bh * a.Dstride + r0 + r] = -acc;  // stored negated: the kernels add it
  }
  __syncthreads();
  for (int c = threadIdx.x; c < D; c += blockDim.x) rep_s[c] = perm[(inv_s[c] / a.G) * a.G];
  __syncthreads();
  for (int i = threadIdx.x; i < rows * CPR; i += blockDim.x) {
    const int r = i / CPR, ch = i % CPR;
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      w[e] = (uint32_t)q_s[r * QP + rep_s[8 * ch + 2 * e]] | ((uint32_t)q_s[r * QP + rep_s[8 * ch + 2 * e + 1]] << 16);
    *reinterpret_cast<uint4*>(a.qt + base + (size_t)r * D + 8 * ch) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

int grid_for(size_t n) { return (int)std::min<size_t>((n + 255) / 256, 148 * 32); }

__global__ void lse_pad_kernel(const float* lse, float* out, int BH, int N, int N_pad) {
  const size_t total = (size_t)BH * N_pad;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t bh = i / N_pad, r = i % N_pad;
    // −lse·log2e, the addend of the backward kernels' exp2 argument; −inf past N: P = 0 there
    out[i] = r < (size_t)N ? -lse[bh * N + r] * 1.4426950408889634f : __int_as_float(0xff800000);
  }
}

}  // namespace

cudaError_t launch_bwd_prologue(const BwdArgs& a, const float* lse, float* lse_pad, int N_pad, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(a.D, 0, (size_t)a.BH * N_pad * 4, st);
  if (e != cudaSuccess) return e;
  const dim3 grid((a.N + 63) / 64, a.BH);
  if (a.d == 32) qtilde_kernel<32><<<grid, 256, 0, st>>>(a);
  else if (a.d == 64) qtilde_kernel<64><<<grid, 256, 0, st>>>(a);
  else qtilde_kernel<128><<<grid, 256, 0, st>>>(a);
  lse_pad_kernel<<<grid_for((size_t)a.BH * N_pad), 256, 0, st>>>(lse, lse_pad, a.BH, a.N, N_pad);
  return cudaGetLastError();
}

}  // namespace da
