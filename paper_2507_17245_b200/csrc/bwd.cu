// bwd.cu — DistrAttention backward (reading R18: the grouping of each Q
// block is held constant). First version: the five attention GEMMs run on cuBLAS (bf16 in, fp32
// accumulate — plain library GEMMs on the tensor cores) over chunks of query rows, with this
// file's kernels for everything the method adds around them:
//
//   Ŝ = scale · Q̂ K̂ᵀ = scale · Q̃ Kᵀ   with Q̃[r][c] = Q[r][rep_j(c)] (each column replaced by its
//   group's representative, per Q block) — the same scores as Eq. 2 (distributivity), so
//   dK = scale · dŜᵀ Q̃ already holds dK̂ copied onto every group member, and dQ̃ = scale · dŜ K
//   folds onto the representatives: dQ[r][rep_j] = Σ_{c ∈ G_j} dQ̃[r][c] (zero elsewhere).
//
// Kernels: qtilde (Q̃ rows + D[r] = Σ dO∘O), softmax (P = exp(Ŝ − lse), causal mask; fp32 + bf16
// copy), dscore (dŜ = P ∘ (dP − D) · scale, bf16), fold (dQ from dQ̃), reduce (per-query-head
// dK/dV accumulators summed over GQA groups, to bf16).
#include <cublas_v2.h>
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

// P = exp(Ŝ·scale − lse) for a chunk [nb][R][ldn] (columns < nk), causal mask; P fp32 in place
// and a bf16 copy.
__global__ void softmax_kernel(float* S, uint16_t* P16, const float* lse, int nb, int R, int Rst, int nk, int ldn,
                               int r0, int bh0, int N, float scale, int causal) {
  const size_t total = (size_t)nb * R * nk;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int col = (int)(i % nk);
    const size_t rr = i / nk;
    const int r = (int)(rr % R), b = (int)(rr / R);
    const int qrow = r0 + r;
    const size_t off = ((size_t)b * Rst + r) * ldn + col;
    float p = 0.f;
    if (qrow < N && !(causal && col > qrow)) p = __expf(S[off] * scale - lse[(size_t)(bh0 + b) * N + qrow]);
    S[off] = p;
    P16[off] = f2bf(p);
  }
}

// dŜ·scale = P ∘ (dP − D) · scale -> bf16 (chain rule through Ŝ = scale · Q̃ Kᵀ).
__global__ void dscore_kernel(const float* P, const float* dP, uint16_t* dS, const float* D, int nb, int R, int Rst,
                              int nk, int ldn, int r0, int bh0, int N, float scale) {
  const size_t total = (size_t)nb * R * nk;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int col = (int)(i % nk);
    const size_t rr = i / nk;
    const int r = (int)(rr % R), b = (int)(rr / R);
    const size_t off = ((size_t)b * Rst + r) * ldn + col;
    const int qrow = r0 + r;
    const float dv = qrow < N ? D[(size_t)(bh0 + b) * N + qrow] : 0.f;  // cuBLAS path: Dstride = N
    dS[off] = f2bf(P[off] * (dP[off] - dv) * scale);
  }
}

// dQ[r][rep_j] = Σ_{c in G_j} dQ̃[r][c]; non-representative columns 0. dQ̃: [nb][R][d] fp32.
__global__ void fold_kernel(const float* dqt, const uint8_t* perm, uint16_t* dq, int nb, int R, int r0, int bh0,
                            int N, int d, int G, int nqb, int block_l) {
  const int b = blockIdx.y, r = blockIdx.x;
  const int qrow = r0 + r;
  if (qrow >= N) return;
  const int bh = bh0 + b;
  const uint8_t* pm = perm + ((size_t)bh * nqb + qrow / block_l) * d;
  const float* src = dqt + ((size_t)b * R + r) * d;
  uint16_t* dst = dq + ((size_t)bh * N + qrow) * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < d / G; j += blockDim.x) {
    float s = 0.f;
    for (int g = 0; g < G; ++g) s += src[pm[j * G + g]];
    dst[pm[j * G]] = f2bf(s);
  }
}

// dk[bhkv] = Σ_{query heads of the group} acc[bh] -> bf16
__global__ void reduce_kernel(const float* acc, uint16_t* dst, int BHkv, int rep, size_t per_head) {
  const size_t total = (size_t)BHkv * per_head;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t hk = i / per_head, e = i % per_head;
    float s = 0.f;
    for (int g = 0; g < rep; ++g) s += acc[(hk * rep + g) * per_head + e];
    dst[i] = f2bf(s);
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

#define CB(x)                                              \
  do {                                                     \
    cublasStatus_t s_ = (x);                               \
    if (s_ != CUBLAS_STATUS_SUCCESS) return (int)s_ + 1000; \
  } while (0)
#define CU(x)                                   \
  do {                                          \
    cudaError_t e_ = (x);                       \
    if (e_ != cudaSuccess) return (int)e_;      \
  } while (0)

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

int run_backward(const BwdArgs& a, void* handle, cudaStream_t st) {
  cublasHandle_t h = static_cast<cublasHandle_t>(handle);
  CB(cublasSetStream(h, st));
  const int BH = a.BH, N = a.N, d = a.d;
  const int rep = a.H / a.Hkv;
  // 1. Q̃ and D
  qtilde_kernel<<<dim3((N + 63) / 64, BH), 256, 0, st>>>(a);
  CU(cudaGetLastError());
  CU(cudaMemsetAsync(a.dk_acc, 0, (size_t)BH * N * d * 4, st));
  CU(cudaMemsetAsync(a.dv_acc, 0, (size_t)BH * N * d * 4, st));
  const float one = 1.f, zero = 0.f;
  // 2. chunks of R query rows for nb heads at a time. The batched-GEMM pointer arrays of every
  // iteration are built on the host once and uploaded in one copy.
  const int n_hg = (BH + a.nb - 1) / a.nb, n_rc = (N + a.R - 1) / a.R;
  const size_t per_it = 11 * (size_t)a.nb;
  const void** hp = a.host_ptrs;
  for (int hg = 0; hg < n_hg; ++hg)
    for (int rc = 0; rc < n_rc; ++rc) {
      const void** it = hp + ((size_t)hg * n_rc + rc) * per_it;
      const int bh0 = hg * a.nb, r0 = rc * a.R;
      for (int b = 0; b < a.nb; ++b) {
        const int bh = std::min(bh0 + b, BH - 1), bhkv = (bh / a.H) * a.Hkv + (bh % a.H) / rep;
        const size_t qo = ((size_t)bh * N + r0) * d, ko = (size_t)bhkv * N * d;
        const size_t so = (size_t)b * a.R * N;
        it[0 * a.nb + b] = a.k + ko;            // K
        it[1 * a.nb + b] = a.qt + qo;           // Q̃ chunk
        it[2 * a.nb + b] = a.S + so;            // Ŝ / P fp32
        it[3 * a.nb + b] = a.v + ko;            // V
        it[4 * a.nb + b] = a.dout + qo;         // dO chunk
        it[5 * a.nb + b] = a.dP + so;           // dP fp32
        it[6 * a.nb + b] = a.P16 + so;          // P bf16
        it[7 * a.nb + b] = a.dv_acc + (size_t)bh * N * d;
        it[8 * a.nb + b] = a.dS16 + so;         // dŜ bf16
        it[9 * a.nb + b] = a.dqt + (size_t)b * a.R * d;
        it[10 * a.nb + b] = a.dk_acc + (size_t)bh * N * d;
      }
    }
  CU(cudaMemcpyAsync(a.dev_ptrs, hp, (size_t)n_hg * n_rc * per_it * sizeof(void*), cudaMemcpyHostToDevice, st));
  for (int hg = 0; hg < n_hg; ++hg) {
    const int bh0 = hg * a.nb, nb = std::min(a.nb, BH - bh0);
    for (int rc = 0; rc < n_rc; ++rc) {
      const int r0 = rc * a.R, R = std::min(a.R, N - r0);
      const int nk = a.causal ? std::min(N, r0 + R) : N;  // keys any row of the chunk can see
      void** P = a.dev_ptrs + ((size_t)hg * n_rc + rc) * per_it;
      auto arr = [&](int i) { return (const void**)(P + i * a.nb); };
      auto arrw = [&](int i) { return (void**)(P + i * a.nb); };
      // Ŝ (R x nk, row-major, ld N) = Q̃ Kᵀ      [column-major: K(T) * Q̃]
      CB(cublasGemmBatchedEx(h, CUBLAS_OP_T, CUBLAS_OP_N, nk, R, d, &one, arr(0), CUDA_R_16BF, d, arr(1),
                             CUDA_R_16BF, d, &zero, arrw(2), CUDA_R_32F, N, nb, CUBLAS_COMPUTE_32F,
                             CUBLAS_GEMM_DEFAULT));
      // dP (R x nk) = dO Vᵀ
      CB(cublasGemmBatchedEx(h, CUBLAS_OP_T, CUBLAS_OP_N, nk, R, d, &one, arr(3), CUDA_R_16BF, d, arr(4),
                             CUDA_R_16BF, d, &zero, arrw(5), CUDA_R_32F, N, nb, CUBLAS_COMPUTE_32F,
                             CUBLAS_GEMM_DEFAULT));
      const size_t tot = (size_t)nb * R * nk;
      softmax_kernel<<<grid_for(tot), 256, 0, st>>>(a.S, a.P16, a.lse, nb, R, a.R, nk, N, r0, bh0, N, a.scale,
                                                    a.causal);
      CU(cudaGetLastError());
      // dV (nk x d) += Pᵀ dO                       [column-major: dO * P(T)]
      CB(cublasGemmBatchedEx(h, CUBLAS_OP_N, CUBLAS_OP_T, d, nk, R, &one, arr(4), CUDA_R_16BF, d, arr(6),
                             CUDA_R_16BF, N, &one, arrw(7), CUDA_R_32F, d, nb, CUBLAS_COMPUTE_32F,
                             CUBLAS_GEMM_DEFAULT));
      dscore_kernel<<<grid_for(tot), 256, 0, st>>>(a.S, a.dP, a.dS16, a.D, nb, R, a.R, nk, N, r0, bh0, N, a.scale);
      CU(cudaGetLastError());
      // dQ̃ (R x d) = dŜ K                          [column-major: K * dŜ]
      CB(cublasGemmBatchedEx(h, CUBLAS_OP_N, CUBLAS_OP_N, d, R, nk, &one, arr(0), CUDA_R_16BF, d, arr(8),
                             CUDA_R_16BF, N, &zero, arrw(9), CUDA_R_32F, d, nb, CUBLAS_COMPUTE_32F,
                             CUBLAS_GEMM_DEFAULT));
      // dK (nk x d) += dŜᵀ Q̃                        [column-major: Q̃ * dŜ(T)]
      CB(cublasGemmBatchedEx(h, CUBLAS_OP_N, CUBLAS_OP_T, d, nk, R, &one, arr(1), CUDA_R_16BF, d, arr(8),
                             CUDA_R_16BF, N, &one, arrw(10), CUDA_R_32F, d, nb, CUBLAS_COMPUTE_32F,
                             CUBLAS_GEMM_DEFAULT));
      fold_kernel<<<dim3(R, nb), 64, 0, st>>>(a.dqt, a.perm, a.dq, nb, a.R, r0, bh0, N, d, a.G, a.nqb, a.block_l);
      CU(cudaGetLastError());
    }
  }
  const size_t per_head = (size_t)N * d;
  reduce_kernel<<<grid_for((size_t)a.BHkv * per_head), 256, 0, st>>>(a.dk_acc, a.dk, a.BHkv, rep, per_head);
  reduce_kernel<<<grid_for((size_t)a.BHkv * per_head), 256, 0, st>>>(a.dv_acc, a.dv, a.BHkv, rep, per_head);
  CU(cudaGetLastError());
  return 0;
}

}  // namespace da
