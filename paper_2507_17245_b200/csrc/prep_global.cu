// prep_global.cu — the "global grouping" variant of DistrAttention (§3.3: "a unique
// grouping strategy over the complete Q and K^T"): ONE LSH per head over all
// N rows instead of one per Q block, so the permutation — and with it the sampled Q̂ and the fused
// K̂ — is fixed for the whole head and can be materialised once, before the attention kernel,
// which then contracts S over d/G* with no per-tile fusion (attn.cu exact flavour with G > 1).
// Reading R17: the global variant is block-wise DistrAttention with one hash block of height N
// (projection matrix 16 x N from (seed, N)); the oracle computes it with block_l = N.
//
// global_hash_kernel, one CTA per (b*H + h, 16 columns), 128 threads: y[k][c] = sum_{r < N}
//   P[k][r] Q[r][c] as ONE fp32 fma chain in ascending r from +0.0f (the bit-exact contract of R6,
//   now over N rows), streamed through shared memory 128 rows at a time with the next chunk's
//   global loads in flight -> 16-bit sign patterns gpat[bh][c].
// global_gather_kernel, one CTA per (b*H + h, 64 rows): patterns -> inverse Gray -> stable rank by
//   (bucket, column) -> perm (CTA 0 of the head writes perm and the exports); Q̂[r][j] = Q[r][perm[jG]] and
//   K̂[r][j] = bf16(sum_g K_kv[r][perm[jG+g]]) (fp32 sum in group order, one rounding: R15),
//   both [BH][N][DR] bf16 with DR = d/G* — K̂ per QUERY head (GQA heads of one KV head have
//   different groupings).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"
#include "ptx.cuh"

namespace da {
namespace {

constexpr int kT = 256;
constexpr int kChunk = 128;

DA_DEV uint32_t inverse_gray16g(uint32_t p) {
  p ^= p >> 1;
  p ^= p >> 2;
  p ^= p >> 4;
  p ^= p >> 8;
  return p & 0xFFFFu;
}

// One CTA per (b*H + h, 16-column slice): thread = (column c of the slice, projection-row pair
// kq), ONE fp32x2 fma chain over all N rows in ascending order (the R6 contract) — 2048 chains
// per head at d = 128 spread over d/16 CTAs, so a handful of heads (C4: 16) still fills the GPU.
// Rows are staged through shared memory 128 at a time with the next chunk's global loads in
// flight. Output: the 16-bit sign pattern of each column (gpat[bh][c]); the gather kernel turns the
// patterns into buckets and the permutation.
constexpr int kHT = 128;   // hash threads: 16 columns x 8 projection-row pairs
constexpr int kHC = 16;    // columns per hash CTA
template <int D>
__global__ void __launch_bounds__(kHT) global_hash_kernel(const GlobalArgs a) {
  __shared__ __align__(16) uint32_t q_s[kChunk * kHC / 2];  // [r][16 columns] bf16 pairs
  __shared__ __align__(16) float proj_t[kChunk * 16];      // [r][16]
  __shared__ uint32_t bits_s[8][kHC];
  const int bh = blockIdx.x, c0 = blockIdx.y * kHC;
  const int cl = threadIdx.x % kHC, kq = threadIdx.x / kHC;  // column of the slice, rows 2kq, 2kq+1
  const uint16_t* qg = a.q + (size_t)bh * a.N * D + c0;
  const int nchunk = (a.N + kChunk - 1) / kChunk;
  float2 y = make_float2(0.0f, 0.0f);
  // staging per chunk: 128 rows x 16 columns bf16 = 256 16-byte vectors (2 per thread) and the
  // projection [16][128 rows] (16 per thread)
  uint4 nq[2];
  float np_[16];
  auto load_chunk = [&](int ci) {
    const int r0 = ci * kChunk, rows = min(kChunk, a.N - r0);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = threadIdx.x + u * kHT, r = i >> 1, half = i & 1;  // 2 vectors per row
      nq[u] = r < rows ? *reinterpret_cast<const uint4*>(qg + (size_t)(r0 + r) * D + half * 8) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = threadIdx.x + u * kHT, k = i / kChunk, r = i % kChunk;  // coalesced in r
      np_[u] = r < rows ? a.proj[(size_t)k * a.N + r0 + r] : 0.0f;
    }
  };
  load_chunk(0);
  for (int ci = 0; ci < nchunk; ++ci) {
    const int rows = min(kChunk, a.N - ci * kChunk);
    __syncthreads();  // previous chunk consumed
#pragma unroll
    for (int u = 0; u < 2; ++u) reinterpret_cast<uint4*>(q_s)[threadIdx.x + u * kHT] = nq[u];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = threadIdx.x + u * kHT;
      proj_t[(i % kChunk) * 16 + i / kChunk] = np_[u];
    }
    __syncthreads();
    if (ci + 1 < nchunk) load_chunk(ci + 1);  // next chunk's loads fly under this chunk's FMAs
    const uint16_t* qc = reinterpret_cast<const uint16_t*>(q_s);
#pragma unroll 8
    for (int r = 0; r < rows; ++r) {  // ascending rows: the R6 fp32 fma chain
      const float qv = __uint_as_float(((uint32_t)qc[r * kHC + cl]) << 16);
      y = fma2(*reinterpret_cast<const float2*>(proj_t + r * 16 + 2 * kq), make_float2(qv, qv), y);
    }
  }
  bits_s[kq][cl] = (y.x > 0.0f ? 1u : 0u) << (2 * kq) | (y.y > 0.0f ? 1u : 0u) << (2 * kq + 1);
  __syncthreads();
  if (threadIdx.x < kHC) {
    uint32_t pattern = 0;
#pragma unroll
    for (int g = 0; g < 8; ++g) pattern |= bits_s[g][threadIdx.x];
    a.gpat[(size_t)bh * D + c0 + threadIdx.x] = (uint16_t)pattern;
  }
}

template <int D, int G>
__global__ void __launch_bounds__(kT) global_gather_kernel(const GlobalArgs a) {
  constexpr int QP = D + 8;
  constexpr int VPR = D / 8;
  constexpr int R = 64;  // rows per CTA
  constexpr int DR = D / G;
  __shared__ __align__(16) uint16_t q_s[R * QP];
  __shared__ __align__(16) uint16_t k_s[R * QP];
  __shared__ uint8_t perm_s[D];
  __shared__ uint32_t key_s[D];
  const int bh = blockIdx.y, r0 = blockIdx.x * R, rows = min(R, a.N - r0);
  const int b = bh / a.H, h = bh % a.H, bhkv = b * a.Hkv + h / (a.H / a.Hkv);
  // buckets (inverse Gray of the sign pattern) and the stable rank by (bucket, column): the same
  // few thousand compares in every CTA of the head; CTA 0 writes the perm and the exports
  if (threadIdx.x < D) {
    const uint32_t bucket = inverse_gray16g(a.gpat[(size_t)bh * D + threadIdx.x]);
    key_s[threadIdx.x] = (bucket << 8) | (uint32_t)threadIdx.x;  // unique (bucket, column) key
    if (blockIdx.x == 0 && a.bucket_out) a.bucket_out[(size_t)bh * D + threadIdx.x] = (uint16_t)bucket;
  }
  __syncthreads();
  if (threadIdx.x < D) {
    const uint32_t mine = key_s[threadIdx.x];
    int rank = 0;
#pragma unroll 16
    for (int j = 0; j < D; ++j) rank += key_s[j] < mine ? 1 : 0;
    perm_s[rank] = (uint8_t)threadIdx.x;
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x < D) {
    a.perm[(size_t)bh * D + threadIdx.x] = perm_s[threadIdx.x];
    if (a.perm_out) a.perm_out[(size_t)bh * D + threadIdx.x] = perm_s[threadIdx.x];
  }
  const uint4* qg = reinterpret_cast<const uint4*>(a.q + ((size_t)bh * a.N + r0) * D);
  const uint4* kg = reinterpret_cast<const uint4*>(a.k + ((size_t)bhkv * a.N + r0) * D);
  constexpr int NIT = R * VPR / kT;
  uint4 vq[NIT], vk[NIT];
#pragma unroll
  for (int u = 0; u < NIT; ++u) {
    const int i = threadIdx.x + u * kT;
    vq[u] = i < rows * VPR ? qg[i] : make_uint4(0, 0, 0, 0);
    vk[u] = i < rows * VPR ? kg[i] : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int u = 0; u < NIT; ++u) {
    const int i = threadIdx.x + u * kT;
    *reinterpret_cast<uint4*>(q_s + (i / VPR) * QP + (i % VPR) * 8) = vq[u];
    *reinterpret_cast<uint4*>(k_s + (i / VPR) * QP + (i % VPR) * 8) = vk[u];
  }
  __syncthreads();
  constexpr int CPR = DR / 8;  // 16-byte output chunks per row
  uint16_t* qh = a.qhat + ((size_t)bh * a.N + r0) * DR;
  uint16_t* kh = a.khat + ((size_t)bh * a.N + r0) * DR;
  for (int i = threadIdx.x; i < rows * CPR; i += kT) {
    const int r = i / CPR, j0 = (i % CPR) * 8;
    uint32_t wq[4], wk[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t q2 = 0, k2 = 0;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int j = j0 + 2 * e + u;
        q2 |= (uint32_t)q_s[r * QP + perm_s[j * G]] << (16 * u);
        float s = 0.0f;
#pragma unroll
        for (int g = 0; g < G; ++g) s += __uint_as_float(((uint32_t)k_s[r * QP + perm_s[j * G + g]]) << 16);
        k2 |= (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(s)) << (16 * u);
      }
      wq[e] = q2;
      wk[e] = k2;
    }
    *reinterpret_cast<uint4*>(qh + (size_t)r * DR + j0) = make_uint4(wq[0], wq[1], wq[2], wq[3]);
    *reinterpret_cast<uint4*>(kh + (size_t)r * DR + j0) = make_uint4(wk[0], wk[1], wk[2], wk[3]);
  }
}

}  // namespace

cudaError_t launch_global_prep(const GlobalArgs& a, cudaStream_t st) {
  const dim3 hgrid(a.BH, a.d / kHC);
  if (a.d == 32)
    global_hash_kernel<32><<<hgrid, kHT, 0, st>>>(a);
  else if (a.d == 64)
    global_hash_kernel<64><<<hgrid, kHT, 0, st>>>(a);
  else
    global_hash_kernel<128><<<hgrid, kHT, 0, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const dim3 grid((a.N + 63) / 64, a.BH);
#define DA_GATHER(D_, G_) \
  if (a.d == D_ && a.G == G_) global_gather_kernel<D_, G_><<<grid, kT, 0, st>>>(a);
  DA_GATHER(32, 1) DA_GATHER(32, 2) DA_GATHER(64, 1) DA_GATHER(64, 2) DA_GATHER(64, 4)
  DA_GATHER(128, 1) DA_GATHER(128, 2) DA_GATHER(128, 4) DA_GATHER(128, 8)
#undef DA_GATHER
  return cudaGetLastError();
}

}  // namespace da
