// internal.h — launcher interfaces shared by the host C-ABI (api.cu) and the kernel translation
// units (prep.cu, attn.cu). Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace da {

// Everything the prep (LSH) kernel needs. All pointers are device pointers.
struct PrepArgs {
  const void* q;       // [BH][N][d] (bf16 or f32)
  const void* k;       // [BHkv][N][d]
  int in_f32;          // input element type: 0 bf16, 1 f32
  int BH, BHkv, N, d, block_l, G, HB, DR, nqb, N_pad;
  const float* proj;   // [16][block_l]
  uint8_t* perm_ws;    // [BH][nqb][d]  (nullable in hash-only mode)
  uint16_t* bucket_out;  // optional export [BH][nqb][d]
  uint8_t* perm_out;     // optional export [BH][nqb][d]
  uint16_t* kt;        // [BHkv][d][N_pad] bf16 bits (nullable)
  int n_hash_ctas;     // Q blocks to hash: BH * nqb (0 = no hashing); two per hash CTA
  int n_kt_ctas;       // BHkv * ceil(N/64) (0 = no K^T pass)
};

// Everything the attention kernel needs besides its three TMA descriptors.
struct AttnArgs {
  int N, H, H_kv, nqt, nkt, nqb, block_l;
  int pair_offset, pair_stride;  // Q-tile-pair shard: CTA x computes slot offset + x * stride
  float scale_log2;  // scale * log2(e)
  int causal;
  int k_per_qhead;      // exact flavour: K (K̂ of the global variant) indexed by the query head
  const uint8_t* perm;  // [BH][nqb][d] precomputed permutations (distr, fp32 inputs) or NULL:
                        // NULL = the attention CTA hashes its own Q blocks (bf16 inputs)
  const float* proj;    // [16][block_l] projection matrix (distr, in-kernel hashing)
  uint16_t* bucket_out; // optional exports [BH][nqb][d] (in-kernel hashing)
  uint8_t* perm_out;
  void* out;            // [BH][N][d]
  int out_f32;
  float* lse;           // optional [BH][N]
  long long* trace;     // optional debug timeline of CTA (0,0): clock64() stamps, [20][256]
  int pdl;              // launched as a programmatic dependent of the K^T prep kernel: the K
                        // producer waits on the grid dependency before its first K^T load
};

cudaError_t launch_prep(const PrepArgs& a, cudaStream_t st);

// Global-grouping variant (prep_global.cu): one LSH per head over all N rows, then Q̂ and K̂
// materialised per query head. All pointers are device pointers; q, k bf16.
struct GlobalArgs {
  const uint16_t* q;     // [BH][N][d]
  const uint16_t* k;     // [BHkv][N][d]
  int BH, H, Hkv, N, d, G;
  const float* proj;     // [16][N] (seed, N)
  uint16_t* gpat;        // [BH][d] workspace: 16-bit sign pattern per column
  uint8_t* perm;         // [BH][d] workspace
  uint16_t* bucket_out;  // optional export [BH][d]
  uint8_t* perm_out;     // optional export [BH][d]
  uint16_t* qhat;        // [BH][N][d/G]
  uint16_t* khat;        // [BH][N][d/G]
};
cudaError_t launch_global_prep(const GlobalArgs& a, cudaStream_t st);

// Backward helpers (bwd.cu). bf16 tensors [B*H][N][d]; everything else workspace.
struct BwdArgs {
  const uint16_t *q, *o, *dout;
  const uint8_t* perm;    // [BH][nqb][d] (hash of q)
  int BH, N, d, G, nqb, block_l;
  uint16_t* qt;           // [BH][N][d] Q̃
  float* D;               // [BH][Dstride]
  int Dstride;            // N_pad (whole 128-row tiles)
};

// Fused tcgen05 backward (bwd_fused.cu), d in {32, 64, 128}. Maps: Q̃, dO [BH][N][d]; K, V
// [BHkv][N][d], all min(d, 64)-column SWIZZLE_{2 min(d, 64)}B boxes of 128 rows.
struct BwdFusedArgs {
  const CUtensorMap *tmQt, *tmdO, *tmK, *tmV;
  const float* lse_pad;  // [BH][N_pad] −lse·log2e (−inf past N)
  const float* D_pad;    // [BH][N_pad] −D (0 past N)
  uint16_t* dq;          // [BH][N][d] bf16 dQ, folded in the dQ̃ kernel's epilogue
  uint16_t *dk, *dv;     // [BHkv][N][d] bf16 outputs
  int BH, BHkv, H, Hkv, N, N_pad, d, causal;
  float scale;
  const uint8_t* perm;   // [BH][nqb][d] permutation of every Q block (the fold's groups)
  int G, nqb, block_l;
  const uint16_t *qt, *dout;  // [BH][N][d] Q̃ and dO (the dQ̃ kernel's stationary TMEM operands)
};
cudaError_t launch_bwd_fused(const BwdFusedArgs& a, cudaStream_t st);
// bwd.cu helpers for the fused path
cudaError_t launch_bwd_prologue(const BwdArgs& a, const float* lse, float* lse_pad, int N_pad, cudaStream_t st);
cudaError_t launch_convert_bf16(const float* src, uint16_t* dst, size_t n, cudaStream_t st);

// Which kernel flavour: DISTR with (d, G, HB) or exact with d.
struct AttnLaunch {
  int d, G, HB, distr;
  int BH;
  const CUtensorMap* tmA;  // Q (exact) or Q̂ (distr)
  const CUtensorMap* tmK;  // K natural (exact) or K^T (distr)
  const CUtensorMap* tmV;
  int emu;                 // exp2 pairs (of 8) evaluated on the FMA pipe: 0, 2, 3 or 4
};
cudaError_t launch_attn(const AttnLaunch& L, const AttnArgs& a, cudaStream_t st);
// Shared memory bytes the attention kernel uses (0 if unsupported combination).
size_t attn_smem_bytes(int d, int G, int HB, int distr);
// Compile-time configuration of the attention kernel for (d, G, HB, distr): S width, ring depths,
// threads, shared memory. Returns false for an unsupported combination.
struct AttnConfig {
  int dr, ns, nkh, threads, smem;
};
bool attn_config(int d, int G, int HB, int distr, AttnConfig* out);

}  // namespace da
