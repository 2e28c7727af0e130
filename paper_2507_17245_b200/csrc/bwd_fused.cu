// bwd_fused.cu — fused tcgen05 backward of DistrAttention (reading R18).
//
// With the grouping held constant, Ŝ = scale·Q̃Kᵀ (Q̃: every column replaced by its group
// representative, per Q block — bwd.cu) and the backward is the attention backward on (Q̃, K, V)
// followed by the dQ fold. Two kernels, no atomics, everything on the tensor cores:
//
//  bwd_kv_kernel — one CTA per (K/V tile of 128 keys, KV head); loops over the query heads of the
//    GQA group and their Q tiles (causal: only tiles at or below the diagonal):
//      Sᵀ  = K Q̃ᵀ    (SS, M = keys, N = queries, K = d)      -> TMEM [0, 128)
//      dPᵀ = V dOᵀ   (SS)                                      -> TMEM [128, 256)
//      8 warps: Pᵀ = exp2(Sᵀ·scale·log2e − lse·log2e), dŜᵀ = Pᵀ ∘ (dPᵀ − D)·scale -> bf16; warp
//      half h (queries [64h, 64h+64)) writes into columns [64h, 64h+32) of the Sᵀ / dPᵀ ranges,
//      its own (thread = key lane; lse, D of the tile's 128 queries arrive by bulk copy)
//      dV += Pᵀ dO   (TS: A = Pᵀ from TMEM, B = dO MN-major)   -> TMEM [256, 256 + d)
//      dK += dŜᵀ Q̃   (TS: A = dŜᵀ from TMEM, B = Q̃ MN-major)  -> TMEM [384, 384 + d)
//    dK, dV of the tile are written (bf16) once at the end — no cross-CTA reduction.
//  bwd_q_kernel — one CTA per (Q tile, query head); loops over K/V tiles:
//      S = Q̃ Kᵀ, dP = dO Vᵀ (SS) -> dŜ (bf16, TMEM) -> dQ̃ += dŜ K (TS, B = K MN-major)
//    dQ̃ (fp32) goes to a workspace; fold_all_kernel (bwd.cu) folds it onto the representatives.
//
// Every operand layout and descriptor is the one the forward kernel (attn.cu) uses: natural
// [rows][d] tiles in RB-column SWIZZLE_{2 RB}B boxes (RB = 64, or 32 for d = 32) serve as K-major
// operands (rows = M or N, d = K) and as MN-major B operands (rows = K, d = N). d in {32, 64, 128}.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "internal.h"
#include "ptx.cuh"

namespace da {
namespace {

constexpr int T = 128;            // rows per tile (queries or keys)
constexpr int kThreadsB = 384;    // warp 0 TMA, warp 1 MMA, warps 4..11 elementwise
// exp2 pairs (of every 8) evaluated by the FMA-pipe polynomial instead of MUFU.EX2 (as the forward's
// EMU); overridable at build time for A/B runs
#ifndef DA_BWD_EMU
#define DA_BWD_EMU 2
#endif
constexpr int kBwdEmu = DA_BWD_EMU;

// SFULL / PFULL per 64-row half h of the tile pair's score block (+h)
enum { BB_KV = 0, BB_FULL = 1, BB_EMPTY = 3, BB_SFULL = 5, BB_PFULL = 7, BB_DONE = 9, BB_TMEM = 10, BB_N = 11 };

template <int D>
struct BCfg {
  static constexpr int TILE = T * D * 2;  // one [128][d] bf16 tile (D/64 boxes of 16 KB)
  static constexpr int VEC = 1024;        // lse + D vectors of a Q tile (2 x 128 fp32)
  // kv kernel: K, V stationary + 2-stage ring of (Q̃, dO, vec)
  static constexpr int KV_SMEM = 2 * TILE + 2 * (2 * TILE + VEC) + 256 + 1024;
  // q kernel: 2-stage ring of (K, V) (Q̃, dO stationary in TMEM)
  static constexpr int Q_SMEM = 2 * (2 * TILE) + 256 + 1024;
};

// Natural [128][d] tiles: boxes of RB columns (RB * 2-byte rows), swizzled SWIZZLE_{2 RB}B.
template <int D>
struct Box {
  static constexpr int RB = D >= 64 ? 64 : D;
  static constexpr int ROW = RB * 2;  // bytes per row inside a box
  static constexpr uint32_t SW = RB == 64 ? kSw128 : kSw64;
};
template <int D>
DA_DEV uint64_t kmaj(uint32_t base, int kk) {  // K-major operand of a [128][d] tile: K-step kk
  using B = Box<D>;
  constexpr int kpb = B::RB / 16;  // K-steps per box
  return make_sdesc(base + (kk / kpb) * (T * B::ROW) + (kk % kpb) * 32, 16, 8 * B::ROW, B::SW);
}
template <int D>
DA_DEV uint64_t mnmaj(uint32_t base, int kk) {  // MN-major B operand: 16 K-rows per step
  using B = Box<D>;
  return make_sdesc(base + kk * 16 * B::ROW, T * B::ROW, 8 * B::ROW, B::SW);
}
template <int D>
DA_DEV void load_tile(uint8_t* dst, const CUtensorMap* m, uint64_t* bar, int row, int plane) {
  using B = Box<D>;
  for (int bx = 0; bx < D / B::RB; ++bx) tma_load_3d(dst + bx * (T * B::ROW), m, bar, bx * B::RB, row, plane);
}
// Epilogue helper: this thread's `cols` = D/2 consecutive fp32 TMEM columns in chunks of NC.
template <int D>
constexpr int epi_nc() { return D / 2 >= 32 ? 32 : D / 2; }

// ------------------------------------------------------------------------------------ dK, dV
template <int D, bool CAUSAL>
__global__ void __launch_bounds__(kThreadsB, 1)
    bwd_kv_kernel(const __grid_constant__ CUtensorMap tmQt, const __grid_constant__ CUtensorMap tmdO,
                  const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                  const BwdFusedArgs a) {
  using C = BCfg<D>;
  constexpr int NC = epi_nc<D>();  // epilogue TMEM columns per load
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sK = smem;
  uint8_t* sV = sK + C::TILE;
  uint8_t* ring = sV + C::TILE;  // stage s: Q̃ tile, dO tile, vec
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + 2 * (2 * C::TILE + C::VEC));
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(bars + BB_TMEM);
  const int warp = warp_id(), lane = lane_id();
  const int kt = blockIdx.x, bhkv = blockIdx.y;
  const int rep = a.H / a.Hkv;
  const int b = bhkv / a.Hkv, hk = bhkv % a.Hkv;
  const int nqt = (a.N + T - 1) / T;
  const int qt_first = CAUSAL ? kt : 0;  // causal: queries >= keys
  const int per_head = nqt - qt_first;
  const int ntiles = rep * per_head;
  auto tile_of = [&](int n, int* bh, int* qt) {
    *bh = b * a.H + hk * rep + n / per_head;
    *qt = qt_first + n % per_head;
  };
  if (threadIdx.x == 0) {
    mbar_init(&bars[BB_KV], 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars[BB_FULL + s], 1);
      mbar_init(&bars[BB_EMPTY + s], 1);
    }
    for (int hh = 0; hh < 2; ++hh) {
      mbar_init(&bars[BB_SFULL + hh], 1);
      mbar_init(&bars[BB_PFULL + hh], 128);  // the 4 elementwise warps of half hh
    }
    mbar_init(&bars[BB_DONE], 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_ptr, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars[BB_KV], 2 * C::TILE);
      load_tile<D>(sK, &tmK, &bars[BB_KV], kt * T, bhkv);
      load_tile<D>(sV, &tmV, &bars[BB_KV], kt * T, bhkv);
      for (int n = 0; n < ntiles; ++n) {
        const int s = n & 1;
        int bh, qt;
        tile_of(n, &bh, &qt);
        mbar_wait(&bars[BB_EMPTY + s], ((n >> 1) & 1) ^ 1);
        uint8_t* st = ring + s * (2 * C::TILE + C::VEC);
        mbar_arrive_expect_tx(&bars[BB_FULL + s], 2 * C::TILE + C::VEC);
        load_tile<D>(st, &tmQt, &bars[BB_FULL + s], qt * T, bh);
        load_tile<D>(st + C::TILE, &tmdO, &bars[BB_FULL + s], qt * T, bh);
        bulk_g2s(st + 2 * C::TILE, a.lse_pad + ((size_t)bh * a.N_pad + qt * T), 512, &bars[BB_FULL + s]);
        bulk_g2s(st + 2 * C::TILE + 512, a.D_pad + ((size_t)bh * a.N_pad + qt * T), 512, &bars[BB_FULL + s]);
      }
    }
  } else if (warp == 1) {
    // whole warp runs the loop (uniform descriptors), one elected lane issues each batch
    // Half-split pipeline: the score block of a tile is computed and consumed in two halves of 64
    // queries (N = 64): while the elementwise warps of one half work, the tensor core runs the
    // other half's dV/dK and the next tile's Sᵀ/dPᵀ half; Sᵀ_h(n+1) overwrites Pᵀ_h(n) in TMEM,
    // so it follows dV/dK_h(n) in the in-order pipe.
    constexpr uint32_t IS = make_idesc_bf16(T, T / 2, false, false);  // Sᵀ, dPᵀ halves
    constexpr uint32_t IG = make_idesc_bf16(T, D, false, true);       // dV, dK (B MN-major)
    mbar_wait(&bars[BB_KV], 0);
    tc_fence_after();
    const uint32_t kb = smem_u32(sK), vb = smem_u32(sV);
    constexpr uint32_t HROW = (T / 2) * Box<D>::ROW;  // byte offset of row 64 inside a box
    auto issue_s = [&](int n, int hh) {  // Sᵀ / dPᵀ of queries [64hh, 64hh + 64) of tile n
      const int s = n & 1;
      if (hh == 0) mbar_wait(&bars[BB_FULL + s], (n >> 1) & 1);
      tc_fence_after();
      const uint32_t qb = smem_u32(ring + s * (2 * C::TILE + C::VEC)) + hh * HROW, ob = qb + C::TILE;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tmem + 64 * hh, kmaj<D>(kb, kk), kmaj<D>(qb, kk), IS, kk > 0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tmem + 128 + 64 * hh, kmaj<D>(vb, kk), kmaj<D>(ob, kk), IS, kk > 0);
        mma_commit(&bars[BB_SFULL + hh]);
      }
      __syncwarp();
    };
    if (ntiles > 0) {
      issue_s(0, 0);
      issue_s(0, 1);
    }
    for (int n = 0; n < ntiles; ++n) {
      const int s = n & 1;
      const uint32_t qb = smem_u32(ring + s * (2 * C::TILE + C::VEC)), ob = qb + C::TILE;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        mbar_wait(&bars[BB_PFULL + hh], n & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            // Pᵀ / dŜᵀ of queries [64hh, 64hh + 64) live in columns [64hh, 64hh + 32)
            const int kk = 4 * hh + k4;
            const uint32_t pc = (uint32_t)(64 * hh + 8 * k4);
            const uint32_t acc = (n > 0 || kk > 0) ? 1u : 0u;
            mma_ts(tmem + 256, tmem + pc, mnmaj<D>(ob, kk), IG, acc);
            mma_ts(tmem + 384, tmem + 128 + pc, mnmaj<D>(qb, kk), IG, acc);
          }
          if (hh == 1) mma_commit(&bars[BB_EMPTY + s]);
        }
        __syncwarp();
        if (n + 1 < ntiles) issue_s(n + 1, hh);
      }
    }
    if (elect_one()) mma_commit(&bars[BB_DONE]);
    __syncwarp();
  } else if (warp >= 4) {
    const int half = (warp - 4) >> 2, quad = warp & 3;
    const int key = kt * T + quad * 32 + lane;  // this thread's key row (TMEM lane)
    const uint32_t lb = (uint32_t)(quad * 32) << 16;
    const float sl2 = a.scale * 1.4426950408889634f;
    const float2 sl2x2 = make_float2(sl2, sl2), zero2 = make_float2(0.f, 0.f), sc2 = make_float2(a.scale, a.scale);
    for (int n = 0; n < ntiles; ++n) {
      const int s = n & 1;
      int bh, qt;
      tile_of(n, &bh, &qt);
      mbar_wait(&bars[BB_SFULL + half], n & 1);
      tc_fence_after();
      const float* vec = reinterpret_cast<const float*>(ring + s * (2 * C::TILE + C::VEC) + 2 * C::TILE);
      // two 32-query chunks of this half: Sᵀ, dPᵀ chunk -> Pᵀ, dŜᵀ (bf16) into the first halves of
      // the chunk's own column ranges (chunk c of half h: queries 64h + 32c + [0, 32))
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2) {
        uint32_t sr[32], pr[32];
        tmem_ld32(tmem + lb + 64 * half + 32 * c2, sr);
        tmem_ld32(tmem + lb + 128 + 64 * half + 32 * c2, pr);
        tmem_ld_wait();
        const int q0 = qt * T + 64 * half + 32 * c2;
        const float* lv = vec + 64 * half + 32 * c2;
        const float* dv = vec + 128 + 64 * half + 32 * c2;
        uint32_t pk[16], dk2[16];
#pragma unroll
        for (int e4 = 0; e4 < 8; ++e4) {
          // the tile's −lse·log2e and −D are the same for every lane (key): one 16-byte broadcast
          // load per 4 queries of each (shared-memory wavefronts are the dK/dV kernel's
          // co-bottleneck with the tensor core's operand reads)
          const float4 nl4 = *reinterpret_cast<const float4*>(lv + 4 * e4);
          const float4 nd4 = *reinterpret_cast<const float4*>(dv + 4 * e4);
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int e = 2 * e4 + h2;
            const float2 nl2 = h2 ? make_float2(nl4.z, nl4.w) : make_float2(nl4.x, nl4.y);
            const float2 nd2 = h2 ? make_float2(nd4.z, nd4.w) : make_float2(nd4.x, nd4.y);
            // x = S·scale·log2e − lse·log2e (FFMA2), exp2 on MUFU or, for kBwdEmu of every 8
            // pairs, the FMA-pipe polynomial (the elementwise phase is MUFU-bound at d <= 64)
            const float2 x = fma2(make_float2(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1])), sl2x2, nl2);
            float2 p = (e & 7) >= 8 - kBwdEmu ? exp2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
            if (CAUSAL) {
              if (key > q0 + 2 * e) p.x = 0.f;
              if (key > q0 + 2 * e + 1) p.y = 0.f;
            }
            const float2 g = fadd2(make_float2(__uint_as_float(pr[2 * e]), __uint_as_float(pr[2 * e + 1])), nd2);
            const float2 ds = fma2(fma2(p, g, zero2), sc2, zero2);
            pk[e] = pack_bf16x2(p.x, p.y);
            dk2[e] = pack_bf16x2(ds.x, ds.y);
          }
        }
        // into this half's own columns (no other warp reads them): no race with the other half
        tmem_st16(tmem + lb + 64 * half + 16 * c2, pk);
        tmem_st16(tmem + lb + 128 + 64 * half + 16 * c2, dk2);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bars[BB_PFULL + half]);
    }
    // epilogue: dV, dK rows of this key (each half writes d/2 columns)
    mbar_wait(&bars[BB_DONE], 0);
    tc_fence_after();
    for (int which = 0; which < 2; ++which) {
      uint16_t* dst = (which == 0 ? a.dv : a.dk) + ((size_t)bhkv * a.N + key) * D + half * (D / 2);
      const uint32_t src = tmem + lb + (which == 0 ? 256 : 384) + half * (D / 2);
#pragma unroll
      for (int c = 0; c < D / 2 / NC; ++c) {
        uint32_t r[NC];
        tmem_ldn<NC>(src + NC * c, r);
        tmem_ld_wait();
        if (key < a.N) {
          uint4* o = reinterpret_cast<uint4*>(dst + NC * c);
#pragma unroll
          for (int e = 0; e < NC / 8; ++e)
            o[e] = make_uint4(pack_bf16x2(__uint_as_float(r[8 * e]), __uint_as_float(r[8 * e + 1])),
                              pack_bf16x2(__uint_as_float(r[8 * e + 2]), __uint_as_float(r[8 * e + 3])),
                              pack_bf16x2(__uint_as_float(r[8 * e + 4]), __uint_as_float(r[8 * e + 5])),
                              pack_bf16x2(__uint_as_float(r[8 * e + 6]), __uint_as_float(r[8 * e + 7])));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------------------------ dQ̃
template <int D, bool CAUSAL>
__global__ void __launch_bounds__(kThreadsB, 1)
    bwd_q_kernel(const __grid_constant__ CUtensorMap tmQt, const __grid_constant__ CUtensorMap tmdO,
                 const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                 const BwdFusedArgs a) {
  using C = BCfg<D>;
  constexpr int NC = epi_nc<D>();  // epilogue TMEM columns per load
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  // Q̃ and dO are stationary A operands in TMEM (TS MMAs), so shared memory holds only the K/V
  // ring and the tensor core reads one B tile per MMA from it.
  uint8_t* ring = smem;  // stage s: K tile, V tile
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + 2 * (2 * C::TILE));
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(bars + BB_TMEM);
  const int warp = warp_id(), lane = lane_id();
  const int qt = blockIdx.x, bh = blockIdx.y;
  const int b = bh / a.H, h = bh % a.H, bhkv = b * a.Hkv + h / (a.H / a.Hkv);
  const int nkt = (a.N + T - 1) / T;
  const int ntiles = CAUSAL ? min(qt + 1, nkt) : nkt;
  // TMEM: S [0, 128), dP [128, 256), dQ̃ [256, 256 + D), Q̃ [256 + D, 256 + 3D/2), dO [.., 256 + 2D)
  constexpr uint32_t kColQ = 256 + D, kColO = 256 + D + D / 2;
  // inverse permutations of the (one or two) Q blocks of this tile, for the folding epilogue
  __shared__ uint8_t pos_s[2 * 128], pm_s[2 * 128];
  {
    const int qb0 = (qt * T) / a.block_l, nb = (T + a.block_l - 1) / a.block_l;
    for (int i = threadIdx.x; i < nb * D; i += blockDim.x) {
      const int bb = i / D, qb = qb0 + bb;
      if (qb < a.nqb) {
        const uint8_t c = a.perm[((size_t)bh * a.nqb + qb) * D + i % D];
        pm_s[i] = c;
        pos_s[bb * D + c] = (uint8_t)(i % D);
      }
    }
  }
  if (threadIdx.x == 0) {
    mbar_init(&bars[BB_KV], 256);  // the elementwise threads: Q̃ / dO rows stored into TMEM
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars[BB_FULL + s], 1);
      mbar_init(&bars[BB_EMPTY + s], 1);
    }
    for (int hh = 0; hh < 2; ++hh) {
      mbar_init(&bars[BB_SFULL + hh], 1);
      mbar_init(&bars[BB_PFULL + hh], 128);  // the 4 elementwise warps of half hh
    }
    mbar_init(&bars[BB_DONE], 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_ptr, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;

  if (warp == 0) {
    if (lane == 0) {
      for (int n = 0; n < ntiles; ++n) {
        const int s = n & 1;
        mbar_wait(&bars[BB_EMPTY + s], ((n >> 1) & 1) ^ 1);
        uint8_t* st = ring + s * (2 * C::TILE);
        mbar_arrive_expect_tx(&bars[BB_FULL + s], 2 * C::TILE);
        load_tile<D>(st, &tmK, &bars[BB_FULL + s], n * T, bhkv);
        load_tile<D>(st + C::TILE, &tmV, &bars[BB_FULL + s], n * T, bhkv);
      }
    }
  } else if (warp == 1) {
    // whole warp runs the loop (uniform descriptors), one elected lane issues each batch
    // Half-split pipeline over the 64-key halves of each K/V tile (see the dK/dV kernel).
    constexpr uint32_t IS = make_idesc_bf16(T, T / 2, false, false);
    constexpr uint32_t IG = make_idesc_bf16(T, D, false, true);
    mbar_wait(&bars[BB_KV], 0);
    tc_fence_after();
    constexpr uint32_t HROW = (T / 2) * Box<D>::ROW;
    auto issue_s = [&](int n, int hh) {  // S / dP of keys [64hh, 64hh + 64) of K/V tile n
      const int s = n & 1;
      if (hh == 0) mbar_wait(&bars[BB_FULL + s], (n >> 1) & 1);
      tc_fence_after();
      const uint32_t kb = smem_u32(ring + s * (2 * C::TILE)) + hh * HROW, vb = kb + C::TILE;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)  // A = Q̃ from TMEM: K-step kk = columns [8kk, 8kk + 8)
          mma_ts(tmem + 64 * hh, tmem + kColQ + 8 * kk, kmaj<D>(kb, kk), IS, kk > 0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ts(tmem + 128 + 64 * hh, tmem + kColO + 8 * kk, kmaj<D>(vb, kk), IS, kk > 0);
        mma_commit(&bars[BB_SFULL + hh]);
      }
      __syncwarp();
    };
    if (ntiles > 0) {
      issue_s(0, 0);
      issue_s(0, 1);
    }
    for (int n = 0; n < ntiles; ++n) {
      const int s = n & 1;
      const uint32_t kb = smem_u32(ring + s * (2 * C::TILE));
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        mbar_wait(&bars[BB_PFULL + hh], n & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const int kk = 4 * hh + k4;
            mma_ts(tmem + 256, tmem + (uint32_t)(64 * hh + 8 * k4), mnmaj<D>(kb, kk), IG,
                   (n > 0 || kk > 0) ? 1u : 0u);
          }
          if (hh == 1) mma_commit(&bars[BB_EMPTY + s]);
        }
        __syncwarp();
        if (n + 1 < ntiles) issue_s(n + 1, hh);
      }
    }
    if (elect_one()) mma_commit(&bars[BB_DONE]);
    __syncwarp();
  } else if (warp >= 4) {
    const int half = (warp - 4) >> 2, quad = warp & 3;
    const int row = qt * T + quad * 32 + lane;
    const uint32_t lb = (uint32_t)(quad * 32) << 16;
    const float sl2 = a.scale * 1.4426950408889634f;
    const float nlse2_r = a.lse_pad[(size_t)bh * a.N_pad + row];  // −lse·log2e
    const float ndd = a.D_pad[(size_t)bh * a.N_pad + row];         // −D
    const float2 sl2x2 = make_float2(sl2, sl2), nlse2 = make_float2(nlse2_r, nlse2_r), nd2 = make_float2(ndd, ndd),
                 zero2 = make_float2(0.f, 0.f), sc2 = make_float2(a.scale, a.scale);
    {
      // stationary A operands into TMEM: half 0 stores this row of Q̃, half 1 this row of dO
      // (column c of the row = bf16 elements 2c, 2c+1; zeros past N)
      const uint16_t* src = (half == 0 ? a.qt : a.dout) + ((size_t)bh * a.N + row) * D;
      constexpr int W = D / 2;  // 32-bit columns per row
      uint32_t w[W];
#pragma unroll
      for (int i = 0; i < W / 4; ++i) {
        const uint4 v = row < a.N ? reinterpret_cast<const uint4*>(src)[i] : make_uint4(0u, 0u, 0u, 0u);
        w[4 * i] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
      }
      const uint32_t dst = tmem + lb + (half == 0 ? kColQ : kColO);
      if constexpr (W >= 32) {
#pragma unroll
        for (int c = 0; c < W / 32; ++c) tmem_st32(dst + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&w[32 * c]));
      } else {
        tmem_st16(dst, *reinterpret_cast<uint32_t(*)[16]>(&w[0]));
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bars[BB_KV]);
    }
    for (int n = 0; n < ntiles; ++n) {
      mbar_wait(&bars[BB_SFULL + half], n & 1);
      tc_fence_after();
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2) {
        uint32_t sr[32], pr[32];
        tmem_ld32(tmem + lb + 64 * half + 32 * c2, sr);
        tmem_ld32(tmem + lb + 128 + 64 * half + 32 * c2, pr);
        tmem_ld_wait();
        const int k0 = n * T + 64 * half + 32 * c2;
        uint32_t dk2[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float2 x = fma2(make_float2(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1])), sl2x2, nlse2);
          float2 p = (e & 7) >= 8 - kBwdEmu ? exp2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
          if (CAUSAL) {
            if (k0 + 2 * e > row) p.x = 0.f;
            if (k0 + 2 * e + 1 > row) p.y = 0.f;
          }
          const float2 g = fadd2(make_float2(__uint_as_float(pr[2 * e]), __uint_as_float(pr[2 * e + 1])), nd2);
          const float2 ds = fma2(fma2(p, g, zero2), sc2, zero2);
          dk2[e] = pack_bf16x2(ds.x, ds.y);
        }
        tmem_st16(tmem + lb + 64 * half + 16 * c2, dk2);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bars[BB_PFULL + half]);
    }
    mbar_wait(&bars[BB_DONE], 0);
    tc_fence_after();
    // Epilogue with the fold (reading R18): dQ[r][rep_j] = Σ_{c ∈ G_j} dQ̃[r][c], 0 off the
    // representatives. The dQ̃ rows go through shared memory (the K/V ring is idle once BB_DONE
    // has fired: every MMA, hence every TMA load, is complete), pitch D+1 floats so that the 32
    // rows of a warp reading one column hit 32 banks; each half then builds D/2 output columns.
    float* rows_s = reinterpret_cast<float*>(ring);  // [128][D + 1]
    const int rl = quad * 32 + lane;
#pragma unroll
    for (int c = 0; c < D / 2 / NC; ++c) {
      uint32_t r[NC];
      tmem_ldn<NC>(tmem + lb + 256 + half * (D / 2) + NC * c, r);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < NC; ++e) rows_s[rl * (D + 1) + half * (D / 2) + NC * c + e] = __uint_as_float(r[e]);
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (row < a.N) {
      const int bb = row / a.block_l - (qt * T) / a.block_l;  // this row's Q block within the tile
      const uint8_t* pm = pm_s + bb * D;
      const uint8_t* pos = pos_s + bb * D;  // inverse permutation
      uint16_t* dst = a.dq + ((size_t)bh * a.N + row) * D + half * (D / 2);
#pragma unroll 1
      for (int c8 = 0; c8 < D / 2; c8 += 8) {
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          float v2[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int col = half * (D / 2) + c8 + e + u, ps = pos[col];
            float acc = 0.f;
            if (ps % a.G == 0)
              for (int g = 0; g < a.G; ++g) acc += rows_s[rl * (D + 1) + pm[ps + g]];
            v2[u] = acc;
          }
          w[e / 2] = pack_bf16x2(v2[0], v2[1]);
        }
        *reinterpret_cast<uint4*>(dst + c8) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D, bool CAUSAL>
cudaError_t launch_fused_c(const BwdFusedArgs& a, cudaStream_t st) {
  using C = BCfg<D>;
  // the causal mask is a template parameter: each kernel's elementwise loop is compiled once per
  // flavour (no masking code in the non-causal loop) instead of depending on the compiler's
  // loop versioning
  cudaError_t e = cudaFuncSetAttribute(bwd_kv_kernel<D, CAUSAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::KV_SMEM);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(bwd_q_kernel<D, CAUSAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::Q_SMEM);
  if (e != cudaSuccess) return e;
  const int nt = (a.N + T - 1) / T;
  bwd_kv_kernel<D, CAUSAL><<<dim3(nt, a.BHkv), kThreadsB, C::KV_SMEM, st>>>(*a.tmQt, *a.tmdO, *a.tmK, *a.tmV, a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  bwd_q_kernel<D, CAUSAL><<<dim3(nt, a.BH), kThreadsB, C::Q_SMEM, st>>>(*a.tmQt, *a.tmdO, *a.tmK, *a.tmV, a);
  return cudaGetLastError();
}
template <int D>
cudaError_t launch_fused_t(const BwdFusedArgs& a, cudaStream_t st) {
  return a.causal ? launch_fused_c<D, true>(a, st) : launch_fused_c<D, false>(a, st);
}

}  // namespace

cudaError_t launch_bwd_fused(const BwdFusedArgs& a, cudaStream_t st) {
  if (a.d == 32) return launch_fused_t<32>(a, st);
  if (a.d == 64) return launch_fused_t<64>(a, st);
  if (a.d == 128) return launch_fused_t<128>(a, st);
  return cudaErrorInvalidValue;
}

}  // namespace da
