// attn.cu — fused DistrAttention / exact attention forward for sm_100a (tcgen05 + TMEM + TMA).
//
// One CTA = one 128-row Q tile of one (b, h) (the outer loop of Fig. 3); the inner
// loop walks 128-key tiles. Warp roles (256 threads):
//   warp 0      TMA producer: Q (exact) or Q̂ (distr) once, then K (exact) or K^T (distr) and V
//               tiles through a 2-stage mbarrier ring.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer:
//                 S_i  = A · B_i^T   (M=128, N=128, K = d or DR = HB*d/G*; fp32 in TMEM)
//                 O   += P_{i-1} · V_{i-1}  (A = P from TMEM, B = V MN-major, N = d)
//   warps 2-3   (distr) fusion: K̂^T_i[j][t] = sum_{c in G_j} K^T_i[c][t] for this tile's own
//               permutation(s) — Eq. 2 with the block-wise grouping of §3.3 (P:306:
//               "the rows of a K block are grouped depending on which Q block is multiplied by").
//   warps 4-7   softmax (thread = query row = TMEM lane): row max, exp2, row sum, P -> TMEM (bf16),
//               lazy O rescale (only when the running max grows by > 2^8), final O / l epilogue.
// S is double-buffered in TMEM (cols 128..383), O lives in cols 0..d-1.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "internal.h"
#include "ptx.cuh"

namespace da {
namespace {

constexpr int kThreads = 256;
constexpr int BM = 128;  // query rows per tile (UMMA M)
constexpr int BN = 128;  // keys per tile (UMMA N of S, K of PV)
constexpr int NS = 2;    // K/V pipeline stages
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColO = 0;
constexpr uint32_t kColS = 128;  // S buffer b at kColS + 128*b; P_b aliases its first 64 cols

template <int D, bool DISTR, int G, int HB>
struct Cfg {
  static constexpr int DR = DISTR ? HB * D / G : D;  // contraction width of S
  static constexpr int A_COLS = DR;
  static constexpr int A_SW = (A_COLS * 2 >= 128) ? 128 : A_COLS * 2;  // swizzle span (bytes)
  static constexpr int A_BOX_COLS = A_SW / 2;
  static constexpr int A_NBOX = A_COLS / A_BOX_COLS;
  static constexpr int A_BOX_BYTES = BM * A_SW;
  static constexpr int A_BYTES = A_NBOX * A_BOX_BYTES;
  static constexpr int K_BYTES = BN * D * 2;  // K tile (exact) or K^T tile (distr)
  static constexpr int V_BYTES = BN * D * 2;
  static constexpr int KH_BYTES = DISTR ? DR * BN * 2 : 0;
  static constexpr int al(int x) { return (x + 1023) / 1024 * 1024; }
  static constexpr int OFF_A = 0;
  static constexpr int OFF_K = al(OFF_A + A_BYTES);
  static constexpr int OFF_V = OFF_K + NS * K_BYTES;
  static constexpr int OFF_KH = OFF_V + NS * V_BYTES;
  static constexpr int OFF_PERM = OFF_KH + 2 * KH_BYTES;
  static constexpr int OFF_BAR = OFF_PERM + 2 * 128;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;  // + slack for 1024-B alignment
  static constexpr uint32_t A_LAYOUT = A_SW == 128 ? kSw128 : (A_SW == 64 ? kSw64 : kSw32);
  static_assert(DR % 16 == 0 && DR >= 16 && DR <= 128, "reduced width");
  static_assert(A_COLS % A_BOX_COLS == 0, "A boxes");
};

// Barrier slots (uint64 each) inside OFF_BAR.
enum {
  B_Q = 0,
  B_KFULL = 1,   // +s
  B_KEMPTY = 3,  // +s
  B_VFULL = 5,   // +s
  B_VEMPTY = 7,  // +s
  B_KHFULL = 9,  // +b
  B_KHEMPTY = 11,
  B_SFULL = 13,  // +b
  B_PFULL = 15,  // +b
  B_O = 17,
  B_TMEMPTR = 18,
  B_COUNT = 19
};

template <int D, bool DISTR, int G, int HB>
__global__ void __launch_bounds__(kThreads, 1)
    attn_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const AttnArgs args) {
  using C = Cfg<D, DISTR, G, HB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = smem + C::OFF_A;
  uint8_t* sK = smem + C::OFF_K;
  uint8_t* sV = smem + C::OFF_V;
  uint8_t* sKh = smem + C::OFF_KH;
  uint8_t* perm_s = smem + C::OFF_PERM;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint32_t* tmem_ptr_s = reinterpret_cast<uint32_t*>(bars + B_TMEMPTR);

  const int warp = warp_id(), lane = lane_id();
  const int bh = blockIdx.y;
  const int qt = args.causal ? (args.nqt - 1 - (int)blockIdx.x) : (int)blockIdx.x;
  const int b = bh / args.H, h = bh % args.H;
  const int bhkv = b * args.H_kv + h / (args.H / args.H_kv);
  const int q0 = qt * BM;
  const int nk = args.causal ? min(qt + 1, args.nkt) : args.nkt;

  if (threadIdx.x == 0) {
    mbar_init(&bars[B_Q], 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bars[B_KFULL + s], 1);
      mbar_init(&bars[B_KEMPTY + s], DISTR ? 64 : 1);
      mbar_init(&bars[B_VFULL + s], 1);
      mbar_init(&bars[B_VEMPTY + s], 1);
    }
    for (int bb = 0; bb < 2; ++bb) {
      mbar_init(&bars[B_KHFULL + bb], 64);
      mbar_init(&bars[B_KHEMPTY + bb], 1);
      mbar_init(&bars[B_SFULL + bb], 1);
      mbar_init(&bars[B_PFULL + bb], 128);
    }
    mbar_init(&bars[B_O], 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_ptr_s, kTmemCols);
    tmem_relinquish();
  }
  if (DISTR && (warp == 2 || warp == 3)) {
    // This tile's permutation(s): hash block(s) covering rows [q0, q0 + 128).
    const int t = threadIdx.x - 64;
    for (int i = t; i < HB * D; i += 64) {
      const int hb = i / D, c = i % D;
      const int qb = q0 / args.block_l + hb;
      perm_s[hb * D + c] = (qb < args.nqb) ? args.perm[((size_t)bh * args.nqb + qb) * D + c] : (uint8_t)c;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr_s;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      mbar_arrive_expect_tx(&bars[B_Q], C::A_BYTES);
      for (int bx = 0; bx < C::A_NBOX; ++bx)
        tma_load_3d(sA + bx * C::A_BOX_BYTES, &tmA, &bars[B_Q], bx * C::A_BOX_COLS, q0, bh);
      for (int i = 0; i < nk; ++i) {
        const int s = i % NS;
        const uint32_t ph = (i / NS) & 1;
        mbar_wait(&bars[B_KEMPTY + s], ph ^ 1);
        mbar_arrive_expect_tx(&bars[B_KFULL + s], C::K_BYTES);
        if (DISTR) {
          tma_load_3d(sK + s * C::K_BYTES, &tmK, &bars[B_KFULL + s], i * BN, 0, bhkv);
        } else {
          for (int bx = 0; bx < D / 64; ++bx)
            tma_load_3d(sK + s * C::K_BYTES + bx * (BN * 128), &tmK, &bars[B_KFULL + s], bx * 64, i * BN, bhkv);
        }
        mbar_wait(&bars[B_VEMPTY + s], ph ^ 1);
        mbar_arrive_expect_tx(&bars[B_VFULL + s], C::V_BYTES);
        for (int bx = 0; bx < D / 64; ++bx)
          tma_load_3d(sV + s * C::V_BYTES + bx * (BN * 128), &tmV, &bars[B_VFULL + s], bx * 64, i * BN, bhkv);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC_S = make_idesc_bf16(BM, BN, false, DISTR);
      constexpr uint32_t IDESC_PV = make_idesc_bf16(BM, D, false, true);
      const uint32_t a_base = smem_u32(sA);
      auto issue_pv = [&](int j) {
        const int s = j % NS;
        mbar_wait(&bars[B_PFULL + (j & 1)], (j >> 1) & 1);
        mbar_wait(&bars[B_VFULL + s], (j / NS) & 1);
        tc_fence_after();
        const uint32_t v_base = smem_u32(sV + s * C::V_BYTES);
        const uint32_t p_tmem = tmem + kColS + 128u * (j & 1);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          // V as the MN-major B operand: 64-column blocks (LBO) of 8-key groups (SBO).
          const uint64_t vdesc = make_sdesc(v_base + kk * 2048, BN * 128, 1024, kSw128);
          mma_ts(tmem + kColO, p_tmem + kk * 8, vdesc, IDESC_PV, (j > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&bars[B_VEMPTY + s]);
        mma_commit(&bars[B_O]);
      };
      mbar_wait(&bars[B_Q], 0);
      tc_fence_after();
      for (int i = 0; i < nk; ++i) {
        const int bb = i & 1;
        const int s = i % NS;
        if (DISTR)
          mbar_wait(&bars[B_KHFULL + bb], (i >> 1) & 1);
        else
          mbar_wait(&bars[B_KFULL + s], (i / NS) & 1);
        tc_fence_after();
        const uint32_t d_s = tmem + kColS + 128u * bb;
#pragma unroll
        for (int kk = 0; kk < C::A_COLS / 16; ++kk) {
          constexpr int kpb = C::A_BOX_COLS / 16;  // K-steps per A box
          const uint64_t adesc = make_sdesc(a_base + (kk / kpb) * C::A_BOX_BYTES + (kk % kpb) * 32, 16,
                                            8 * C::A_SW, C::A_LAYOUT);
          uint64_t bdesc;
          if (DISTR) {
            // K̂^T as the MN-major B operand: 64-key blocks (LBO = DR*128 B), 8-row groups (SBO).
            bdesc = make_sdesc(smem_u32(sKh + bb * C::KH_BYTES) + kk * 2048, C::DR * 128, 1024, kSw128);
          } else {
            bdesc = make_sdesc(smem_u32(sK + s * C::K_BYTES) + (kk / 4) * (BN * 128) + (kk % 4) * 32, 16, 1024,
                               kSw128);
          }
          mma_ss(d_s, adesc, bdesc, IDESC_S, kk > 0 ? 1u : 0u);
        }
        mma_commit(&bars[B_SFULL + bb]);
        if (DISTR)
          mma_commit(&bars[B_KHEMPTY + bb]);
        else
          mma_commit(&bars[B_KEMPTY + s]);
        if (i > 0) issue_pv(i - 1);
      }
      issue_pv(nk - 1);
    }
  } else if (warp == 2 || warp == 3) {
    // ------------------------------------------------------------------ fusion (distr only)
    if (DISTR) {
      const int ft = threadIdx.x - 64;  // 0..63
      constexpr int NT = C::DR * 16 / 64;  // 16-byte tasks per thread per tile
      constexpr int DG = D / G;
      uint16_t src[NT][G];
      uint32_t dst[NT];
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int task = n * 64 + ft;
        const int j = task >> 4, ch = task & 15;
        const int hb = j / DG, jj = j % DG;
#pragma unroll
        for (int g = 0; g < G; ++g) src[n][g] = (uint16_t)(perm_s[hb * D + jj * G + g] * (BN * 2) + ch * 16);
        dst[n] = (uint32_t)((ch >> 3) * (C::DR * 128) + j * 128 + (((ch & 7) ^ (j & 7)) << 4));
      }
      for (int i = 0; i < nk; ++i) {
        const int s = i % NS, bb = i & 1;
        mbar_wait(&bars[B_KFULL + s], (i / NS) & 1);
        mbar_wait(&bars[B_KHEMPTY + bb], ((i >> 1) & 1) ^ 1);
        const uint8_t* kt = sK + s * C::K_BYTES;
        uint8_t* kh = sKh + bb * C::KH_BYTES;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          uint4 o;
          if (G == 1) {
            o = *reinterpret_cast<const uint4*>(kt + src[n][0]);
          } else {
            float acc[8];
            {
              const uint4 x = *reinterpret_cast<const uint4*>(kt + src[n][0]);
              const uint32_t xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = unpack_bf16x2(xv[e]);
                acc[2 * e] = f.x;
                acc[2 * e + 1] = f.y;
              }
            }
#pragma unroll
            for (int g = 1; g < G; ++g) {
              const uint4 x = *reinterpret_cast<const uint4*>(kt + src[n][g]);
              const uint32_t xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = unpack_bf16x2(xv[e]);
                acc[2 * e] += f.x;
                acc[2 * e + 1] += f.y;
              }
            }
            o = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]), pack_bf16x2(acc[4], acc[5]),
                           pack_bf16x2(acc[6], acc[7]));
          }
          *reinterpret_cast<uint4*>(kh + dst[n]) = o;
        }
        fence_proxy_async_smem();
        mbar_arrive(&bars[B_KHFULL + bb]);
        mbar_arrive(&bars[B_KEMPTY + s]);
      }
    }
  } else {
    // ------------------------------------------------------------------ softmax (warps 4..7)
    const int row = (warp - 4) * 32 + lane;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const int q_row = q0 + row;
    const float sl2 = args.scale_log2;
    float m = -INFINITY;  // running max of scaled log2 scores (possibly stale by <= 8)
    float l = 0.0f;
    int o_seen = 0;
    for (int i = 0; i < nk; ++i) {
      const int bb = i & 1;
      if (i >= 2) {
        while (o_seen < i - 1) {  // PV_{i-2} completed before S_i was committed
          mbar_wait(&bars[B_O], o_seen & 1);
          ++o_seen;
        }
      }
      mbar_wait(&bars[B_SFULL + bb], (i >> 1) & 1);
      tc_fence_after();
      float s[BN];
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_base + kColS + 128u * bb + 32u * c, r);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) s[32 * c + e] = __uint_as_float(r[e]);
      }
      const int kbase = i * BN;
      if (kbase + BN > args.N || (args.causal && kbase + BN - 1 > q0)) {
        const int lim = args.causal ? min(args.N - 1, q_row) : args.N - 1;
#pragma unroll
        for (int e = 0; e < BN; ++e)
          if (kbase + e > lim) s[e] = -INFINITY;
      }
      float mx = s[0];
#pragma unroll
      for (int e = 1; e < BN; ++e) mx = fmaxf(mx, s[e]);
      const float mnew = fmaxf(m, mx * sl2);
      if (i == 0) {
        m = mnew;
      } else {
        const bool need = mnew > m + 8.0f;
        if (__any_sync(0xffffffffu, need)) {
          while (o_seen < i) {  // O must hold exactly sum_{t<i} P_t V_t before rescaling
            mbar_wait(&bars[B_O], o_seen & 1);
            ++o_seen;
          }
          tc_fence_after();
          const float f = need ? ex2(m - mnew) : 1.0f;
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(tmem + lane_base + kColO + 32u * c, r);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * f);
            tmem_st32(tmem + lane_base + kColO + 32u * c, r);
          }
          tmem_st_wait();
          if (need) {
            l *= f;
            m = mnew;
          }
        }
      }
      const float nm = -m;
      float sum = 0.0f;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t pr[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float p0 = ex2(fmaf(s[64 * c + 2 * e], sl2, nm));
          const float p1 = ex2(fmaf(s[64 * c + 2 * e + 1], sl2, nm));
          sum += p0 + p1;
          pr[e] = pack_bf16x2(p0, p1);
        }
        tmem_st32(tmem + lane_base + kColS + 128u * bb + 32u * c, pr);
      }
      l += sum;
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bars[B_PFULL + bb]);
    }
    while (o_seen < nk) {
      mbar_wait(&bars[B_O], o_seen & 1);
      ++o_seen;
    }
    tc_fence_after();
    const float inv = 1.0f / l;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_base + kColO + 32u * c, r);
      tmem_ld_wait();
      if (q_row < args.N) {
        const size_t off = ((size_t)bh * args.N + q_row) * D + 32 * c;
        if (args.out_f32) {
          float4* o = reinterpret_cast<float4*>(static_cast<float*>(args.out) + off);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            o[e] = make_float4(__uint_as_float(r[4 * e]) * inv, __uint_as_float(r[4 * e + 1]) * inv,
                               __uint_as_float(r[4 * e + 2]) * inv, __uint_as_float(r[4 * e + 3]) * inv);
        } else {
          uint4* o = reinterpret_cast<uint4*>(static_cast<uint16_t*>(args.out) + off);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            o[e] = make_uint4(pack_bf16x2(__uint_as_float(r[8 * e]) * inv, __uint_as_float(r[8 * e + 1]) * inv),
                              pack_bf16x2(__uint_as_float(r[8 * e + 2]) * inv, __uint_as_float(r[8 * e + 3]) * inv),
                              pack_bf16x2(__uint_as_float(r[8 * e + 4]) * inv, __uint_as_float(r[8 * e + 5]) * inv),
                              pack_bf16x2(__uint_as_float(r[8 * e + 6]) * inv, __uint_as_float(r[8 * e + 7]) * inv));
        }
      }
    }
    if (args.lse && q_row < args.N) args.lse[(size_t)bh * args.N + q_row] = (m + log2f(l)) * 0.69314718055994531f;
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

template <int D, bool DISTR, int G, int HB>
cudaError_t launch_one(const AttnLaunch& L, const AttnArgs& a, cudaStream_t st) {
  using C = Cfg<D, DISTR, G, HB>;
  auto kern = attn_kernel<D, DISTR, G, HB>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  dim3 grid(a.nqt, L.BH);
  kern<<<grid, kThreads, C::SMEM, st>>>(*L.tmA, *L.tmK, *L.tmV, a);
  return cudaGetLastError();
}

template <int D, bool DISTR, int G, int HB>
constexpr size_t smem_of() {
  return (size_t)Cfg<D, DISTR, G, HB>::SMEM;
}

}  // namespace

#define DA_DISPATCH(MACRO)                                                          \
  if (!distr) {                                                                     \
    if (d == 64) MACRO(64, false, 1, 1);                                            \
    if (d == 128) MACRO(128, false, 1, 1);                                          \
  } else {                                                                          \
    if (d == 64 && G == 1 && HB == 1) MACRO(64, true, 1, 1);                        \
    if (d == 64 && G == 1 && HB == 2) MACRO(64, true, 1, 2);                        \
    if (d == 64 && G == 2 && HB == 1) MACRO(64, true, 2, 1);                        \
    if (d == 64 && G == 2 && HB == 2) MACRO(64, true, 2, 2);                        \
    if (d == 64 && G == 4 && HB == 1) MACRO(64, true, 4, 1);                        \
    if (d == 64 && G == 4 && HB == 2) MACRO(64, true, 4, 2);                        \
    if (d == 128 && G == 1 && HB == 1) MACRO(128, true, 1, 1);                      \
    if (d == 128 && G == 2 && HB == 1) MACRO(128, true, 2, 1);                      \
    if (d == 128 && G == 2 && HB == 2) MACRO(128, true, 2, 2);                      \
    if (d == 128 && G == 4 && HB == 1) MACRO(128, true, 4, 1);                      \
    if (d == 128 && G == 4 && HB == 2) MACRO(128, true, 4, 2);                      \
  }

size_t attn_smem_bytes(int d, int G, int HB, int distr) {
#define DA_SMEM(D_, DI_, G_, HB_) return smem_of<D_, DI_, G_, HB_>()
  DA_DISPATCH(DA_SMEM)
#undef DA_SMEM
  return 0;
}

cudaError_t launch_attn(const AttnLaunch& L, const AttnArgs& a, cudaStream_t st) {
  const int d = L.d, G = L.G, HB = L.HB, distr = L.distr;
#define DA_LAUNCH(D_, DI_, G_, HB_) return launch_one<D_, DI_, G_, HB_>(L, a, st)
  DA_DISPATCH(DA_LAUNCH)
#undef DA_LAUNCH
  return cudaErrorInvalidValue;
}

}  // namespace da
