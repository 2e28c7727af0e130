// attn.cu — fused DistrAttention / exact attention forward for sm_100a (tcgen05 + TMEM + TMA).
//
// One CTA = TWO 128-row Q tiles of one (b, h) (the outer loop of Fig. 3, two
// iterations per CTA); the inner loop walks 128-key tiles that both Q tiles share in smem.
// Warp roles (exact: 384 threads; distr: 512):
//   warp 0      TMA producer of the K ring: K tiles (exact, K-major SW128) or K^T tiles (distr,
//               128 keys x d rows). The A operand (Q for exact; the natural Q tiles the distr
//               prologue hashes) is loaded once by thread 0 before the roles start.
//   warp 1      TMEM allocator (512 columns) + tcgen05.mma issuer (warp-uniform loop, one elected
//               lane issues), in the order
//               PV_0(i-1), S_0(i), PV_1(i-1), S_1(i):
//                 S_t  = A_t · B_t^T        (M=128, N=128, K = d or DR = HB*d/G*; fp32 in TMEM)
//                 O_t += P_t · V            (A = P_t bf16 read from TMEM, B = V MN-major, N = d)
//   warp 2      TMA producer of the V ring (SW128); warp 3 idle.
//   warps 4-11  softmax, two warpgroups (DA_PINGPONG = 1, the default): warps 4-7 own Q tile 0,
//               warps 8-11 tile 1; thread = query row = TMEM lane with all 128 keys of a tile, so
//               no row-max exchange, and one tile's S load / max / hand-off overlaps the other
//               tile's exps. Lazy O rescale (only when the running max grows by > 2^8); exp2 on
//               MUFU for the first pass over the row and the FMA-pipe polynomial for EMU/8 of the
//               pairs in a second pass (DA_EXP_SPLIT); P -> TMEM (bf16); O / l epilogue.
//               DA_PINGPONG = 0 keeps the round-2 layout: all 8 warps on one tile at a time,
//               alternating tiles, two warps per row splitting the keys (row max exchanged
//               through shared memory).
//   warps 12-15 (distr) fusion: K̂_t^T[j][key] = sum_{c in G_j} K^T[c][key] with each tile's own
//               permutation(s) — Eq. 2 with the block-wise grouping of §3.3 (P:306:
//               "the rows of a K block are grouped depending on which Q block is multiplied by").
//   distr prologue (warps 4-15, qhat_prologue): hash the CTA's Q blocks from the staged natural
//               Q tiles (fp32 fma chain -> sign bits -> inverse Gray -> stable rank -> perm) and
//               gather Q̂ into the swizzled A operand, before the roles above start.
// TMEM (512 columns): O_0 [0, d), O_1 [d, 2d), S_0 [256, 384), S_1 [384, 512); P_t aliases the
// first 64 columns of S_t.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "internal.h"
#include "ptx.cuh"

#ifndef DA_SPLIT
#define DA_SPLIT 2
#endif
#ifndef DA_WARP_ARRIVE
#define DA_WARP_ARRIVE 0
#endif
#ifndef DA_DIAG_NOFUSE
#define DA_DIAG_NOFUSE 0
#endif
#ifndef DA_EMU_SPREAD
#define DA_EMU_SPREAD 0
#endif
// Experimental (off): FA4-style ping-pong softmax — warps 4-7 own Q tile 0, warps 8-11 tile 1,
// thread = query row with all 128 keys of a tile (no row-max exchange), so one tile's S load / max
// overlaps the other tile's exps.
#ifndef DA_PINGPONG
#define DA_PINGPONG 1
#endif
// DA_PINGPONG = 2 additionally computes S_t(i+1) in two 64-key halves: P_t(i) goes to the upper
// 64 columns of S_t, so the lower half of S_t(i+1) is issued as soon as the tile's softmax has
// loaded S_t(i) (B_SLD), and only the upper half waits for PV_t(i).
// DA_EXP_SPLIT (ping-pong softmax): the MUFU pairs of a row first, the FMA-pipe polynomial pairs
// after them (tools/mb/softmax2.cu: 8 % shorter exp phase with one warp per sub-partition).
#ifndef DA_EXP_SPLIT
#define DA_EXP_SPLIT 1
#endif
// DA_PV_SPLIT (ping-pong, with DA_EXP_SPLIT): the softmax finishes keys 0-63 of a row first and
// signals B_PHALF, so PV over those keys runs during the second half's exps and only PV over keys
// 64-127 (then S_t(i+1)) remains on the P -> S chain.
#ifndef DA_PV_SPLIT
#define DA_PV_SPLIT 1
#endif
// Consumer-release barriers (P ready, K̂ ready, K stage free, Q̂ built) take one arrival per warp
// (lane 0 after __syncwarp) instead of one per thread. Measured on B200: no gain (the MMA warp's
// wake-up after the last arrival stays ~300 clk), so off by default.
constexpr int kArrive = DA_WARP_ARRIVE ? 32 : 1;  // threads per arrival
// Softmax warps per query row: the 128 key columns of a tile are split SPLIT ways (4 x SPLIT
// softmax warps, 128/SPLIT columns per thread).
constexpr int kSplit = DA_SPLIT;
static_assert(kSplit == 2 || kSplit == 4, "softmax split");

namespace da {
namespace {

// TMA/MMA warpgroup + SPLIT softmax warpgroups (+ the fusion warpgroup for distr):
// SPLIT = 4 -> 640 threads (exact) / 768 (distr).
constexpr int kSoftmaxWarps = 4 * kSplit;
constexpr int kSoftmaxThreads = 32 * kSoftmaxWarps;
constexpr int kCW = 128 / kSplit;  // key columns per softmax thread
template <bool DISTR>
constexpr int threads_of() { return 128 + kSoftmaxThreads + (DISTR ? 128 : 0); }
constexpr int kFusionThreads = 128;
constexpr int kWorkers = kSoftmaxThreads + kFusionThreads;  // distr: threads running qhat_prologue
constexpr int kXchBytes = 6 * kSplit * 128 * 4;  // row max [2 parity][2 t][SPLIT][128] + sums [2 t][SPLIT][128]
constexpr int BM = 128;  // query rows per tile (UMMA M)
constexpr int BN = 128;  // keys per tile (UMMA N of S, K of PV)
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS = 256;  // S_t at kColS + 128*t
constexpr int kSmemMax = 232448 - 1024;

// HB = hash blocks per 128-row Q tile: 2 (block_l = 64), 1 (block_l = 128), or 0 = one hash block
// spanning both Q tiles of the CTA (block_l = 256): one grouping, one K̂ per key tile for both.
template <int D, bool DISTR, int G, int HB>
struct Cfg {
  static constexpr bool SHARED = DISTR && HB == 0;
  static constexpr int HBE = HB == 0 ? 1 : HB;   // hash blocks stacked in one tile's Q̂
  static constexpr int NKT = SHARED ? 1 : 2;     // K̂ buffer sets (one per Q tile, or one shared)
  // contraction width of S: block-wise distr HBE*d/G*; exact d (G = 1); global grouping d/G*
  static constexpr int DR = DISTR ? HBE * D / G : D / G;
  static constexpr int A_COLS = DR;
  static constexpr int A_SW = (A_COLS * 2 >= 128) ? 128 : A_COLS * 2;  // swizzle span (bytes)
  static constexpr int A_BOX_COLS = A_SW / 2;
  static constexpr int A_NBOX = A_COLS / A_BOX_COLS;
  static constexpr int A_BOX_BYTES = BM * A_SW;
  static constexpr int A_BYTES = A_NBOX * A_BOX_BYTES;  // one Q tile
  static constexpr int K_BYTES = BN * (DISTR ? D : DR) * 2;  // K^T tile (distr), K / K̂ tile (exact/global)
  static constexpr int V_BYTES = BN * D * 2;
  static constexpr int KH_BYTES = DISTR ? DR * BN * 2 : 0;
  // the K̂ region doubles as the prologue's scratch: projection [l][16] fp32, then keys and parts
  static constexpr int PROJ_BYTES = (SHARED ? 256 : 128) * 16 * 4;
  static constexpr int kh_region(int nkh) {
    return DISTR ? (NKT * nkh * KH_BYTES > PROJ_BYTES + 2048 ? NKT * nkh * KH_BYTES : PROJ_BYTES + 2048) : 0;
  }
  static constexpr int al(int x) { return (x + 1023) / 1024 * 1024; }
  static constexpr int bytes(int ns, int nkh) {
    return al(2 * A_BYTES) + ns * (K_BYTES + V_BYTES) + kh_region(nkh) + 1024 + 256 + kXchBytes;
  }
  // Deepest K/V ring (NS) and K̂ ring (NKH) that fit the 227 KB of shared memory.
  static constexpr int NKH = !DISTR ? 0 : (bytes(2, 2) <= kSmemMax ? 2 : 1);
  static constexpr int NS = bytes(2, NKH) <= kSmemMax ? 2 : 1;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_K = al(2 * A_BYTES);
  static constexpr int OFF_V = OFF_K + NS * K_BYTES;
  static constexpr int OFF_KH = OFF_V + NS * V_BYTES;
  static constexpr int OFF_PERM = OFF_KH + kh_region(NKH);
  static constexpr int OFF_BAR = OFF_PERM + 2 * 2 * 128;
  static constexpr int SMEM = OFF_BAR + 256 + kXchBytes + 1024;  // barriers, row-max/sum exchange, align slack
  static constexpr uint32_t A_LAYOUT = A_SW == 128 ? kSw128 : (A_SW == 64 ? kSw64 : kSw32);
  static constexpr int A_SWB = A_SW == 128 ? 3 : (A_SW == 64 ? 2 : 1);  // Swizzle<B,4,3> bits
  // distr: the natural Q tiles (K-major SW128 boxes, 128 rows x d) are staged for the in-CTA
  // hash / Q̂ build in the V ring, or in the K+V rings when the V ring alone is too small.
  static constexpr int QT_BYTES = BM * D * 2;
  // natural Q / V tiles in smem: boxes of RB columns (64, or 32 for d = 32), RB*2-byte rows,
  // swizzled SWIZZLE_{RB*2}B
  static constexpr int RB = D >= 64 ? 64 : D;
  static constexpr int RB_SWB = RB == 64 ? 3 : 2;
  static constexpr bool STAGE_IN_V = NS * V_BYTES >= 2 * QT_BYTES;
  static_assert(DR % 16 == 0 && DR >= 16 && DR <= 128, "reduced width");
  static_assert(A_COLS % A_BOX_COLS == 0, "A boxes");
  static_assert(SMEM <= 232448, "shared memory");
};

// Barrier slots (uint64 each) inside OFF_BAR.
enum {
  B_Q = 0,
  B_KFULL = 1,    // +s (2)
  B_KEMPTY = 3,   // +s
  B_VFULL = 5,    // +s
  B_VEMPTY = 7,   // +s
  B_KHFULL = 9,   // + t*2 + stage (4)
  B_KHEMPTY = 13, // + t*2 + stage (4)
  B_SFULL = 17,   // +t
  B_PFULL = 19,   // +t
  B_OFULL = 21,   // +t
  B_QHAT = 23,    // distr: Q̂ of both tiles built in sA (kWorkers hashing threads arrive)
  B_TMEMPTR = 24,
  B_SLD = 25,     // +t: ping-pong split S (DA_PINGPONG = 2): the tile's softmax has loaded S_t(i)
  B_PHALF = 27,   // +t: DA_PV_SPLIT: P_t(i) of keys 0-63 is in TMEM
  B_COUNT = 29
};

// Release arrival of a whole warp: every lane's prior writes (and fences) are ordered before lane
// 0's arrive by the warp barrier (kArrive == 32), or every thread arrives (kArrive == 1).
DA_DEV void warp_arrive(uint64_t* bar) {
  if constexpr (kArrive == 32) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
  } else {
    mbar_arrive(bar);
  }
}

// Swizzle<B,4,3>: XOR byte-address bits [4, 4+B) with bits [7, 7+B) — the TMA / UMMA
// SWIZZLE_{32,64,128}B layouts (B = 1, 2, 3), valid inside 1024-byte aligned regions.
DA_DEV uint32_t swz(uint32_t a, int B) { return a ^ (((a >> 7) & ((1u << B) - 1u)) << 4); }

DA_DEV uint32_t inverse_gray16(uint32_t p) {
  p ^= p >> 1;
  p ^= p >> 2;
  p ^= p >> 4;
  p ^= p >> 8;
  return p & 0xFFFFu;
}

// LSH + grouping + sampling of the CTA's two Q tiles (§3.2-3.3), run by the kWorkers
// worker threads (the softmax and fusion warps) before their roles start. Same arithmetic as prep.cu hash_cta
// (bit-exact contract with the oracle: fp32 fma chain in ascending rows from +0, strict y > 0,
// LSB = projection row 0, inverse Gray, stable rank by (bucket, column)):
//   staged Q (natural, SW128 K-major boxes) -> y[16] per (tile, hash block, column) -> perm_s
//   -> Q̂ rows gathered into sA in the A operand's swizzled K-major layout.
// With args.perm set (fp32 inputs) the permutations come from the prep kernel instead.
template <class C, int D, int G, int HB>
DA_DEV void qhat_prologue(const AttnArgs& args, uint64_t* bars, const uint8_t* sQ, uint8_t* sA, uint8_t* scratch,
                          uint8_t* perm_s, int bh, int qt0, int ntile, int ht, long long* trace) {
#define PT(i) if (trace && ht == 0) trace[15 * 256 + (i)] = clock64();
  PT(0)
  constexpr int NW = kWorkers;
  constexpr int DG = D / G;
  const int L = args.block_l;
  float* proj_t = reinterpret_cast<float*>(scratch);           // [l][16]
  uint32_t* key_s = reinterpret_cast<uint32_t*>(scratch + C::PROJ_BYTES);  // [2][HB][D] keys, then u8 parts
  auto wsync = [] { asm volatile("bar.sync 5, %0;" ::"n"(kWorkers) : "memory"); };
  // byte offset of staged Q(t, r, c): box c / RB, RB*2-byte rows, SWIZZLE_{RB*2}B
  auto q_off = [&](int t, int r, int c) -> uint32_t {
    return (uint32_t)(t * C::QT_BYTES + (c / C::RB) * (BM * C::RB * 2)) +
           swz((uint32_t)(r * C::RB * 2 + (c % C::RB) * 2), C::RB_SWB);
  };
  const bool hash = args.perm == nullptr;
  if (hash)
    for (int i = ht; i < 16 * L; i += NW) proj_t[(i % L) * 16 + i / L] = args.proj[i];
  mbar_wait(&bars[B_Q], 0);
  wsync();
  PT(1)
  if (hash) {
    // Projection: unit = (tile, hash block, column pair, group of KG of the 16 projection rows):
    // per row one 4-byte load of the two columns, KG/4 16-byte (broadcast) projection loads, KG
    // FFMA2. KG = 8 for the per-tile blocks; the 256-row SHARED block has half as many blocks and
    // takes KG = d/16 (measured hash phase, C3 d=64: KG 2/4/8 = 9.9k/7.8k/10.7k clk; C4 d=128:
    // KG 4/8 = 12.7k/10.8k clk). The groups' KG-bit patterns are OR-ed through shared memory.
    constexpr int KG = !C::SHARED ? 8 : D / 16;
    constexpr int NKG = 16 / KG;
    const int nunits = (C::SHARED ? 1 : ntile * HB) * (D / 2) * NKG;  // (hash block, column pair, group)
    uint8_t* parts = reinterpret_cast<uint8_t*>(key_s + 2 * C::HBE * D);  // [block, column][NKG]
    for (int u2 = ht; u2 < nunits; u2 += NW) {
      const int kg = u2 % NKG, cp = u2 / NKG;    // cp indexes (t, hb, c/2)
      const int t = cp / (C::HBE * D / 2), hb = (cp / (D / 2)) % C::HBE, c = (cp % (D / 2)) * 2;
      const int row0 = (qt0 + t) * BM + hb * L;  // first global row of this hash block
      const int rows = max(0, min(L, args.N - row0));
      float2 ya[KG / 2], yb[KG / 2];  // column c / c+1, projection rows KG*kg .. KG*kg + KG-1
#pragma unroll
      for (int m = 0; m < KG / 2; ++m) ya[m] = yb[m] = make_float2(0.0f, 0.0f);
      const float* pr = proj_t + KG * kg;
      // staged-Q address of row rr (of the hash block) for this thread's column pair: the swizzle
      // XOR term depends only on rr % 8, so the 8 per-row column offsets are precomputed and the
      // row loop runs in blocks of 8 (one add per row instead of the full swizzle arithmetic)
      constexpr uint32_t ROWB = C::RB * 2;
      uint32_t xo[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) xo[j] = swz(j * ROWB + (uint32_t)(c % C::RB) * 2, C::RB_SWB) - j * ROWB;
      const uint32_t cbase = (uint32_t)((c / C::RB) * (BM * C::RB * 2));
      auto hash_row = [&](int r, uint32_t x) {  // ascending rows: the R6 fp32 fma chain
        const uint32_t addr = C::SHARED ? (uint32_t)((r >> 7) * C::QT_BYTES) + cbase + (r & (BM - 1)) * ROWB + x
                                        : (uint32_t)(t * C::QT_BYTES) + cbase + (hb * L + r) * ROWB + x;
        const uint32_t q2 = *reinterpret_cast<const uint32_t*>(sQ + addr);
        const float qa = __uint_as_float(q2 << 16), qb = __uint_as_float(q2 & 0xFFFF0000u);
        float2 pk[KG / 2];
        if constexpr (KG == 2) {
          pk[0] = *reinterpret_cast<const float2*>(pr + r * 16);
        } else {
#pragma unroll
          for (int v4 = 0; v4 < KG / 4; ++v4) {
            const float4 p4 = *reinterpret_cast<const float4*>(pr + r * 16 + 4 * v4);
            pk[2 * v4] = make_float2(p4.x, p4.y);
            pk[2 * v4 + 1] = make_float2(p4.z, p4.w);
          }
        }
#pragma unroll
        for (int m = 0; m < KG / 2; ++m) {
          ya[m] = fma2(pk[m], make_float2(qa, qa), ya[m]);
          yb[m] = fma2(pk[m], make_float2(qb, qb), yb[m]);
        }
      };
      int r = 0;
      for (; r + 8 <= rows; r += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) hash_row(r + j, xo[j]);
      }
      for (; r < rows; ++r)  // ragged tail of the block (rare): the swizzle term recomputed
        hash_row(r, swz((r & 7) * ROWB + (uint32_t)(c % C::RB) * 2, C::RB_SWB) - (r & 7) * ROWB);
      uint32_t ba = 0, bb = 0;
#pragma unroll
      for (int m = 0; m < KG / 2; ++m) {
        ba |= (ya[m].x > 0.0f ? 1u : 0u) << (2 * m) | (ya[m].y > 0.0f ? 1u : 0u) << (2 * m + 1);
        bb |= (yb[m].x > 0.0f ? 1u : 0u) << (2 * m) | (yb[m].y > 0.0f ? 1u : 0u) << (2 * m + 1);
      }
      const int u = (t * C::HBE + hb) * D + c;
      parts[u * NKG + kg] = (uint8_t)ba;
      parts[(u + 1) * NKG + kg] = (uint8_t)bb;
    }
    wsync();
    const int ncols = (C::SHARED ? 1 : ntile * HB) * D;  // (hash block, column) units
    for (int u = ht; u < ncols; u += NW) {
      uint32_t pattern = 0;
#pragma unroll
      for (int g = 0; g < NKG; ++g) pattern |= (uint32_t)parts[u * NKG + g] << (KG * g);
      const uint32_t bucket = inverse_gray16(pattern);
      const int t = u / (C::HBE * D), hb = (u / D) % C::HBE, c = u % D;
      key_s[u] = (bucket << 8) | (uint32_t)c;
      const int row0 = (qt0 + t) * BM + hb * L;
      if (args.bucket_out && row0 < args.N)
        args.bucket_out[((size_t)bh * args.nqb + row0 / L) * D + c] = (uint16_t)bucket;
    }
    wsync();
    PT(2)
    for (int u = ht; u < ncols; u += NW) {
      const uint4* ks = reinterpret_cast<const uint4*>(key_s + (u / D) * D);
      const uint32_t mine = key_s[u];
      int rank = 0;
#pragma unroll 8
      for (int j = 0; j < D / 4; ++j) {
        const uint4 k4 = ks[j];
        rank += (k4.x < mine ? 1 : 0) + (k4.y < mine ? 1 : 0) + (k4.z < mine ? 1 : 0) + (k4.w < mine ? 1 : 0);
      }
      const int c = u % D;
      perm_s[(u / D) * D + rank] = (uint8_t)c;
      if (C::SHARED) perm_s[D + rank] = (uint8_t)c;  // tile 1 uses the same grouping
      const int qb = ((qt0 + u / (C::HBE * D)) * BM) / L + (u / D) % C::HBE;
      if (args.perm_out && qb < args.nqb)
        args.perm_out[((size_t)bh * args.nqb + qb) * D + rank] = (uint8_t)c;
    }
  } else {
    for (int u = ht; u < ntile * C::HBE * D; u += NW) {
      const int t = u / (C::HBE * D), hb = (u / D) % C::HBE, c = u % D;
      const int qb = (qt0 + t) * BM / L + hb;
      perm_s[u] = (qb < args.nqb) ? args.perm[((size_t)bh * args.nqb + qb) * D + c] : (uint8_t)c;
    }
  }
  wsync();
  PT(3)
  // Q̂[r][j] = Q[r][perm[j G]] (sampling); block_l = 64 stacks the two hash blocks of a tile
  // block-diagonally (columns [hb*d/G*, (hb+1)*d/G*) of rows of hash block hb, zeros elsewhere).
  // Thread ht owns output column pair p = ht % CP (CP divides NW, so p is fixed for the thread)
  // and every (NW/CP)-th row: the 32 lanes of a warp gather from one or a few rows of the staged Q
  // (few bank conflicts) and store 4 bytes each into the swizzled K-major A operand.
  constexpr int CP = C::DR / 2;
  static_assert(NW % CP == 0, "column pairs per worker");
  const int p = ht % CP, j0 = 2 * p;
  const uint32_t dcol = (uint32_t)((j0 / C::A_BOX_COLS) * C::A_BOX_BYTES + (j0 % C::A_BOX_COLS) * 2);
  for (int t = 0; t < ntile; ++t) {
#pragma unroll
    for (int hbr = 0; hbr < (HB == 2 ? 2 : 1); ++hbr) {
      int src[2];  // source columns of the pair (-1: zero, the off-diagonal block of l = 64)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = j0 + e, hbj = j / DG, jj = j % DG;
        src[e] = (HB == 2 && hbj != hbr) ? -1 : perm_s[(t * C::HBE + hbj) * D + jj * G];
      }
      const int rlo = HB == 2 ? 64 * hbr : 0, rhi = HB == 2 ? rlo + 64 : BM;
#pragma unroll 4
      for (int r = rlo + ht / CP; r < rhi; r += NW / CP) {
        const uint32_t v0 = src[0] < 0 ? 0u : *reinterpret_cast<const uint16_t*>(sQ + q_off(t, r, src[0]));
        const uint32_t v1 = src[1] < 0 ? 0u : *reinterpret_cast<const uint16_t*>(sQ + q_off(t, r, src[1]));
        *reinterpret_cast<uint32_t*>(sA + t * C::A_BYTES + swz(dcol + r * C::A_SW, C::A_SWB)) = v0 | (v1 << 16);
      }
    }
  }
  fence_proxy_async_smem();
  warp_arrive(&bars[B_QHAT]);
  PT(4)
#undef PT
}

// EMU: number of every 8 column pairs whose exp2 runs as a polynomial on the FMA pipe instead of
// MUFU.EX2 (16 ex2/clk/SM, one per (query, key) pair — it co-bounds the tile with the tensor
// core; moving EMU/8 of the exps to the FMA pipe rebalances the two).
template <int D, bool DISTR, int G, int HB, int EMU>
__global__ void __launch_bounds__(threads_of<DISTR>(), 1)
    attn_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const AttnArgs args) {
  using C = Cfg<D, DISTR, G, HB>;
  constexpr int NS = C::NS, NKH = C::NKH > 0 ? C::NKH : 1;
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
  long long* const trace = (args.trace && blockIdx.x == 0 && blockIdx.y == 0) ? args.trace : nullptr;
#define DA_TRACE(slot, idx, cond) \
  if (trace && (cond)) trace[(slot) * 256 + ((idx) & 255)] = clock64();
  // Slot of this CTA. Q-block sharding: round x of a zigzag over `stride` ranks (rank `offset`
  // takes slot offset in even rounds, stride-1-offset in odd ones); causal: heaviest pairs first.
  const int npairs = (args.nqt + 1) / 2;
  const int rx = (int)blockIdx.x;
  const int slot = rx * args.pair_stride + ((rx & 1) ? args.pair_stride - 1 - args.pair_offset : args.pair_offset);
  if (slot >= npairs) return;  // past the end in the last round of this shard
  const int pair = args.causal ? (npairs - 1 - slot) : slot;
  const int b = bh / args.H, h = bh % args.H;
  const int bhkv = b * args.H_kv + h / (args.H / args.H_kv);
  const int qt0 = 2 * pair;
  // key tiles each Q tile visits (0 = tile absent)
  int nkt_t[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int qt = qt0 + t;
    nkt_t[t] = qt >= args.nqt ? 0 : (args.causal ? min(qt + 1, args.nkt) : args.nkt);
  }
  const int nk = max(nkt_t[0], nkt_t[1]);

  if (threadIdx.x == 0) {
    mbar_init(&bars[B_Q], 1);
    mbar_init(&bars[B_QHAT], kWorkers / kArrive);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bars[B_KFULL + s], 1);
      mbar_init(&bars[B_KEMPTY + s], DISTR ? kFusionThreads / kArrive : 1);
      mbar_init(&bars[B_VFULL + s], 1);
      mbar_init(&bars[B_VEMPTY + s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      for (int st = 0; st < 2; ++st) {
        mbar_init(&bars[B_KHFULL + 2 * t + st], kFusionThreads / kArrive);
        mbar_init(&bars[B_KHEMPTY + 2 * t + st], 1);
      }
      mbar_init(&bars[B_SFULL + t], 1);
#if DA_PINGPONG
      mbar_init(&bars[B_PFULL + t], kSoftmaxThreads / 2 / kArrive);  // one softmax warpgroup per tile
#else
      mbar_init(&bars[B_PFULL + t], kSoftmaxThreads / kArrive);
#endif
      mbar_init(&bars[B_OFULL + t], 1);
      mbar_init(&bars[B_SLD + t], kSoftmaxThreads / 2);
      mbar_init(&bars[B_PHALF + t], kSoftmaxThreads / 2);
    }
    fence_mbar_init();
    // A operand, issued before anything else: exact -> Q tiles straight into sA; distr -> natural
    // Q tiles into the staging area, from which the 384 worker threads hash the Q blocks and
    // build Q̂ in sA (qhat_prologue).
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    const int ntile = nkt_t[1] > 0 ? 2 : 1;
    if (DISTR) {
      uint8_t* sQ0 = C::STAGE_IN_V ? sV : sK;
      mbar_arrive_expect_tx(&bars[B_Q], ntile * C::QT_BYTES);
      for (int t = 0; t < ntile; ++t)
        for (int bx = 0; bx < D / C::RB; ++bx)
          tma_load_3d(sQ0 + t * C::QT_BYTES + bx * (BM * C::RB * 2), &tmA, &bars[B_Q], bx * C::RB, (qt0 + t) * BM,
                      bh);
    } else {
      mbar_arrive_expect_tx(&bars[B_Q], ntile * C::A_BYTES);
      for (int t = 0; t < ntile; ++t)
        for (int bx = 0; bx < C::A_NBOX; ++bx)
          tma_load_3d(sA + t * C::A_BYTES + bx * C::A_BOX_BYTES, &tmA, &bars[B_Q], bx * C::A_BOX_COLS,
                      (qt0 + t) * BM, bh);
    }
  }
  if (warp == 1) {
    tmem_alloc(tmem_ptr_s, kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr_s;

  uint8_t* sQst = C::STAGE_IN_V ? sV : sK;
  if (DISTR && warp >= 4)
    qhat_prologue<C, D, G, HB>(args, bars, sQst, sA, sKh, perm_s, bh, qt0, nkt_t[1] > 0 ? 2 : 1,
                               (int)threadIdx.x - 128, trace);

  // Register split (SPLIT = 2 only; distr, 512 threads at 128 registers): the TMA/MMA warpgroup
  // gives 64 of its registers to the softmax warpgroups (128*64 + 256*160 + 128*128 = 512*128; an
  // .inc that exceeds what the .dec released would block forever). The exact kernel (384 threads at
  // 168) needs no split. With SPLIT = 4 every thread holds 32 scores and the launch-time budget
  // (80 registers at 768 threads, 96 at 640) suffices. Each setmaxnreg sits at the head of its
  // warpgroup's branch so ptxas budgets each region separately.
  if (warp < 4) {
  if constexpr (kSplit == 2) {
    if (DISTR)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 48;");
    else
      asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
  }
  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      // the staging area overlaps the K ring: wait until Q̂ is built
      if (DISTR && !C::STAGE_IN_V) mbar_wait(&bars[B_QHAT], 0);
      // K^T is written by the prep kernel this grid may overlap (programmatic dependent launch)
      if (DISTR && args.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
      // K (or K^T) ring; V has its own producer (warp 2) so K prefetch never waits behind the
      // PV that frees a V stage.
      for (int i = 0; i < nk; ++i) {
        const int s = i % NS;
        const uint32_t ph = (i / NS) & 1;
        mbar_wait(&bars[B_KEMPTY + s], ph ^ 1);
        mbar_arrive_expect_tx(&bars[B_KFULL + s], C::K_BYTES);
        if (DISTR) {
          tma_load_3d(sK + s * C::K_BYTES, &tmK, &bars[B_KFULL + s], i * BN, 0, bhkv);
        } else {
          for (int bx = 0; bx < C::A_NBOX; ++bx)  // K (G = 1) or K̂ of this query head (global)
            tma_load_3d(sK + s * C::K_BYTES + bx * C::A_BOX_BYTES, &tmK, &bars[B_KFULL + s], bx * C::A_BOX_COLS,
                        i * BN, args.k_per_qhead ? bh : bhkv);
        }
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------------ TMA producer (V ring)
    if (lane == 0) {
      if (DISTR) mbar_wait(&bars[B_QHAT], 0);  // the V ring doubles as the Q staging area
      for (int i = 0; i < nk; ++i) {
        const int s = i % NS;
        const uint32_t ph = (i / NS) & 1;
        mbar_wait(&bars[B_VEMPTY + s], ph ^ 1);
        mbar_arrive_expect_tx(&bars[B_VFULL + s], C::V_BYTES);
        for (int bx = 0; bx < D / C::RB; ++bx)
          tma_load_3d(sV + s * C::V_BYTES + bx * (BN * C::RB * 2), &tmV, &bars[B_VFULL + s], bx * C::RB, i * BN,
                      bhkv);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    // The whole warp runs the issue loop (warp-uniform control flow, so descriptors and indices
    // live in uniform registers and each batch of tcgen05.mma issues back to back); one elected
    // lane issues the MMAs and commits.
    {
      constexpr uint32_t IDESC_S = make_idesc_bf16(BM, BN, false, DISTR);
      constexpr uint32_t IDESC_PV = make_idesc_bf16(BM, D, false, true);
      constexpr int KS = C::A_COLS / 16;       // K-steps of S
      constexpr int kpb = C::A_BOX_COLS / 16;  // K-steps per A box
      const uint32_t a_base = smem_u32(sA);
      const bool lead = lane == 0;
      auto issue_s = [&](int t, int i) {
        const int s = i % NS;
        const int tk = C::SHARED ? 0 : t;  // K̂ buffer set this tile reads
        if (DISTR)
          mbar_wait(&bars[B_KHFULL + 2 * tk + i % NKH], (i / NKH) & 1);
        else if (t == 0 || nkt_t[0] <= i)  // first consumer of K tile i waits for it
          mbar_wait(&bars[B_KFULL + s], (i / NS) & 1);
        tc_fence_after();
        const uint32_t d_s = tmem + kColS + 128u * t;
        uint64_t ad[KS], bd[KS];
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          ad[kk] = make_sdesc(a_base + t * C::A_BYTES + (kk / kpb) * C::A_BOX_BYTES + (kk % kpb) * 32, 16,
                              8 * C::A_SW, C::A_LAYOUT);
          if (DISTR)  // K̂^T as the MN-major B operand: 64-key blocks (LBO = DR*128 B), 8-row groups (SBO)
            bd[kk] = make_sdesc(smem_u32(sKh + (tk * NKH + i % NKH) * C::KH_BYTES) + kk * 2048, C::DR * 128, 1024,
                                kSw128);
          else
            bd[kk] = make_sdesc(smem_u32(sK + s * C::K_BYTES) + (kk / kpb) * C::A_BOX_BYTES + (kk % kpb) * 32, 16,
                                8 * C::A_SW, C::A_LAYOUT);
        }
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < KS; ++kk) mma_ss(d_s, ad[kk], bd[kk], IDESC_S, kk > 0 ? 1u : 0u);
          mma_commit(&bars[B_SFULL + t]);
          // K̂ stage free once its last reader has issued (SHARED: tile 1 if it uses key tile i;
          // tile 1 never uses fewer key tiles than tile 0)
          if (DISTR && (!C::SHARED || t == 1 || i >= nkt_t[1])) mma_commit(&bars[B_KHEMPTY + 2 * tk + i % NKH]);
        }
        __syncwarp();
        if (lead) DA_TRACE(6 + t, i, true);
      };
      auto issue_pv = [&](int t, int j) {
        const int s = j % NS;
#if DA_PV_SPLIT
        // keys 0-63 of P_t(j) as soon as the softmax has stored them
        mbar_wait(&bars[B_PHALF + t], j & 1);
        if (t == 0 || nkt_t[0] <= j) mbar_wait(&bars[B_VFULL + s], (j / NS) & 1);
        tc_fence_after();
        {
          const uint32_t v_base = smem_u32(sV + s * C::V_BYTES);
          const uint32_t p_tmem = tmem + kColS + 128u * t;
          uint64_t vd[BN / 32];
#pragma unroll
          for (int kk = 0; kk < BN / 32; ++kk)
            vd[kk] = make_sdesc(v_base + kk * 16 * C::RB * 2, BN * C::RB * 2, 8 * C::RB * 2, C::RB == 64 ? kSw128 : kSw64);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BN / 32; ++kk)
              mma_ts(tmem + (uint32_t)(t * D), p_tmem + kk * 8, vd[kk], IDESC_PV, (j > 0 || kk > 0) ? 1u : 0u);
          }
          __syncwarp();
        }
        mbar_wait(&bars[B_PFULL + t], j & 1);
        if (lead) DA_TRACE(8 + t, j, true);
        tc_fence_after();
        constexpr int kk0 = BN / 32;  // the second half's K-steps
#else
        mbar_wait(&bars[B_PFULL + t], j & 1);
        if (lead) DA_TRACE(8 + t, j, true);
        if (t == 0 || nkt_t[0] <= j) mbar_wait(&bars[B_VFULL + s], (j / NS) & 1);
        tc_fence_after();
        constexpr int kk0 = 0;
#endif
        const uint32_t v_base = smem_u32(sV + s * C::V_BYTES);
        const uint32_t p_tmem = tmem + kColS + 128u * t + (DA_PINGPONG == 2 ? 64u : 0u);
        uint64_t vd[BN / 16];
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)  // V as the MN-major B operand: RB-column blocks (LBO), 8-key groups (SBO)
          vd[kk] = make_sdesc(v_base + kk * 16 * C::RB * 2, BN * C::RB * 2, 8 * C::RB * 2, C::RB == 64 ? kSw128 : kSw64);
        if (elect_one()) {
#pragma unroll
          for (int kk = kk0; kk < BN / 16; ++kk)
            mma_ts(tmem + (uint32_t)(t * D), p_tmem + kk * 8, vd[kk], IDESC_PV, (j > 0 || kk > 0) ? 1u : 0u);
          if (j == nkt_t[t] - 1) mma_commit(&bars[B_OFULL + t]);
        }
        __syncwarp();
      };
      // release K / V stage i once every tile that uses it has issued its MMA on it
      auto release_k = [&](int i) {
        if (!DISTR) {
          if (elect_one()) mma_commit(&bars[B_KEMPTY + i % NS]);
          __syncwarp();
        }
      };
      auto release_v = [&](int j) {
        if (elect_one()) mma_commit(&bars[B_VEMPTY + j % NS]);
        __syncwarp();
      };

      mbar_wait(&bars[DISTR ? B_QHAT : B_Q], 0);
      tc_fence_after();
#if DA_PINGPONG == 2
      constexpr uint32_t IDESC_SH = make_idesc_bf16(BM, BN / 2, false, DISTR);
      // half h of S_t(i): keys [64h, 64h + 64) -> columns [64h, 64h + 64) of S_t
      auto issue_sh = [&](int t, int i, int h) {
        const int s = i % NS;
        const int tk = C::SHARED ? 0 : t;
        if (h == 0) {
          if (DISTR)
            mbar_wait(&bars[B_KHFULL + 2 * tk + i % NKH], (i / NKH) & 1);
          else if (t == 0 || nkt_t[0] <= i)
            mbar_wait(&bars[B_KFULL + s], (i / NS) & 1);
          tc_fence_after();
        }
        const uint32_t d_s = tmem + kColS + 128u * t + 64u * h;
        uint64_t ad[KS], bd[KS];
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          ad[kk] = make_sdesc(a_base + t * C::A_BYTES + (kk / kpb) * C::A_BOX_BYTES + (kk % kpb) * 32, 16,
                              8 * C::A_SW, C::A_LAYOUT);
          if (DISTR)  // 64-key block h of K̂^T
            bd[kk] = make_sdesc(smem_u32(sKh + (tk * NKH + i % NKH) * C::KH_BYTES) + kk * 2048 + h * (C::DR * 128),
                                C::DR * 128, 1024, kSw128);
          else  // key rows [64h, 64h + 64) of the K tile
            bd[kk] = make_sdesc(smem_u32(sK + s * C::K_BYTES) + (kk / kpb) * C::A_BOX_BYTES + (kk % kpb) * 32 +
                                    h * 64 * C::A_SW,
                                16, 8 * C::A_SW, C::A_LAYOUT);
        }
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < KS; ++kk) mma_ss(d_s, ad[kk], bd[kk], IDESC_SH, kk > 0 ? 1u : 0u);
          if (h == 1) {
            mma_commit(&bars[B_SFULL + t]);
            if (DISTR && (!C::SHARED || t == 1 || i >= nkt_t[1])) mma_commit(&bars[B_KHEMPTY + 2 * tk + i % NKH]);
          }
        }
        __syncwarp();
        if (lead && h == 1) DA_TRACE(6 + t, i, true);
      };
#pragma unroll
      for (int t = 0; t < 2; ++t)
        if (0 < nkt_t[t]) {
          issue_sh(t, 0, 0);
          issue_sh(t, 0, 1);
        }
      if (nk > 0) release_k(0);
      for (int i = 0; i < nk; ++i) {
        // lower halves of step i+1 as soon as each tile's softmax holds S_t(i) in registers
#pragma unroll
        for (int t = 0; t < 2; ++t)
          if (i + 1 < nkt_t[t]) {
            mbar_wait(&bars[B_SLD + t], i & 1);
            issue_sh(t, i + 1, 0);
          }
#pragma unroll
        for (int t = 0; t < 2; ++t)
          if (i < nkt_t[t]) {
            issue_pv(t, i);
            if (t == 1 || !(i < nkt_t[1])) release_v(i);
            if (i + 1 < nkt_t[t]) issue_sh(t, i + 1, 1);  // upper half: in-order after PV_t(i) read P_t(i)
          }
        if (i + 1 < nk) release_k(i + 1);
      }
#else
      for (int i = 0; i < nk; ++i) {
        // tile 0: PV_0(i-1) then S_0(i)   (S_0(i) overwrites P_0(i-1): in-order after the PV)
        if (i >= 1 && i - 1 < nkt_t[0]) issue_pv(0, i - 1);
        if (i >= 1 && !(i - 1 < nkt_t[1])) release_v(i - 1);
        if (i < nkt_t[0]) issue_s(0, i);
        if (i >= 1 && i - 1 < nkt_t[1]) {
          issue_pv(1, i - 1);
          release_v(i - 1);
        }
        if (i < nkt_t[1]) issue_s(1, i);
        release_k(i);
      }
      if (nk - 1 < nkt_t[0]) issue_pv(0, nk - 1);
      if (nk - 1 < nkt_t[1]) issue_pv(1, nk - 1);
      release_v(nk - 1);
#endif
    }
  }  // warp 3 idle
  } else if (warp < 4 + kSoftmaxWarps) {
#if DA_PINGPONG
    static_assert(kSplit == 2, "ping-pong uses the 8 softmax warps as two warpgroups");
    if (DISTR)
      asm volatile("setmaxnreg.inc.sync.aligned.u32 184;");
    else
      asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
    {
      const int t = (warp - 4) >> 2;
      const int nkt = nkt_t[t];
      const int row = (warp & 3) * 32 + lane;
      const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
      const uint32_t tS = tmem + lane_base + kColS + 128u * t;
      const uint32_t tO = tmem + lane_base + (uint32_t)(t * D);
      const int q0 = (qt0 + t) * BM;
      const int q_row = q0 + row;
      const float sl2 = args.scale_log2;
      const bool tr = row == 0;
      float m = -INFINITY, l = 0.0f;
      for (int i = 0; i < nkt; ++i) {
        DA_TRACE(13 + t, i, tr);
        mbar_wait(&bars[B_SFULL + t], i & 1);
        DA_TRACE(3 * t, i, tr);
        tc_fence_after();
        uint32_t sr[BN];
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) tmem_ld32(tS + 32u * c, *reinterpret_cast<uint32_t(*)[32]>(&sr[32 * c]));
        tmem_ld_wait();
#if DA_PINGPONG == 2
        tc_fence_before();
        mbar_arrive(&bars[B_SLD + t]);  // S_t(i) is in registers: the lower half of S_t(i+1) may land
#endif
        float sv[BN];
#pragma unroll
        for (int e = 0; e < BN; ++e) sv[e] = __uint_as_float(sr[e]);
        const int kbase = i * BN;
        if (kbase + BN > args.N || (args.causal && kbase + BN - 1 > q0)) {
          const int lim = args.causal ? min(args.N - 1, q_row) : args.N - 1;
#pragma unroll
          for (int e = 0; e < BN; ++e)
            if (kbase + e > lim) sv[e] = -INFINITY;
        }
        float mx8[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) mx8[j] = max3(sv[j], sv[8 + j], sv[120 + j]);
#pragma unroll
        for (int e = 16; e < 120; e += 16)
#pragma unroll
          for (int j = 0; j < 8; ++j) mx8[j] = max3(mx8[j], sv[e + j], sv[e + 8 + j]);
        const float mx = max3(max3(mx8[0], mx8[1], mx8[2]), max3(mx8[3], mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]));
        const float mnew = fmaxf(m, mx * sl2);
        DA_TRACE(3 * t + 1, i, tr);
        if (i == 0) {
          m = mnew;
        } else {
          const bool need = mnew > m + 8.0f;
          if (__any_sync(0xffffffffu, need)) {
            const float f = need ? ex2(m - mnew) : 1.0f;
#pragma unroll 1
            for (int c = 0; c < D / 16; ++c) {
              uint32_t r[16];
              tmem_ld16(tO + 16u * c, r);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * f);
              tmem_st16(tO + 16u * c, r);
            }
            if (need) {
              l *= f;
              m = mnew;
            }
          }
        }
        const float2 sl2x2 = make_float2(sl2, sl2), nm2 = make_float2(-m, -m);
        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};
        uint32_t pr[64];
        constexpr uint32_t kPcol = DA_PINGPONG == 2 ? 64u : 0u;  // P_t columns inside S_t
#if DA_EXP_SPLIT && DA_PV_SPLIT
        // keys 0-63, then 64-127; in each half the MUFU pairs first, the polynomial pairs after
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
          for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
            for (int e = 32 * hh; e < 32 * hh + 32; ++e) {
              const bool poly = (e & 7) >= 8 - EMU;
              if (poly != (pass == 1)) continue;
              const float2 x = fma2(make_float2(sv[2 * e], sv[2 * e + 1]), sl2x2, nm2);
              const float2 p = poly ? exp2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
              acc[e & 3] = fadd2(acc[e & 3], p);
              pr[e] = pack_bf16x2(p.x, p.y);
            }
          }
          tmem_st32(tS + kPcol + 32u * hh, *reinterpret_cast<uint32_t(*)[32]>(&pr[32 * hh]));
          if (hh == 0) {
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&bars[B_PHALF + t]);
          }
        }
#elif DA_EXP_SPLIT
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
          for (int e = 0; e < 64; ++e) {
            const bool poly = (e & 7) >= 8 - EMU;
            if (poly != (pass == 1)) continue;
            const float2 x = fma2(make_float2(sv[2 * e], sv[2 * e + 1]), sl2x2, nm2);
            const float2 p = poly ? exp2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
            acc[e & 3] = fadd2(acc[e & 3], p);
            pr[e] = pack_bf16x2(p.x, p.y);
          }
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) tmem_st32(tS + kPcol + 32u * c, *reinterpret_cast<uint32_t(*)[32]>(&pr[32 * c]));
#else
#pragma unroll
        for (int e = 0; e < 64; ++e) {
          const float2 x = fma2(make_float2(sv[2 * e], sv[2 * e + 1]), sl2x2, nm2);
          float2 p;
          if ((e & 7) >= 8 - EMU)
            p = exp2_poly2(x);
          else
            p = make_float2(ex2(x.x), ex2(x.y));
          acc[e & 3] = fadd2(acc[e & 3], p);
          pr[e] = pack_bf16x2(p.x, p.y);
          if ((e & 7) == 7) tmem_st8(tS + kPcol + (e - 7), &pr[e - 7]);
        }
#endif
        DA_TRACE(16 + t, i, tr);
        const float2 a = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
        l += a.x + a.y;
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&bars[B_PFULL + t]);
        DA_TRACE(3 * t + 2, i, tr);
      }
      if (nkt > 0) {
        mbar_wait(&bars[B_OFULL + t], 0);
        tc_fence_after();
        const float inv = 1.0f / l;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tO + 32u * c, r);
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
        if (args.lse && q_row < args.N)
          args.lse[(size_t)bh * args.N + q_row] = (m + log2f(l)) * 0.69314718055994531f;
      }
    }
  } else if (false) {
#endif
    if constexpr (kSplit == 2) {
      if (DISTR) asm volatile("setmaxnreg.inc.sync.aligned.u32 160;");
    }
    // ------------------------------------------------------------------ softmax (warps 4..4+4*SPLIT)
    // All softmax warps work on ONE Q tile at a time, alternating tiles (t = 0, 1, 0, 1, ...) in
    // the MMA's issue order. The SPLIT warps w = 4 + quad + 4*part own the same 32 TMEM lanes
    // (rows) and split the 128 key columns: part takes columns [CW*part, CW*part + CW). The row max
    // is combined through shared memory with a (32*SPLIT)-thread named barrier per quad; the
    // running max m is therefore identical in every part, so each part keeps its own partial row
    // sum and rescales its own D/SPLIT columns of O; the parts' sums are combined once, at the end.
    // While these warps run tile t's exp phase the tensor core computes the other tile.
    constexpr int CW = kCW;
    const int part = (warp - 4) >> 2;
    const int quad = warp & 3;
    constexpr int DP = D / kSplit;             // O columns per part
    constexpr int OC = DP >= 32 ? 32 : DP;     // O columns per TMEM load in the rescale / epilogue
    const int row = quad * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    // max [2 parity][2 t][SPLIT][128], sums [2 t][SPLIT][128]
    float* xmax = reinterpret_cast<float*>(bars + B_COUNT);
    float* xsum = xmax + 4 * kSplit * 128;
    const float sl2 = args.scale_log2;
    float m[2] = {-INFINITY, -INFINITY};  // running max per tile (scaled log2; stale by <= 8)
    float l[2] = {0.0f, 0.0f};            // this part's partial row sums
    auto quad_sync = [&]() {  // the SPLIT warps of this quad (same rows, all parts)
      asm volatile("bar.sync %0, %1;" ::"r"(1 + quad), "n"(32 * kSplit) : "memory");
    };
    for (int i = 0; i < nk; ++i) {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (i >= nkt_t[t]) continue;
        const uint32_t tS = tmem + lane_base + kColS + 128u * t + (uint32_t)(CW * part);
        const uint32_t tO = tmem + lane_base + (uint32_t)(t * D) + (uint32_t)(part * DP);
        const int q0 = (qt0 + t) * BM;
        const int q_row = q0 + row;
        DA_TRACE(13 + t, i, row == 0 && part == 0);
        mbar_wait(&bars[B_SFULL + t], i & 1);
        DA_TRACE(3 * t, i, row == 0 && part == 0);
        tc_fence_after();
        uint32_t sr[CW];
#pragma unroll
        for (int c = 0; c < CW / 32; ++c) tmem_ld32(tS + 32u * c, *reinterpret_cast<uint32_t(*)[32]>(&sr[32 * c]));
        tmem_ld_wait();
        float sv[CW];
#pragma unroll
        for (int e = 0; e < CW; ++e) sv[e] = __uint_as_float(sr[e]);
        const int kbase = i * BN + CW * part;
        if (kbase + CW > args.N || (args.causal && kbase + CW - 1 > q0)) {
          const int lim = args.causal ? min(args.N - 1, q_row) : args.N - 1;
#pragma unroll
          for (int e = 0; e < CW; ++e)
            if (kbase + e > lim) sv[e] = -INFINITY;
        }
        // Row max over this part: 8 independent FMNMX3 chains; then combine the parts.
        float mx8[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) mx8[j] = max3(sv[j], sv[8 + j], sv[16 + j]);
#pragma unroll
        for (int e = 24; e + 16 <= CW; e += 16)
#pragma unroll
          for (int j = 0; j < 8; ++j) mx8[j] = max3(mx8[j], sv[e + j], sv[e + 8 + j]);
        static_assert((CW - 24) % 16 == 8, "max tree tail");
#pragma unroll
        for (int j = 0; j < 8; ++j) mx8[j] = fmaxf(mx8[j], sv[CW - 8 + j]);
        float mx = max3(max3(mx8[0], mx8[1], mx8[2]), max3(mx8[3], mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]));
        float* xm = xmax + ((i & 1) * 2 + t) * kSplit * 128 + row;
        xm[part * 128] = mx;
        quad_sync();
#pragma unroll
        for (int o = 1; o < kSplit; ++o) mx = fmaxf(mx, xm[((part + o) % kSplit) * 128]);
        const float mnew = fmaxf(m[t], mx * sl2);
        DA_TRACE(3 * t + 1, i, row == 0 && part == 0);
        if (i == 0) {
          m[t] = mnew;
        } else {
          // S_t(i) was committed after PV_t(i-1) was issued, so O_t holds sum_{<i} P V.
          const bool need = mnew > m[t] + 8.0f;
          if (__any_sync(0xffffffffu, need)) {
            const float f = need ? ex2(m[t] - mnew) : 1.0f;
#pragma unroll
            for (int c = 0; c < DP / OC; ++c) {
              uint32_t r[OC];
              tmem_ldn<OC>(tO + (uint32_t)(OC * c), r);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < OC; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * f);
              tmem_stn<OC>(tO + (uint32_t)(OC * c), r);
            }
            if (need) {
              l[t] *= f;
              m[t] = mnew;
            }
          }
        }
        // p = 2^(s*scale*log2e - m): FFMA2 for the affine part, EMU/8 of the pairs on the FMA
        // pipe, the rest on MUFU; 4 independent FADD2 partial sums.
        const float2 sl2x2 = make_float2(sl2, sl2), nm2 = make_float2(-m[t], -m[t]);
        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};
        uint32_t pr[CW / 2];
#pragma unroll
        for (int e = 0; e < CW / 2; ++e) {
          const float2 x = fma2(make_float2(sv[2 * e], sv[2 * e + 1]), sl2x2, nm2);
          float2 p;
          // polynomial pairs: the last EMU of every 8, or (DA_EMU_SPREAD) spread evenly so the
          // MUFU and FMA-pipe instructions interleave in each warp's stream
          if (DA_EMU_SPREAD ? ((e * EMU) & 7) < EMU : (e & 7) >= 8 - EMU)
            p = exp2_poly2(x);
          else
            p = make_float2(ex2(x.x), ex2(x.y));
          acc[e & 3] = fadd2(acc[e & 3], p);
          pr[e] = pack_bf16x2(p.x, p.y);
          // P of keys [CW*part, CW*part + CW) -> columns [CW/2*part, CW/2*part + CW/2) of S_t,
          // stored in 8-column chunks as they complete so the TMEM writes drain under the
          // remaining exps
          if ((e & 7) == 7)
            tmem_st8(tmem + lane_base + kColS + 128u * t + (uint32_t)(CW / 2 * part) + (e - 7), &pr[e - 7]);
        }
        DA_TRACE(16 + t, i, row == 0 && part == 0);
        const float2 a = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
        l[t] += a.x + a.y;
        tmem_st_wait();
        tc_fence_before();
        warp_arrive(&bars[B_PFULL + t]);
        DA_TRACE(3 * t + 2, i, row == 0 && part == 0);
      }
    }
    // Epilogue: all parts' row sums, each part writes its D/SPLIT output columns.
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if (nkt_t[t] == 0) continue;
      const int q_row = (qt0 + t) * BM + row;
      const uint32_t tO = tmem + lane_base + (uint32_t)(t * D) + (uint32_t)(part * DP);
      float* xs = xsum + t * kSplit * 128 + row;
      xs[part * 128] = l[t];
      quad_sync();
      float lt = l[t];
#pragma unroll
      for (int o = 1; o < kSplit; ++o) lt += xs[((part + o) % kSplit) * 128];
      mbar_wait(&bars[B_OFULL + t], 0);
      tc_fence_after();
      const float inv = 1.0f / lt;
#pragma unroll
      for (int c = 0; c < DP / OC; ++c) {
        uint32_t r[OC];
        tmem_ldn<OC>(tO + (uint32_t)(OC * c), r);
        tmem_ld_wait();
        if (q_row < args.N) {
          const size_t off = ((size_t)bh * args.N + q_row) * D + part * DP + OC * c;
          if (args.out_f32) {
            float4* o = reinterpret_cast<float4*>(static_cast<float*>(args.out) + off);
#pragma unroll
            for (int e = 0; e < OC / 4; ++e)
              o[e] = make_float4(__uint_as_float(r[4 * e]) * inv, __uint_as_float(r[4 * e + 1]) * inv,
                                 __uint_as_float(r[4 * e + 2]) * inv, __uint_as_float(r[4 * e + 3]) * inv);
          } else {
            uint4* o = reinterpret_cast<uint4*>(static_cast<uint16_t*>(args.out) + off);
#pragma unroll
            for (int e = 0; e < OC / 8; ++e)
              o[e] = make_uint4(pack_bf16x2(__uint_as_float(r[8 * e]) * inv, __uint_as_float(r[8 * e + 1]) * inv),
                                pack_bf16x2(__uint_as_float(r[8 * e + 2]) * inv, __uint_as_float(r[8 * e + 3]) * inv),
                                pack_bf16x2(__uint_as_float(r[8 * e + 4]) * inv, __uint_as_float(r[8 * e + 5]) * inv),
                                pack_bf16x2(__uint_as_float(r[8 * e + 6]) * inv, __uint_as_float(r[8 * e + 7]) * inv));
          }
        }
      }
      if (args.lse && q_row < args.N && part == 0)
        args.lse[(size_t)bh * args.N + q_row] = (m[t] + log2f(lt)) * 0.69314718055994531f;
    }
  } else {
#if DA_PINGPONG
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;");
#endif
    // ------------------------------------------------------------------ fusion (warps 12..15)
    // Thread f owns 16-byte chunk ch = f % 16 (8 keys) of K̂^T rows j = f/16 + 8n, n < DR/8.
    // Its source-row byte offsets (perm rows * 256 + ch * 16) are fixed for the CTA's lifetime,
    // so the per-tile work is G 16-byte loads, a bf16x2 add chain and one 16-byte store per task.
    // 16 lanes read one whole 256-byte K^T row (conflict-free); stores land in the UMMA
    // MN-major SWIZZLE_128B layout (chunk ^= row % 8, row % 8 == f/16 for every task).
    if (DISTR) {
      const int f = threadIdx.x - (128 + kSoftmaxThreads);
      const int ch = f & 15, jb = f >> 4;
      constexpr int NT = C::DR / 8;  // tasks per thread per (tile, key tile)
      constexpr int DG = D / G;
      constexpr int NW = (NT * G + 1) / 2;
      uint32_t offs[2][NW];  // packed u16 source offsets, entry e = n*G + g
#pragma unroll
      for (int t = 0; t < 2; ++t) {
#pragma unroll
        for (int w = 0; w < NW; ++w) offs[t][w] = 0;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const int j = jb + 8 * n, hb = j / DG, jj = j % DG;
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const int e = n * G + g;
            const uint32_t o = (uint32_t)perm_s[(t * C::HBE + hb) * D + jj * G + g] * (BN * 2) + ch * 16;
            offs[t][e >> 1] |= o << (16 * (e & 1));
          }
        }
      }
      const uint32_t dbase = (uint32_t)((ch >> 3) * (C::DR * 128) + jb * 128 + (((ch & 7) ^ jb) << 4));
      for (int i = 0; i < nk; ++i) {
        const int s = i % NS;
        mbar_wait(&bars[B_KFULL + s], (i / NS) & 1);
        DA_TRACE(10, i, f == 0);
        const uint8_t* kt = sK + s * C::K_BYTES;
#pragma unroll
        for (int t = 0; t < C::NKT; ++t) {  // SHARED: one K̂ for both Q tiles (i < nk: someone uses it)
          if (!C::SHARED && i >= nkt_t[t]) continue;
          const int st = i % NKH;
          mbar_wait(&bars[B_KHEMPTY + 2 * t + st], ((i / NKH) & 1) ^ 1);
          uint8_t* kh = sKh + (t * NKH + st) * C::KH_BYTES + dbase;
          if constexpr (DA_DIAG_NOFUSE) {
            // diagnostic only (wrong results): no fusion work, to measure its interference
          } else
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            uint32_t src[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
              const int e = n * G + g;
              src[g] = (offs[t][e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
            }
            uint4 o;
            if (G == 1) {
              o = *reinterpret_cast<const uint4*>(kt + src[0]);
            } else if (G == 2) {
              // one RN rounding of the exact sum == RN(fp32 sum) for two bf16 operands
              const uint4 x = *reinterpret_cast<const uint4*>(kt + src[0]);
              const uint4 y = *reinterpret_cast<const uint4*>(kt + src[G - 1]);
              o = make_uint4(hadd2_bf16(x.x, y.x), hadd2_bf16(x.y, y.y), hadd2_bf16(x.z, y.z), hadd2_bf16(x.w, y.w));
            } else {
              float acc[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
#pragma unroll
              for (int g = 0; g < G; ++g) {
                const uint4 x = *reinterpret_cast<const uint4*>(kt + src[g]);
                const uint32_t xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) add_bf16x2_f32(xv[e], acc[2 * e], acc[2 * e + 1]);
              }
              o = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]), pack_bf16x2(acc[4], acc[5]),
                             pack_bf16x2(acc[6], acc[7]));
            }
            *reinterpret_cast<uint4*>(kh + n * 1024) = o;
          }
          fence_proxy_async_smem();
          warp_arrive(&bars[B_KHFULL + 2 * t + st]);
          DA_TRACE(11 + t, i, f == 0);
        }
        warp_arrive(&bars[B_KEMPTY + s]);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

template <int D, bool DISTR, int G, int HB, int EMU>
cudaError_t launch_one(const AttnLaunch& L, const AttnArgs& a, cudaStream_t st) {
  using C = Cfg<D, DISTR, G, HB>;
  auto kern = attn_kernel<D, DISTR, G, HB, EMU>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  const int npairs = (a.nqt + 1) / 2;
  dim3 grid((npairs + a.pair_stride - 1) / a.pair_stride, L.BH);  // rounds of the zigzag
  if (!a.pdl) {
    kern<<<grid, threads_of<DISTR>(), C::SMEM, st>>>(*L.tmA, *L.tmK, *L.tmV, a);
    return cudaGetLastError();
  }
  // programmatic dependent launch: CTAs may start (and hash their Q blocks) while the K^T prep
  // kernel still runs; the K producer waits on the grid dependency before its first K^T load
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads_of<DISTR>());
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, *L.tmA, *L.tmK, *L.tmV, a);
}

template <int D, bool DISTR, int G, int HB>
constexpr size_t smem_of() {
  return (size_t)Cfg<D, DISTR, G, HB>::SMEM;
}

}  // namespace

#define DA_DISPATCH(MACRO)                                                          \
  if (!distr) {                                                                     \
    if (d == 32 && G == 1) MACRO(32, false, 1, 1);                                  \
    if (d == 32 && G == 2) MACRO(32, false, 2, 1);                                  \
    if (d == 64 && G == 1) MACRO(64, false, 1, 1);                                  \
    if (d == 64 && G == 2) MACRO(64, false, 2, 1);                                  \
    if (d == 64 && G == 4) MACRO(64, false, 4, 1);                                  \
    if (d == 128 && G == 1) MACRO(128, false, 1, 1);                                \
    if (d == 128 && G == 2) MACRO(128, false, 2, 1);                                \
    if (d == 128 && G == 4) MACRO(128, false, 4, 1);                                \
    if (d == 128 && G == 8) MACRO(128, false, 8, 1);                                \
  } else {                                                                          \
    if (d == 32 && G == 1 && HB == 1) MACRO(32, true, 1, 1);                        \
    if (d == 32 && G == 1 && HB == 2) MACRO(32, true, 1, 2);                        \
    if (d == 32 && G == 2 && HB == 1) MACRO(32, true, 2, 1);                        \
    if (d == 32 && G == 2 && HB == 2) MACRO(32, true, 2, 2);                        \
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
    if (d == 128 && G == 8 && HB == 1) MACRO(128, true, 8, 1);                      \
    if (d == 128 && G == 8 && HB == 2) MACRO(128, true, 8, 2);                      \
    if (d == 32 && G == 2 && HB == 0) MACRO(32, true, 2, 0);                        \
    if (d == 64 && G == 2 && HB == 0) MACRO(64, true, 2, 0);                        \
    if (d == 64 && G == 4 && HB == 0) MACRO(64, true, 4, 0);                        \
    if (d == 128 && G == 2 && HB == 0) MACRO(128, true, 2, 0);                      \
    if (d == 128 && G == 4 && HB == 0) MACRO(128, true, 4, 0);                      \
  }

size_t attn_smem_bytes(int d, int G, int HB, int distr) {
#define DA_SMEM(D_, DI_, G_, HB_) return smem_of<D_, DI_, G_, HB_>()
  DA_DISPATCH(DA_SMEM)
#undef DA_SMEM
  return 0;
}

template <int D, bool DI, int G, int HB>
AttnConfig config_of() {
  using C = Cfg<D, DI, G, HB>;
  return AttnConfig{C::DR, C::NS, C::NKH, threads_of<DI>(), C::SMEM};
}

bool attn_config(int d, int G, int HB, int distr, AttnConfig* out) {
#define DA_CFG(D_, DI_, G_, HB_) \
  {                              \
    *out = config_of<D_, DI_, G_, HB_>(); \
    return true;                 \
  }
  DA_DISPATCH(DA_CFG)
#undef DA_CFG
  return false;
}

cudaError_t launch_attn(const AttnLaunch& L, const AttnArgs& a, cudaStream_t st) {
  const int d = L.d, G = L.G, HB = L.HB, distr = L.distr;
  // EMU (pairs of 8 on the FMA pipe): default per flavour, overridable for tuning (DA_EMU env).
  const int emu = L.emu;
#define DA_LAUNCH(D_, DI_, G_, HB_)                                                \
  switch (emu) {                                                                   \
    case 0: return launch_one<D_, DI_, G_, HB_, 0>(L, a, st);                      \
    case 2: return launch_one<D_, DI_, G_, HB_, 2>(L, a, st);                      \
    case 3: return launch_one<D_, DI_, G_, HB_, 3>(L, a, st);                      \
    default: return launch_one<D_, DI_, G_, HB_, 4>(L, a, st);                     \
  }
  DA_DISPATCH(DA_LAUNCH)
#undef DA_LAUNCH
  return cudaErrorInvalidValue;
}

}  // namespace da
