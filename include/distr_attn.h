/*
 * distr_attn.h — C-ABI boundary of the B200 (sm_100a) DistrAttention forward hot path.
 *
 * DistrAttention (arXiv 2507.17245, /root/reference/PAPER.md "P:<line>"): for every query block
 * of block_l rows, the d columns of Q are hashed with a 16-bit sign-random-projection LSH over the
 * block's rows and Gray-ranked, stably sorted into groups of G* (Fig. 5), one
 * representative Q column per group is sampled and the group's K columns are sum-fused (P:288,
 * Eq. 2), and the reduced-d scores feed a blocked online-softmax attention with a
 * full-d PV (Fig. 3). Readings of ambiguous passages: DESIGN.md §3.
 *
 * Conventions for every entry point below
 *   - Tensor pointers are DEVICE pointers on the current CUDA device unless the name says host.
 *     Q and O are [B, H, N, d] contiguous; K and V are [B, H_kv, N, d] contiguous
 *     (H % H_kv == 0; query head h reads KV head h / (H / H_kv)). Element type = params.dtype
 *     (DA_BF16: bfloat16, DA_F32: float; fp32 inputs are hashed in fp32 and rounded to bf16
 *     for the tensor-core contractions, output written in fp32).
 *   - The caller owns q, k, v, out, lse and the export buffers; the library owns its projection
 *     cache and, when workspace == NULL, stream-ordered scratch: cudaMallocAsync on the call's
 *     stream before the launches and cudaFreeAsync after them, from the device's default memory
 *     pool (its release threshold is raised once per device, so steady-state calls neither
 *     cudaMalloc nor synchronise). The first use of a (seed, block_l) projection allocates and
 *     uploads it synchronously (cudaMalloc + cudaMemcpy) — do that once before graph capture.
 *   - Calls are stream-ordered and asynchronous (`cuda_stream` is a cudaStream_t, NULL = legacy
 *     default stream); synchronisation is the caller's job. Nothing throws across the ABI.
 *   - Every argument is validated before anything is enqueued. On DA_ERR_INVALID /
 *     DA_ERR_PRECONDITION nothing was enqueued and `out` is untouched. DA_ERR_CUDA means a CUDA
 *     call failed (detail in distr_attn_last_error()); `out` is then unspecified.
 *   - Thread safety: the projection cache is mutex-protected; library scratch is per call and
 *     stream-ordered, so concurrent calls on different streams / host threads never share it. A
 *     caller-owned workspace must not be used by two calls that can run concurrently.
 *
 * Supported envelope: d in {32, 64, 128}; block_l in {64, 128, 256}; G* (group_size) in {1, 2, 4, 8}
 * with d % G* == 0 and the reduced width max(1, 128 / block_l) * d / G* in [16, 128]; block_l = 256
 * (one hash block = the 256 query rows one CTA owns, so both of its 128-row tiles share one
 * grouping and one fused K̂ per key tile; P:306's "Q block" at the B200 CTA granularity) takes
 * G* in {2, 4}; any N >= 1 (ragged tails handled); any B, H >= 1 with B*H, B*H_kv < 65536.
 */
#ifndef DISTR_ATTN_H
#define DISTR_ATTN_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (mirroring the SPEC CLI convention S:537: 1 usage, 2 precondition, 3 runtime). */
enum {
  DA_OK = 0,
  DA_ERR_INVALID = 1,      /* null pointer, non-positive dims, H % H_kv != 0, bad dtype flag */
  DA_ERR_PRECONDITION = 2, /* d % G* != 0, reduced width < 16, unsupported
                              d / block_l / G*, workspace too small */
  DA_ERR_CUDA = 3          /* a CUDA runtime/driver call failed */
};

enum { DA_BF16 = 0, DA_F32 = 1 };

typedef struct da_params {
  int B, H, H_kv, N, d;        /* shapes, see above */
  int block_l;                 /* Q-block height l: hashing block AND outer-loop block */
  int group_size;              /* G*: constant group size */
  unsigned long long seed;     /* projection-matrix seed ("randomly generated in prior") */
  int causal;                  /* 0/1: query i attends keys 0..i (N_q == N_k); mask applied
                                  after the approximation (reading R11) */
  float scale;                 /* score scale; <= 0 selects 1/sqrt(d) with the ORIGINAL d (R12) */
  int dtype;                   /* DA_BF16 | DA_F32 (inputs and output) */
  void* workspace;             /* optional caller-owned device workspace; NULL = library pool */
  size_t workspace_bytes;      /* size of `workspace` (>= distr_attn_workspace_size()) */
  float* lse;                  /* optional [B, H, N] fp32 natural-log sum-exp of scaled scores */
  unsigned short* bucket_ids;  /* optional [B, H, ceil(N/l), d] uint16 LSH bucket ids (tests) */
  unsigned char* perm;         /* optional [B, H, ceil(N/l), d] uint8 stable sort permutation */
  int q_shard_offset;          /* Q-block (sequence) sharding: with stride S > 0 */
  int q_shard_stride;          /* this call computes only the 256-row Q tile pairs dealt to rank
                                  `offset` of S in a zigzag: slot x*S + offset for even rounds x,
                                  x*S + S-1-offset for odd x (slots are visited heaviest-first when
                                  causal, so the split balances causal work). 0 / 0 (the defaults)
                                  = all pairs. Rows outside the shard are not written (out, lse).
                                  Requires 0 <= offset < stride when stride > 0. */
} da_params;

/* Fill `p` with defaults: H_kv = H, non-causal, bf16, scale = 1/sqrt(d), library workspace,
 * no exports. Returns DA_OK, or DA_ERR_INVALID if p is NULL. */
int distr_attn_init_params(da_params* p, int B, int H, int N, int d, int block_l, int group_size,
                           unsigned long long seed);

/* North-star entry point (BASELINE.json): DistrAttention forward with H_kv = H, non-causal,
 * bf16, scale 1/sqrt(d), legacy default stream, library-managed workspace. */
int distr_attn_fwd(const void* q, const void* k, const void* v, void* out, int B, int H, int N,
                   int d, int block_l, int group_size, unsigned long long seed);

/* DistrAttention forward, all options. Launches, on `cuda_stream`:
 *   bf16 inputs (2 launches): (1) prep_kernel = the K^T layout pass only ([B*H_kv][d][N_pad]
 *     bf16 in the workspace); (2) the fused tcgen05 attention kernel, whose CTAs each hash their
 *     own Q blocks in shared memory (projection fp32 fma chain -> sign bits -> inverse Gray ->
 *     stable rank -> perm -> sampled Q̂; exports bucket_ids / perm when set) and then run the
 *     per-tile fusion of K columns, the reduced-d QK^T, the online softmax and the full-d PV.
 *   fp32 inputs (4 launches): a bf16 conversion of V; prep_kernel hashing the fp32 Q blocks
 *     (-> perm workspace + exports) and the K^T pass; a bf16 conversion of Q; the attention
 *     kernel reading the perm instead of hashing. */
int distr_attn_fwd_ex(const void* q, const void* k, const void* v, void* out, const da_params* p,
                      void* cuda_stream);

/* Same as distr_attn_fwd_ex, but q/k/v/out (and lse/bucket_ids/perm if set) are HOST pointers.
 * The job is cut into chunks of whole KV heads (b, h_kv) with their query heads; per chunk the
 * inputs are copied to a library-owned device staging slot on an internal copy stream, the
 * forward runs on `cuda_stream`, and the results are copied back on a second internal copy
 * stream, through 3 slots, so the copies of neighbouring chunks overlap the kernels (the
 * double buffering of P:749). Bit-identical to distr_attn_fwd_ex on the same data. With a
 * Q-tile-pair shard only the shard's rows of out / lse (and its blocks of the exports) are
 * written. Returns after all work has completed. Host buffers should be pinned (cudaHostAlloc /
 * torch pin_memory), otherwise the copies are synchronous. One host call runs at a time per
 * process (internal mutex). */
int distr_attn_fwd_host(const void* q, const void* k, const void* v, void* out,
                        const da_params* p, void* cuda_stream);

/* Exact softmax attention (§2.1) on the same sm_100a tiling (G* ignored, no prep for
 * bf16 inputs): the reference point for the speed-up. */
int exact_attn_fwd_ex(const void* q, const void* k, const void* v, void* out, const da_params* p,
                      void* cuda_stream);

/* DistrAttention with GLOBAL grouping ("a unique grouping strategy over the complete Q
 * and K^T", which the paper reports as less accurate than block-wise grouping):
 * one LSH per (b, h) over all N rows (projection 16 x N from (seed, N); reading R17), one
 * permutation per head, Q̂ and K̂ = grouped sums of K columns materialised once per query head in
 * the workspace, then attention with S contracted over d/G* and no per-tile fusion. Same
 * params as distr_attn_fwd_ex except: bf16 only, block_l is not used by the method (tiles are 128
 * rows) but must be valid, and the optional bucket_ids / perm exports are [B, H, 1, d].
 * Workspace: distr_attn_workspace_size() covers it. Status codes as distr_attn_fwd_ex. */
int distr_attn_global_fwd_ex(const void* q, const void* k, const void* v, void* out, const da_params* p,
                             void* cuda_stream);

/* Backward pass of DistrAttention (reading R18: the grouping of each Q
 * block is held constant, so dQ lands on the representative columns only and every member of a
 * group receives its fused column's dK). Inputs: the forward's q, k, v, out and its natural-log
 * LSE (da_params.lse of the forward call, [B, H, N] fp32), and dout = dL/dout; outputs dq
 * [B,H,N,d], dk, dv [B,H_kv,N,d] (bf16, overwritten). Same params as the forward (block_l,
 * group_size, seed select the grouping; causal, scale; group_size = 1 gives exact attention
 * gradients). bf16 only, d in {32, 64, 128}: five launches of this library's kernels — the prep
 * hash (perm per Q block), Q̃ (every column replaced by its group representative) + D =
 * rowsum(dO*O), the LSE scaled by -log2(e) and padded with -inf, the fused tcgen05 dK/dV kernel,
 * and the fused tcgen05 dQ̃ kernel, whose epilogue folds dQ̃ onto the representative columns and
 * writes dq; stream-ordered, no host sync.
 * Workspace: the caller's (p->workspace, >= distr_attn_bwd_workspace_size(p) bytes) or
 * stream-ordered library scratch. */
int distr_attn_bwd_ex(const void* q, const void* k, const void* v, const void* out, const void* dout,
                      const float* lse, void* dq, void* dk, void* dv, const da_params* p, void* cuda_stream);

/* Run only the LSH step of the prep kernel and export p->bucket_ids and/or p->perm (at least one
 * must be non-NULL). Bit-exact contract with the CPU oracle (fp32 fma chain, ascending rows). */
int distr_attn_hash(const void* q, const da_params* p, void* cuda_stream);

/* Host-side copy of the projection matrix for (seed, block_l): host_out = float[16 * block_l],
 * row-major [k][r]. SplitMix64 counter stream + Box-Muller in double rounded to fp32 (R4). */
int distr_attn_projection(unsigned long long seed, int block_l, float* host_out);

/* Device workspace bytes needed by distr_attn_fwd_ex / exact_attn_fwd_ex /
 * distr_attn_global_fwd_ex for these params (0 if the params are invalid). Host-only. */
size_t distr_attn_workspace_size(const da_params* p);

/* Device workspace bytes distr_attn_bwd_ex needs for these params (0 if invalid). Host-only. */
size_t distr_attn_bwd_workspace_size(const da_params* p);

/* Block-size planner: the B200 analogue of "Block size selection" (§3.3.1, Eq. 4-5,
 * Table 2). Host-only (no CUDA call, no GPU needed). For (N, d, block_l, group_size, distr) it
 * reports the tiling the attention kernel is compiled with and the quantities the paper's rules
 * are stated in, re-derived for tcgen05/TMEM/TMA:
 *   - I/O model (unnumbered equation): I(l, m) = N/l * (l d + 2 N d + l d) elements, i.e.
 *     each Q block re-reads all of K and V; on B200 the two Q tiles of a CTA share every K/V tile
 *     and the re-reads across CTAs of a head are served by the 126 MB L2, so HBM sees Q, K, V, O
 *     about once (plus the K^T layout pass for distr);
 *   - Eq. 4: l, m multiples of the tensor-core tile N' -> l = UMMA M = 128 rows per Q
 *     tile (block_l = 64 stacks two hash blocks in one tile), m = UMMA N of S, a multiple of 16
 *     and <= 256;
 *   - Eq. 5: enough work per SM to keep the tensor core busy -> two Q tiles per CTA (the
 *     softmax of one overlaps the MMAs of the other), subject to TMEM (tiles * (d + m) <= 512
 *     columns) and shared memory (Q/Q̂ tiles + K/V ring + K̂ ring <= 227 KB per CTA).
 * distr = 0 describes the exact kernel (group_size ignored). Returns DA_OK, DA_ERR_INVALID (NULL
 * out, N < 1) or DA_ERR_PRECONDITION (combination outside the supported envelope). */
typedef struct da_plan {
  int tile_m;            /* query rows per Q tile (UMMA M) */
  int tiles_per_cta;     /* Q tiles per CTA */
  int tile_n;            /* keys per K/V tile: m (UMMA N of S, K of PV) */
  int s_width;           /* contraction width of S: d (exact) or max(1, 128 / block_l) * d / G* */
  int kv_stages;         /* K (or K^T) and V TMA ring depth */
  int khat_stages;       /* fused K̂^T buffers per Q tile (distr) */
  int threads;           /* threads per CTA */
  int smem_bytes;        /* dynamic shared memory per CTA */
  int tmem_cols;         /* TMEM columns allocated per CTA */
  int m_max_tmem;        /* largest m (multiple of 16, <= 256) the TMEM budget admits at tiles_per_cta */
  int ctas;              /* CTAs of one launch for (B*H = 1, N) */
  double mma_clk_per_tile;   /* ideal tcgen05 clk per 128 x m tile: 2*128*m*(s_width + d) / 8192 */
  double exp_clk_per_tile;   /* MUFU clk for the tile's 128*m exp2 at 16 per clk per SM */
  double fusion_smem_bytes_per_tile; /* distr: K^T tile read + K̂^T tile written per (Q tile, K tile) */
  double hbm_bytes_paper;    /* I(l, m) * 2 bytes for one head (bf16), l = block_l */
  double hbm_bytes_b200;     /* one head on this kernel: Q + K + V + O (+ K^T write and read, distr) */
} da_plan;
int distr_attn_plan(int N, int d, int block_l, int group_size, int distr, da_plan* out);

/* Planner that CHOOSES (the Table 2 step of §3.3.1, decided on B200 by a cost model
 * calibrated on this build's kernels): for a job (B, H, H_kv, N, d, causal) it
 * predicts the forward time of the exact kernel and of every DistrAttention setting with
 * block_l in {64 (d <= 64), 128, 256} and G* in {2, 4, 8} up to max_group_size (the caller's
 * accuracy bound: G* = 1 is exact attention, error grows with G*, Tables 3-4), and returns the
 * fastest. Model per CTA (two 128-row Q tiles): prologue clk + key-tile steps x step clk (CTA
 * timelines, tools/calibrate.sh), CTAs list-scheduled over 148 SMs at clk_mhz (<= 0: 1800), plus
 * the K^T pass (HBM-bound) and launch overhead; DistrAttention is chosen only when predicted >= 2 %
 * faster than the exact kernel (the model's spread; exact attention is the more accurate). Host-only. Returns DA_OK, DA_ERR_INVALID (NULL
 * out, non-positive dims, H % H_kv) or DA_ERR_PRECONDITION (d not in {32, 64, 128}). */
typedef struct da_choice {
  int distr;                  /* 1: DistrAttention (block_l, group_size below); 0: exact kernel */
  int block_l;                /* chosen Q-block height (0 when distr = 0) */
  int group_size;             /* chosen G* (1 when distr = 0) */
  double predicted_us;        /* predicted forward time of the choice */
  double predicted_exact_us;  /* predicted forward time of the exact kernel */
  double predicted_distr_us;  /* fastest DistrAttention setting's predicted time */
} da_choice;
int distr_attn_choose(int B, int H, int H_kv, int N, int d, int causal, int max_group_size, double clk_mhz,
                      da_choice* out);

/* Static description of a status code. */
const char* distr_attn_status_string(int status);

/* Thread-local detail of the last error raised on the calling thread ("" if none). */
const char* distr_attn_last_error(void);

/* Number of kernel launches the last successful forward call on this thread enqueued. */
int distr_attn_last_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* DISTR_ATTN_H */
