/*
 * oracle.c — CPU ORACLE for DistrAttention (arXiv 2507.17245). TEST INFRASTRUCTURE ONLY.
 *
 * This file is the plain, slow, obviously-correct reference that the CUDA path is checked
 * against. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it. It shares NO code, header, table or constant generator with
 * paper_2507_17245_b200/ (the product path); the product never loads this library.
 *
 * Citation convention: "P:<line> (§x)" = /root/reference/PAPER.md line, "S:<line>" = SPEC.md.
 * Readings taken where the paper is silent/ambiguous are listed in DESIGN.md §3 and repeated
 * beside the function that applies them.
 *
 * Precision: projections are an fp32 fma chain (the one place where the result must be
 * bit-exact with the GPU, reading R6); everything downstream (fusion, scores,
 * softmax, PV) is computed in double.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared (no -ffast-math).
 *
 * Parity pins (tests/test_oracle_*.py, -m "not gpu"):
 *   oracle_projection   — N(0,1) moments + KS test, determinism; pinned (statistics).
 *   oracle_gray_rank    — bijection on 2^16, Hamming-1 adjacency, S:128-130 examples.
 *   oracle_hash_block   — zero column -> 0, 2^k scaling invariance, sign symmetry,
 *                          agreement with an fp64 numpy projection on margin columns.
 *   oracle_sort_perm    — Fig. 5 worked example, stability.
 *   oracle_distr_scores — G*=1 == QK^T, duplicated columns exact (Eq. 1), distributive
 *                          identity vs expanded-Q GEMM, d=6 brute force (Eq. 3), Tables 3-4 band.
 *   oracle_attn_items   — torch fp64 SDPA (exact), N=1, S=0 column mean, causal row 0, GQA.
 *
 * Global grouping ("a unique grouping strategy over the complete Q and K^T", DESIGN.md
 * reading R17) needs no separate code: it is this block-wise method with block_l = N (one hash
 * block spanning every row of the head, projection (seed, N)).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#if defined(__x86_64__)
#include <xmmintrin.h>
#endif

#define NPRIME 16 /* N' = 16 hash bits ("N' is set to 16") */

/* Reading R7: no flush-to-zero / denormals-are-zero on either side. The oracle may be
 * loaded into a process (torch) that changed MXCSR, so clear FTZ (bit 15) and DAZ (bit 6). */
static void clear_ftz_daz(void) {
#if defined(__x86_64__)
  _mm_setcsr(_mm_getcsr() & ~((1u << 15) | (1u << 6)));
#endif
}

int oracle_ftz_daz_clear(void) {
#if defined(__x86_64__)
  clear_ftz_daz();
  return (_mm_getcsr() & ((1u << 15) | (1u << 6))) == 0;
#else
  return 1;
#endif
}

/* ---------------------------------------------------------------------------------------------
 * Projection matrix ("The projection matrix is randomly generated in prior";
 * S:113-117 build_projection: i.i.d. standard normal, built once, reused by every block/head).
 * Reading R4: SplitMix64 counter stream, n-th draw = mix(seed + (n+1)*golden); uniform
 * u = (top 53 bits + 0.5) * 2^-53 in (0,1); Box-Muller in double on consecutive pairs
 * (z0 = r cos(2 pi u2), z1 = r sin(2 pi u2), r = sqrt(-2 ln u1)); entries filled row-major [k][r]
 * (k < 16 projection rows, r < block_l); each z rounded to fp32.
 * ------------------------------------------------------------------------------------------- */
static uint64_t splitmix64_draw(uint64_t seed, uint64_t n) {
  uint64_t z = seed + (n + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static double uniform_open01(uint64_t seed, uint64_t n) {
  return ((double)(splitmix64_draw(seed, n) >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}

void oracle_projection(uint64_t seed, int block_l, float* out /* [16][block_l] */) {
  const int total = NPRIME * block_l; /* always even */
  for (int e = 0; e < total; e += 2) {
    double u1 = uniform_open01(seed, (uint64_t)e);
    double u2 = uniform_open01(seed, (uint64_t)e + 1);
    double r = sqrt(-2.0 * log(u1));
    double th = 6.283185307179586476925286766559 * u2;
    out[e] = (float)(r * cos(th));
    out[e + 1] = (float)(r * sin(th));
  }
}

/* ---------------------------------------------------------------------------------------------
 * Gray-code table lookup ("the binary sequence is used as the index to select a value from
 * a table of Gray code at the size of 2^N'"). Reading R2: the table maps a bit pattern to its rank
 * in the binary-reflected Gray sequence, i.e. the inverse of g = b ^ (b >> 1):
 * rank = b ^ (b>>1) ^ (b>>2) ^ ... Written out as the definition: XOR of all right shifts.
 * ------------------------------------------------------------------------------------------- */
uint32_t oracle_gray_rank(uint32_t pattern) {
  uint32_t rank = 0;
  for (int s = 0; s < 32; ++s) rank ^= pattern >> s;
  return rank;
}

/* ---------------------------------------------------------------------------------------------
 * LSH of one Q block (block-wise grouping P:304-306 §3.3).
 *   y_k,c = sum_{r < rows} P[k][r] * q[r][c]   as an fp32 fma chain, ascending r, from +0.0f (R6)
 *   bit_k = (y_k,c > 0)                         strictly positive -> 1, "the others" -> 0 (R5)
 *   pattern = sum_k bit_k << k                  bit k = projection row k, LSB first (R3)
 *   bucket_c = gray_rank(pattern)
 * A ragged last block (rows < block_l) uses only its rows == zero padding (R9).
 * q: row-major [rows][ldq] fp32 (exact upcast of the kernel's input), proj: [16][block_l].
 * ------------------------------------------------------------------------------------------- */
void oracle_hash_block(const float* q, int rows, int ldq, int d, const float* proj, int block_l,
                       uint16_t* bucket /* [d] */) {
  (void)block_l;
  for (int c = 0; c < d; ++c) {
    uint32_t pattern = 0;
    for (int k = 0; k < NPRIME; ++k) {
      float y = 0.0f;
      for (int r = 0; r < rows; ++r) y = fmaf(proj[k * block_l + r], q[(size_t)r * ldq + c], y);
      if (y > 0.0f) pattern |= 1u << k;
    }
    bucket[c] = (uint16_t)oracle_gray_rank(pattern);
  }
}

/* Permutation ("The hash values are monotonically sorted and thus an index permutation of
 * represented columns is generated"; Fig. 5). Reading R8: stable ascending sort, ties in
 * column order. Written as a plain insertion sort over (bucket, column). */
void oracle_sort_perm(const uint16_t* bucket, int d, uint8_t* perm /* [d] */) {
  int idx[256];
  for (int c = 0; c < d; ++c) idx[c] = c;
  for (int a = 1; a < d; ++a) {
    int cur = idx[a];
    int b = a - 1;
    while (b >= 0 && bucket[idx[b]] > bucket[cur]) { /* strict > keeps equal keys in order */
      idx[b + 1] = idx[b];
      --b;
    }
    idx[b + 1] = cur;
  }
  for (int c = 0; c < d; ++c) perm[c] = (uint8_t)idx[c];
}

/* Hash every Q block of Q [B,H,N,d] (fp32). buckets/perm: [B*H][ceil(N/block_l)][d]. */
int oracle_hash(const float* q, int B, int H, int N, int d, int block_l, uint64_t seed,
                uint16_t* buckets, uint8_t* perm) {
  if (!q || B <= 0 || H <= 0 || N <= 0 || d <= 0 || d > 256 || block_l <= 0) return 1;
  clear_ftz_daz();
  float* proj = (float*)malloc(sizeof(float) * NPRIME * block_l);
  oracle_projection(seed, block_l, proj);
  const int nqb = (N + block_l - 1) / block_l;
  const long total = (long)B * H * nqb;
#pragma omp parallel for schedule(dynamic, 4)
  for (long it = 0; it < total; ++it) {
    clear_ftz_daz();
    long bh = it / nqb;
    int qb = (int)(it % nqb);
    int r0 = qb * block_l;
    int rows = (N - r0) < block_l ? (N - r0) : block_l;
    uint16_t bk[256];
    oracle_hash_block(q + ((size_t)bh * N + r0) * d, rows, d, d, proj, block_l, bk);
    if (buckets) memcpy(buckets + (size_t)it * d, bk, sizeof(uint16_t) * d);
    if (perm) oracle_sort_perm(bk, d, perm + (size_t)it * d);
  }
  free(proj);
  return 0;
}

/* ---------------------------------------------------------------------------------------------
 * Approximate scores of one Q block against keys [0, nk) (Eq. 2; §3.2).
 * Groups (R10): G_j = { perm[j G*], ..., perm[j G* + G* - 1] }, representative = perm[j G*]
 *   sampling: qhat_j = q[:, rep_j]                      (exact copy)
 *   fusion:   khat_j = sum_{i in G_j} k[:, i]           (K columns — R1: P:288 says "v", Eq. 2 /
 *                                                         Fig. 4 / P:309 say K; V is never reduced)
 *   shat[r][t] = scale * sum_j qhat_j[r] * khat_j[t]   (double)
 * q: [rows][ldq], k: [nk][ldk]; out: [rows][nk] double.
 * ------------------------------------------------------------------------------------------- */
void oracle_grouped_scores(const float* q, int rows, int ldq, const float* k, int nk, int ldk, int d,
                           int G, const uint8_t* perm, double scale, double* out) {
  const int ng = d / G;
  double* khat = (double*)malloc(sizeof(double) * (size_t)nk * ng);
  for (int t = 0; t < nk; ++t)
    for (int j = 0; j < ng; ++j) {
      double acc = 0.0;
      for (int g = 0; g < G; ++g) acc += (double)k[(size_t)t * ldk + perm[j * G + g]];
      khat[(size_t)t * ng + j] = acc;
    }
  for (int r = 0; r < rows; ++r)
    for (int t = 0; t < nk; ++t) {
      double acc = 0.0;
      for (int j = 0; j < ng; ++j) acc += (double)q[(size_t)r * ldq + perm[j * G]] * khat[(size_t)t * ng + j];
      out[(size_t)r * nk + t] = scale * acc;
    }
  free(khat);
}

/* Exact scores S = scale * q k^T (§2.1) in double. */
static void exact_scores(const float* q, int rows, int ldq, const float* k, int nk, int ldk, int d,
                         double scale, double* out) {
  for (int r = 0; r < rows; ++r)
    for (int t = 0; t < nk; ++t) {
      double acc = 0.0;
      for (int c = 0; c < d; ++c) acc += (double)q[(size_t)r * ldq + c] * (double)k[(size_t)t * ldk + c];
      out[(size_t)r * nk + t] = scale * acc;
    }
}

/* Ŝ for one Q block computed end to end from the raw block (hash -> perm -> grouped scores).
 * Used by the Tables 3-4 band pin (unscaled scores) and the brute-force pin. */
int oracle_distr_scores(const float* q, int rows, int ldq, const float* k, int nk, int ldk, int d,
                        int block_l, int G, uint64_t seed, double scale, double* out, uint8_t* perm_out) {
  if (G <= 0 || d % G != 0 || d > 256 || rows > block_l) return 2;
  clear_ftz_daz();
  float* proj = (float*)malloc(sizeof(float) * NPRIME * block_l);
  oracle_projection(seed, block_l, proj);
  uint16_t bk[256];
  uint8_t perm[256];
  oracle_hash_block(q, rows, ldq, d, proj, block_l, bk);
  oracle_sort_perm(bk, d, perm);
  oracle_grouped_scores(q, rows, ldq, k, nk, ldk, d, G, perm, scale, out);
  if (perm_out) memcpy(perm_out, perm, d);
  free(proj);
  return 0;
}

/* ---------------------------------------------------------------------------------------------
 * Attention output for a list of work items (one item = one Q block of one (b, h)).
 *   G == 0 : exact attention, O = softmax(scale * Q K^T) V              (§2.1)
 *   G >= 1 : DistrAttention, O = softmax(Ŝ) V with Ŝ from Eq. 2 using the block's own grouping
 *            (§3.3: "across Q blocks, we generate different permutations"); V is
 *            used at full d (R1).
 * Masks (R11): causal keeps keys t <= r (N_q == N_k); applied after the approximation. Key head
 * for query head h is h / (H / H_kv) (GQA). Softmax: row max subtracted, exp, normalised, all in
 * double (masked entries contribute 0).
 * items: n_items pairs (bh, qb) with bh = b*H + h. out: [n_items][block_l][d] double (rows past N
 * untouched). lse (optional): [n_items][block_l] natural-log sum-exp of the scaled scores.
 * ------------------------------------------------------------------------------------------- */
int oracle_attn_items(const float* q, const float* k, const float* v, int B, int H, int H_kv, int N,
                      int d, int block_l, int G, uint64_t seed, int causal, double scale,
                      const int* items, int n_items, double* out, double* lse) {
  if (!q || !k || !v || !items || !out) return 1;
  if (B <= 0 || H <= 0 || H_kv <= 0 || N <= 0 || d <= 0 || block_l <= 0 || H % H_kv) return 1;
  if (G < 0 || (G > 0 && d % G) || d > 256) return 2;
  clear_ftz_daz();
  const int nqb = (N + block_l - 1) / block_l;
  float* proj = (float*)malloc(sizeof(float) * NPRIME * block_l);
  oracle_projection(seed, block_l, proj);
  const int grp = H / H_kv;
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int it = 0; it < n_items; ++it) {
    clear_ftz_daz();
    const int bh = items[2 * it], qb = items[2 * it + 1];
    if (bh < 0 || bh >= B * H || qb < 0 || qb >= nqb) {
      bad = 1;
      continue;
    }
    const int b = bh / H, h = bh % H;
    const size_t kvh = (size_t)b * H_kv + h / grp;
    const float* qh = q + (size_t)bh * N * d;
    const float* kh = k + kvh * N * d;
    const float* vh = v + kvh * N * d;
    const int r0 = qb * block_l;
    const int rows = (N - r0) < block_l ? (N - r0) : block_l;
    const float* qblk = qh + (size_t)r0 * d;
    double* s = (double*)malloc(sizeof(double) * (size_t)rows * N);
    if (G == 0) {
      exact_scores(qblk, rows, d, kh, N, d, d, scale, s);
    } else {
      uint16_t bk[256];
      uint8_t perm[256];
      oracle_hash_block(qblk, rows, d, d, proj, block_l, bk);
      oracle_sort_perm(bk, d, perm);
      oracle_grouped_scores(qblk, rows, d, kh, N, d, d, G, perm, scale, s);
    }
    for (int r = 0; r < rows; ++r) {
      const int qi = r0 + r;
      const int nvalid = causal ? qi + 1 : N;
      double* srow = s + (size_t)r * N;
      double m = -INFINITY;
      for (int t = 0; t < nvalid; ++t) m = srow[t] > m ? srow[t] : m;
      double l = 0.0;
      for (int t = 0; t < nvalid; ++t) {
        srow[t] = exp(srow[t] - m);
        l += srow[t];
      }
      double* orow = out + ((size_t)it * block_l + r) * d;
      for (int c = 0; c < d; ++c) orow[c] = 0.0;
      for (int t = 0; t < nvalid; ++t) {
        const double p = srow[t] / l;
        const float* vrow = vh + (size_t)t * d;
        for (int c = 0; c < d; ++c) orow[c] += p * (double)vrow[c];
      }
      if (lse) lse[(size_t)it * block_l + r] = m + log(l);
    }
    free(s);
  }
  free(proj);
  return bad ? 1 : 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
