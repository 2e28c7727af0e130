// api.cu — the C-ABI declared in include/distr_attn.h: validation, projection matrix, workspace,
// TMA descriptors and launches. Host code only; kernels live in prep.cu / attn.cu.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/distr_attn.h"
#include "../../include/distr_attn_profile.h"
#include "internal.h"

namespace {

thread_local std::string g_last_error;
thread_local int g_last_launches = 0;
thread_local cudaEvent_t g_ev[3] = {nullptr, nullptr, nullptr};
thread_local long long* g_trace = nullptr;

void record_ev(int i, cudaStream_t st) {
  if (g_ev[i]) cudaEventRecord(g_ev[i], st);
}

int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return status;
}

#define DA_CUDA(expr)                                                                               \
  do {                                                                                              \
    cudaError_t e_ = (expr);                                                                        \
    if (e_ != cudaSuccess)                                                                          \
      return fail(DA_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

// ---------------------------------------------------------------------------- projection (R4)
// SplitMix64 counter stream: n-th draw = mix(seed + (n + 1) * 0x9E3779B97F4A7C15); uniform in
// (0,1) from the top 53 bits + 0.5; Box-Muller on consecutive pairs in double; rounded to fp32;
// entries row-major [k][r]. (Independent implementation of the same generator as the oracle.)
inline uint64_t sm64_mix(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
void make_projection(uint64_t seed, int block_l, float* out) {
  const uint64_t gamma = 0x9E3779B97F4A7C15ULL;
  const int n = 16 * block_l;
  uint64_t ctr = seed;
  for (int e = 0; e < n; e += 2) {
    ctr += gamma;
    const double u1 = (double)(sm64_mix(ctr) >> 11) * 0x1.0p-53 + 0x1.0p-54;
    ctr += gamma;
    const double u2 = (double)(sm64_mix(ctr) >> 11) * 0x1.0p-53 + 0x1.0p-54;
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double ang = 6.283185307179586476925286766559 * u2;
    out[e] = (float)(rad * std::cos(ang));
    out[e + 1] = (float)(rad * std::sin(ang));
  }
}

std::mutex g_mu;
// (device, seed, block_l) -> device ptr. Block-wise projections (block_l <= 256) are few and kept
// for the process lifetime; the global variant's [16][N] projections (one per sequence length)
// are kept in a small LRU: evicting one waits for the device to go idle first (a kernel in
// flight may still read it).
std::map<std::tuple<int, uint64_t, int>, float*> g_proj;
std::vector<std::tuple<int, uint64_t, int>> g_proj_lru;  // global-variant keys, oldest first
constexpr size_t kGlobalProjKeep = 8;

int get_projection(int dev, uint64_t seed, int block_l, cudaStream_t st, const float** out) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_tuple(dev, seed, block_l);
  auto it = g_proj.find(key);
  if (it != g_proj.end()) {
    if (block_l > 256) {  // refresh LRU position
      for (size_t i = 0; i < g_proj_lru.size(); ++i)
        if (g_proj_lru[i] == key) {
          g_proj_lru.erase(g_proj_lru.begin() + i);
          break;
        }
      g_proj_lru.push_back(key);
    }
    *out = it->second;
    return DA_OK;
  }
  if (block_l > 256 && g_proj_lru.size() >= kGlobalProjKeep) {
    const auto old = g_proj_lru.front();
    DA_CUDA(cudaDeviceSynchronize());
    DA_CUDA(cudaFree(g_proj[old]));
    g_proj.erase(old);
    g_proj_lru.erase(g_proj_lru.begin());
  }
  std::vector<float> h(16 * (size_t)block_l);
  make_projection(seed, block_l, h.data());
  float* d = nullptr;
  DA_CUDA(cudaMalloc(&d, h.size() * sizeof(float)));
  // Synchronous copy on first use of (seed, block_l) only; never on the steady-state path.
  DA_CUDA(cudaMemcpy(d, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
  (void)st;
  g_proj[key] = d;
  if (block_l > 256) g_proj_lru.push_back(key);
  *out = d;
  return DA_OK;
}

// Library-managed scratch is stream-ordered: cudaMallocAsync on the call's stream before the
// launches, cudaFreeAsync after them, from the device's default memory pool (release threshold
// raised once per device so the pool keeps its memory between calls: no cudaMalloc /
// synchronisation on the steady-state path). Calls on different streams or host threads never
// share scratch, and a scratch block is reused only after the stream work that used it.
struct Scratch {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  ~Scratch() {
    if (p) cudaFreeAsync(p, st);
  }
};
int scratch_alloc(Scratch& sc, size_t bytes, int dev, cudaStream_t st) {
  {
    static std::vector<int> configured;
    std::lock_guard<std::mutex> lk(g_mu);
    bool done = false;
    for (int d : configured) done |= d == dev;
    if (!done) {
      cudaMemPool_t pool;
      DA_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
      uint64_t thr = ~0ull;
      DA_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
      configured.push_back(dev);
    }
  }
  DA_CUDA(cudaMallocAsync(&sc.p, bytes, st));
  sc.st = st;
  return DA_OK;
}

// ---------------------------------------------------------------------------- plan
struct Plan {
  int B, H, Hkv, N, d, l, G, HB, DR, nqb, nqt, nkt, N_pad, f32, causal;
  int KHB;  // attention-kernel HB: 128/block_l, or 0 for block_l = 256 (one grouping per CTA)
  int pair_off, pair_stride;  // Q-tile-pair shard (stride 1 = all pairs)
  float scale;
  size_t off_perm, off_qhat, off_kt, off_qc, off_kc, off_vc, total;
};

inline size_t al256(size_t x) { return (x + 255) / 256 * 256; }

int validate(const da_params* p, bool distr, Plan* P) {
  if (!p) return fail(DA_ERR_INVALID, "params is NULL");
  if (p->B <= 0 || p->H <= 0 || p->H_kv <= 0 || p->N <= 0 || p->d <= 0 || p->block_l <= 0)
    return fail(DA_ERR_INVALID, "non-positive dimension (B=%d H=%d H_kv=%d N=%d d=%d block_l=%d)", p->B, p->H,
                p->H_kv, p->N, p->d, p->block_l);
  if (p->H % p->H_kv) return fail(DA_ERR_INVALID, "H (%d) not a multiple of H_kv (%d)", p->H, p->H_kv);
  if (p->dtype != DA_BF16 && p->dtype != DA_F32) return fail(DA_ERR_INVALID, "dtype %d", p->dtype);
  if (p->causal != 0 && p->causal != 1) return fail(DA_ERR_INVALID, "causal must be 0/1");
  if ((long long)p->B * p->H >= 65536 || (long long)p->B * p->H_kv >= 65536)
    return fail(DA_ERR_INVALID, "B*H too large");
  if (p->d != 32 && p->d != 64 && p->d != 128)
    return fail(DA_ERR_PRECONDITION, "d=%d unsupported (32|64|128)", p->d);
  if (p->block_l != 64 && p->block_l != 128 && p->block_l != 256)
    return fail(DA_ERR_PRECONDITION, "block_l=%d unsupported (64|128|256)", p->block_l);
  const int G = distr ? p->group_size : 1;
  if (distr) {
    if (G <= 0) return fail(DA_ERR_INVALID, "group_size=%d", G);
    if (p->d % G) return fail(DA_ERR_PRECONDITION, "d %% G* != 0 (d=%d, G*=%d)", p->d, G);
    if (G != 1 && G != 2 && G != 4 && G != 8) return fail(DA_ERR_PRECONDITION, "G*=%d unsupported (1|2|4|8)", G);
    if (p->d / G < 16) return fail(DA_ERR_PRECONDITION, "d/G* = %d < 16", p->d / G);
    if (p->block_l == 256 && G != 2 && G != 4)
      return fail(DA_ERR_PRECONDITION, "block_l=256 supports G* in {2,4} (got %d)", G);
  }
  Plan& q = *P;
  q.B = p->B; q.H = p->H; q.Hkv = p->H_kv; q.N = p->N; q.d = p->d; q.l = p->block_l; q.G = G;
  q.HB = p->block_l >= 128 ? 1 : 128 / p->block_l;
  q.KHB = p->block_l == 256 ? 0 : q.HB;
  q.DR = q.HB * q.d / G;
  if (distr && (q.DR > 128 || q.DR < 16))
    return fail(DA_ERR_PRECONDITION, "reduced width (128/block_l)*d/G* = %d outside [16,128]", q.DR);
  q.nqb = (q.N + q.l - 1) / q.l;
  q.nqt = (q.N + 127) / 128;
  q.nkt = (q.N + 127) / 128;
  q.N_pad = (q.N + 7) / 8 * 8;
  q.f32 = p->dtype == DA_F32;
  q.causal = p->causal;
  if (p->q_shard_stride < 0 || (p->q_shard_stride == 0 && p->q_shard_offset != 0) ||
      (p->q_shard_stride > 0 && (p->q_shard_offset < 0 || p->q_shard_offset >= p->q_shard_stride)))
    return fail(DA_ERR_INVALID, "q shard offset %d / stride %d", p->q_shard_offset, p->q_shard_stride);
  q.pair_off = p->q_shard_offset;
  q.pair_stride = p->q_shard_stride > 0 ? p->q_shard_stride : 1;
  q.scale = p->scale > 0.f ? p->scale : (float)(1.0 / std::sqrt((double)q.d));
  const size_t BH = (size_t)q.B * q.H, BHkv = (size_t)q.B * q.Hkv;
  size_t o = 0;
  q.off_perm = q.off_qhat = q.off_kt = q.off_qc = q.off_kc = q.off_vc = 0;
  if (distr) {
    // bf16: the attention CTA hashes its own Q blocks, only K^T is precomputed.
    // fp32: the prep kernel hashes the fp32 values (bit-exact contract) -> perm; Q, V -> bf16.
    if (q.f32) { q.off_perm = o; o = al256(o + BH * q.nqb * q.d); }
    q.off_kt = o; o = al256(o + BHkv * q.d * q.N_pad * 2);
    if (q.f32) { q.off_qc = o; o = al256(o + BH * q.N * q.d * 2); }
  } else if (q.f32) {
    q.off_qc = o; o = al256(o + BH * q.N * q.d * 2);
    q.off_kc = o; o = al256(o + BHkv * q.N * q.d * 2);
  }
  if (q.f32) { q.off_vc = o; o = al256(o + BHkv * q.N * q.d * 2); }
  q.total = o;
  return DA_OK;
}

// ---------------------------------------------------------------------------- TMA descriptors
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int get_encode(EncodeTiledFn* fn) {
  static EncodeTiledFn cached = nullptr;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    if (err == cudaSuccess && q == cudaDriverEntryPointSuccess) cached = reinterpret_cast<EncodeTiledFn>(f);
  });
  if (!cached) return fail(DA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (%s)", cudaGetErrorString(err));
  *fn = cached;
  return DA_OK;
}

// 3-D bf16 tensor [d2][d1][d0] (d0 innermost), box {b0, b1, 1}.
int make_map(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1,
             int swizzle_bytes) {
  EncodeTiledFn enc;
  if (int s = get_encode(&enc)) return s;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * 2, d0 * d1 * 2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUtensorMapSwizzle sw = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(DA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) dims=[%llu,%llu,%llu] box=[%u,%u]", (int)r,
                (unsigned long long)d0, (unsigned long long)d1, (unsigned long long)d2, b0, b1);
  return DA_OK;
}

int current_device(int* dev) {
  DA_CUDA(cudaGetDevice(dev));
  return DA_OK;
}

// Share of exp2 pairs (out of 8) evaluated by polynomial on the FMA pipe instead of MUFU.EX2.
// The exp phase of a tile is MUFU-bound (16 ex2/clk/SM); moving 2/8 of the pairs to the FMA pipe
// shortens it. With the round-2 alternating softmax the exact kernel was best at 0 (its longer
// tensor block co-bound it, profiles/r01_v9/emu_ab); with the ping-pong softmax (one warp per SM
// sub-partition per tile) both flavours are best at 2. DA_EMU (distr) and DA_EMU_EXACT (exact)
// override (0, 2, 3, 4) for tuning.
int default_emu(const Plan& P, bool distr) {
  static const int env[2] = {[] {
                               const char* e = getenv("DA_EMU_EXACT");
                               return e ? atoi(e) : -1;
                             }(),
                             [] {
                               const char* e = getenv("DA_EMU");
                               return e ? atoi(e) : -1;
                             }()};
  (void)P;
  if (env[distr ? 1 : 0] >= 0) return env[distr ? 1 : 0];
  // ping-pong softmax (attn.cu, the default): EMU = 2 is the best setting of both flavours
  // (C5, alternating runs on one box, profiles/r02_v6/fwd_ab2: exact EMU 0 / 2 = 118.8 / 117.7 ms)
  return 2;
}

// ---------------------------------------------------------------------------- forward
int forward(const void* q, const void* k, const void* v, void* out, const da_params* p, cudaStream_t st,
            bool distr) {
  Plan P;
  if (int s = validate(p, distr, &P)) return s;
  if (!q || !k || !v || !out) return fail(DA_ERR_INVALID, "null tensor pointer");
  int dev;
  if (int s = current_device(&dev)) return s;
  uint8_t* ws = nullptr;
  Scratch sc;  // freed (stream-ordered) after the launches below
  if (P.total) {
    if (p->workspace) {
      if (p->workspace_bytes < P.total)
        return fail(DA_ERR_PRECONDITION, "workspace too small (%zu < %zu)", p->workspace_bytes, P.total);
      ws = static_cast<uint8_t*>(p->workspace);
    } else {
      if (int s = scratch_alloc(sc, P.total, dev, st)) return s;
      ws = static_cast<uint8_t*>(sc.p);
    }
  }
  const float* proj = nullptr;
  if (distr)
    if (int s = get_projection(dev, p->seed, P.l, st, &proj)) return s;

  const size_t BH = (size_t)P.B * P.H, BHkv = (size_t)P.B * P.Hkv;
  int launches = 0;
  record_ev(0, st);
  const void* kv_v = v;
  if (P.f32) {
    uint16_t* vc = reinterpret_cast<uint16_t*>(ws + P.off_vc);
    DA_CUDA(da::launch_convert_bf16(static_cast<const float*>(v), vc, BHkv * P.N * P.d, st));
    ++launches;
    kv_v = vc;
  }
  const void* a_src;
  const void* k_src;
  if (distr) {
    da::PrepArgs a{};
    a.q = q; a.k = k; a.in_f32 = P.f32;
    a.BH = (int)BH; a.BHkv = (int)BHkv; a.N = P.N; a.d = P.d; a.block_l = P.l; a.G = P.G; a.HB = P.HB;
    a.DR = P.DR; a.nqb = P.nqb; a.N_pad = P.N_pad; a.proj = proj;
    a.kt = reinterpret_cast<uint16_t*>(ws + P.off_kt);
    a.n_kt_ctas = (int)(BHkv * ((P.N + 63) / 64));
    if (P.f32) {  // hash the fp32 values in the prep kernel; the attention kernel reads perm
      a.perm_ws = ws + P.off_perm;
      a.bucket_out = p->bucket_ids;
      a.perm_out = p->perm;
      a.n_hash_ctas = (int)(BH * P.nqb);
    }
    DA_CUDA(da::launch_prep(a, st));
    ++launches;
    if (P.f32) {
      uint16_t* qc = reinterpret_cast<uint16_t*>(ws + P.off_qc);
      DA_CUDA(da::launch_convert_bf16(static_cast<const float*>(q), qc, BH * P.N * P.d, st));
      ++launches;
      a_src = qc;
    } else {
      a_src = q;
    }
    k_src = a.kt;
  } else if (P.f32) {
    uint16_t* qc = reinterpret_cast<uint16_t*>(ws + P.off_qc);
    uint16_t* kc = reinterpret_cast<uint16_t*>(ws + P.off_kc);
    DA_CUDA(da::launch_convert_bf16(static_cast<const float*>(q), qc, BH * P.N * P.d, st));
    DA_CUDA(da::launch_convert_bf16(static_cast<const float*>(k), kc, BHkv * P.N * P.d, st));
    launches += 2;
    a_src = qc;
    k_src = kc;
  } else {
    a_src = q;
    k_src = k;
  }

  CUtensorMap tmA, tmK, tmV;
  const uint32_t rb = P.d >= 64 ? 64 : (uint32_t)P.d;  // natural-row box: 64 columns (32 for d = 32)
  if (int s = make_map(&tmA, a_src, P.d, P.N, BH, rb, 128, (int)rb * 2)) return s;  // natural Q tiles
  if (distr) {
    if (int s = make_map(&tmK, k_src, P.N_pad, P.d, BHkv, 128, P.d, 0)) return s;
  } else {
    if (int s = make_map(&tmK, k_src, P.d, P.N, BHkv, rb, 128, (int)rb * 2)) return s;
  }
  if (int s = make_map(&tmV, kv_v, P.d, P.N, BHkv, rb, 128, (int)rb * 2)) return s;

  da::AttnArgs aa{};
  aa.N = P.N; aa.H = P.H; aa.H_kv = P.Hkv; aa.nqt = P.nqt; aa.nkt = P.nkt; aa.nqb = P.nqb; aa.block_l = P.l;
  aa.pair_offset = P.pair_off; aa.pair_stride = P.pair_stride;
  aa.scale_log2 = P.scale * 1.4426950408889634f;
  aa.causal = P.causal;
  aa.perm = (distr && P.f32) ? ws + P.off_perm : nullptr;
  aa.proj = distr ? proj : nullptr;
  aa.bucket_out = (distr && !P.f32) ? p->bucket_ids : nullptr;
  aa.perm_out = (distr && !P.f32) ? p->perm : nullptr;
  aa.out = out;
  aa.out_f32 = P.f32;
  aa.lse = p->lse;
  aa.trace = g_trace;
  g_trace = nullptr;
  // bf16 distr: the attention kernel overlaps the K^T pass (its prologue reads only Q); not when
  // profile events sit between the two launches (bench.py's kernel split) or DA_PDL=0
  static const bool pdl_env = [] {
    const char* e = getenv("DA_PDL");
    return !(e && e[0] == '0');
  }();
  aa.pdl = distr && !P.f32 && pdl_env && !g_ev[1];
  da::AttnLaunch L{P.d, P.G, distr ? P.KHB : 1, distr ? 1 : 0, (int)BH, &tmA, &tmK, &tmV, default_emu(P, distr)};
  record_ev(1, st);
  DA_CUDA(da::launch_attn(L, aa, st));
  record_ev(2, st);
  g_ev[0] = g_ev[1] = g_ev[2] = nullptr;
  ++launches;
  g_last_launches = launches;
  return DA_OK;
}

// Workspace of the global-grouping variant: perm [BH][d] u8, sign patterns [BH][d] u16, Q̂ and K̂
// [BH][N][d/G*] bf16.
size_t global_ws_bytes(const Plan& P, size_t* off_qhat, size_t* off_khat) {
  const size_t BH = (size_t)P.B * P.H, DR = (size_t)P.d / P.G;
  size_t o = al256(BH * P.d) + al256(BH * P.d * 2);
  *off_qhat = o;
  o = al256(o + BH * P.N * DR * 2);
  *off_khat = o;
  return al256(o + BH * P.N * DR * 2);
}

int forward_global(const void* q, const void* k, const void* v, void* out, const da_params* p, cudaStream_t st) {
  Plan P;
  if (!p) return fail(DA_ERR_INVALID, "params is NULL");
  da_params pg = *p;  // block_l is not used by the global variant: validate its tiling (128 rows)
  pg.block_l = 128;
  if (int s = validate(&pg, true, &P)) return s;
  if (!q || !k || !v || !out) return fail(DA_ERR_INVALID, "null tensor pointer");
  if (P.f32) return fail(DA_ERR_PRECONDITION, "global grouping: bf16 inputs only");
  int dev;
  if (int s = current_device(&dev)) return s;
  size_t off_qh, off_kh;
  const size_t need = global_ws_bytes(P, &off_qh, &off_kh);
  uint8_t* ws;
  Scratch sc;
  if (p->workspace) {
    if (p->workspace_bytes < need)
      return fail(DA_ERR_PRECONDITION, "workspace too small (%zu < %zu)", p->workspace_bytes, need);
    ws = static_cast<uint8_t*>(p->workspace);
  } else {
    if (int s = scratch_alloc(sc, need, dev, st)) return s;
    ws = static_cast<uint8_t*>(sc.p);
  }
  const float* proj = nullptr;  // one projection over all N rows: (seed, N) -> [16][N]
  if (int s = get_projection(dev, p->seed, P.N, st, &proj)) return s;
  const size_t BH = (size_t)P.B * P.H, BHkv = (size_t)P.B * P.Hkv;
  const int DR = P.d / P.G;
  record_ev(0, st);
  da::GlobalArgs g{};
  g.q = static_cast<const uint16_t*>(q);
  g.k = static_cast<const uint16_t*>(k);
  g.BH = (int)BH; g.H = P.H; g.Hkv = P.Hkv; g.N = P.N; g.d = P.d; g.G = P.G;
  g.proj = proj;
  g.perm = ws;
  g.gpat = reinterpret_cast<uint16_t*>(ws + al256(BH * P.d));
  g.bucket_out = p->bucket_ids;
  g.perm_out = p->perm;
  g.qhat = reinterpret_cast<uint16_t*>(ws + off_qh);
  g.khat = reinterpret_cast<uint16_t*>(ws + off_kh);
  DA_CUDA(da::launch_global_prep(g, st));
  // the exact-flavour kernel with S contracted over DR = d/G* (A = Q̂, B = K̂, both K-major)
  const int sw = DR * 2 >= 128 ? 128 : DR * 2;
  CUtensorMap tmA, tmK, tmV;
  if (int s = make_map(&tmA, g.qhat, DR, P.N, BH, sw / 2, 128, sw)) return s;
  if (int s = make_map(&tmK, g.khat, DR, P.N, BH, sw / 2, 128, sw)) return s;
  const uint32_t rb = P.d >= 64 ? 64 : (uint32_t)P.d;
  if (int s = make_map(&tmV, v, P.d, P.N, BHkv, rb, 128, (int)rb * 2)) return s;
  da::AttnArgs aa{};
  aa.N = P.N; aa.H = P.H; aa.H_kv = P.Hkv; aa.nqt = P.nqt; aa.nkt = P.nkt; aa.nqb = P.nqb; aa.block_l = P.l;
  aa.pair_offset = P.pair_off; aa.pair_stride = P.pair_stride;
  aa.scale_log2 = P.scale * 1.4426950408889634f;
  aa.causal = P.causal;
  aa.k_per_qhead = 1;  // K̂ is materialised per query head
  aa.out = out;
  aa.lse = p->lse;
  aa.trace = g_trace;
  g_trace = nullptr;
  da::AttnLaunch L{P.d, P.G, 1, 0, (int)BH, &tmA, &tmK, &tmV, default_emu(P, true)};
  record_ev(1, st);
  DA_CUDA(da::launch_attn(L, aa, st));
  record_ev(2, st);
  g_ev[0] = g_ev[1] = g_ev[2] = nullptr;
  g_last_launches = 3;
  return DA_OK;
}

// Backward workspace: the caller's (p->workspace, at least distr_attn_bwd_workspace_size bytes) or
// stream-ordered library scratch.
constexpr int kSizeOnly = 100;      // internal status: size query answered, nothing launched
thread_local bool g_bwd_size_only = false;
thread_local size_t g_bwd_query = 0;
int bwd_workspace(const da_params* p, size_t need, int* dev, cudaStream_t st, Scratch& sc, uint8_t** ws) {
  if (g_bwd_size_only) {
    g_bwd_query = need;
    return kSizeOnly;
  }
  if (int s = current_device(dev)) return s;
  if (p->workspace) {
    if (p->workspace_bytes < need)
      return fail(DA_ERR_PRECONDITION, "backward workspace too small (%zu < %zu)", p->workspace_bytes, need);
    *ws = static_cast<uint8_t*>(p->workspace);
    return DA_OK;
  }
  if (int s = scratch_alloc(sc, need, *dev, st)) return s;
  *ws = static_cast<uint8_t*>(sc.p);
  return DA_OK;
}

// Fused tcgen05 backward (bwd_fused.cu): hash -> Q̃ + D + padded lse -> dK/dV kernel -> dQ̃ kernel
// (dQ̃ folded onto the representatives in its epilogue). d in {32, 64, 128}.
int backward_fused(const void* q, const void* k, const void* v, const void* o, const void* dout, const float* lse,
                   void* dq, void* dk, void* dv, const da_params* p, const Plan& P, cudaStream_t st) {
  int dev = 0;
  const size_t BH = (size_t)P.B * P.H, BHkv = (size_t)P.B * P.Hkv, N = P.N, d = P.d;
  const size_t N_pad = (N + 127) / 128 * 128;
  size_t o_ = 0;
  auto take = [&](size_t bytes) { size_t at = o_; o_ = al256(o_ + bytes); return at; };
  const size_t off_perm = take(BH * P.nqb * d), off_qt = take(BH * N * d * 2), off_D = take(BH * N_pad * 4);
  const size_t off_lse = take(BH * N_pad * 4);
  Scratch sc;
  uint8_t* ws;
  if (int s = bwd_workspace(p, o_, &dev, st, sc, &ws)) return s;
  const float* proj = nullptr;
  if (int s = get_projection(dev, p->seed, P.l, st, &proj)) return s;
  da::PrepArgs pa{};
  pa.q = q; pa.k = k; pa.in_f32 = 0;
  pa.BH = (int)BH; pa.BHkv = (int)BHkv; pa.N = P.N; pa.d = P.d; pa.block_l = P.l; pa.G = P.G; pa.HB = P.HB;
  pa.DR = P.DR; pa.nqb = P.nqb; pa.N_pad = P.N_pad; pa.proj = proj;
  pa.perm_ws = ws + off_perm;
  pa.n_hash_ctas = (int)(BH * P.nqb);
  DA_CUDA(da::launch_prep(pa, st));
  da::BwdArgs a{};
  a.q = static_cast<const uint16_t*>(q); a.o = static_cast<const uint16_t*>(o);
  a.dout = static_cast<const uint16_t*>(dout); a.perm = ws + off_perm;
  a.BH = (int)BH; a.N = P.N; a.d = P.d; a.G = P.G; a.nqb = P.nqb; a.block_l = P.l;
  a.qt = reinterpret_cast<uint16_t*>(ws + off_qt);
  a.D = reinterpret_cast<float*>(ws + off_D);
  a.Dstride = (int)N_pad;
  float* lse_pad = reinterpret_cast<float*>(ws + off_lse);
  DA_CUDA(da::launch_bwd_prologue(a, lse, lse_pad, (int)N_pad, st));
  CUtensorMap tmQt, tmdO, tmK, tmV;
  const uint32_t rb = d >= 64 ? 64 : (uint32_t)d;  // natural-row boxes: 64 columns (32 for d = 32)
  if (int s = make_map(&tmQt, a.qt, d, N, BH, rb, 128, (int)rb * 2)) return s;
  if (int s = make_map(&tmdO, dout, d, N, BH, rb, 128, (int)rb * 2)) return s;
  if (int s = make_map(&tmK, k, d, N, BHkv, rb, 128, (int)rb * 2)) return s;
  if (int s = make_map(&tmV, v, d, N, BHkv, rb, 128, (int)rb * 2)) return s;
  da::BwdFusedArgs f{};
  f.tmQt = &tmQt; f.tmdO = &tmdO; f.tmK = &tmK; f.tmV = &tmV;
  f.lse_pad = lse_pad; f.D_pad = a.D;
  f.dq = static_cast<uint16_t*>(dq);
  f.perm = a.perm; f.G = P.G; f.nqb = P.nqb; f.block_l = P.l;
  f.qt = a.qt; f.dout = a.dout;
  f.dk = static_cast<uint16_t*>(dk); f.dv = static_cast<uint16_t*>(dv);
  f.BH = (int)BH; f.BHkv = (int)BHkv; f.H = P.H; f.Hkv = P.Hkv; f.N = P.N; f.N_pad = (int)N_pad; f.d = P.d;
  f.causal = P.causal; f.scale = P.scale;
  record_ev(0, st);
  DA_CUDA(da::launch_bwd_fused(f, st));
  record_ev(1, st);
  record_ev(2, st);
  g_ev[0] = g_ev[1] = g_ev[2] = nullptr;
  g_last_launches = 5;  // hash, Q̃/D, lse pad, dK/dV, dQ̃ (+ fold in its epilogue)
  return DA_OK;
}

int backward(const void* q, const void* k, const void* v, const void* o, const void* dout, const float* lse,
             void* dq, void* dk, void* dv, const da_params* p, cudaStream_t st) {
  Plan P;
  if (int s = validate(p, true, &P)) return s;
  if (!q || !k || !v || !o || !dout || !lse || !dq || !dk || !dv) return fail(DA_ERR_INVALID, "null pointer");
  if (P.f32) return fail(DA_ERR_PRECONDITION, "backward: bf16 tensors only");
  return backward_fused(q, k, v, o, dout, lse, dq, dk, dv, p, P, st);
}

// ---------------------------------------------------------------------------- host entry point
// distr_attn_fwd_host: the job is cut into chunks of whole KV units (u = b*H_kv + h_kv with its
// H/H_kv query heads: contiguous in Q, K, V, O, lse and the exports), and chunk c runs
//   H2D(q, k, v of c) on s_in  ->  forward(c) on the caller's stream  ->  D2H(out, ... of c) on s_out
// through kSlots staging slots, so the copies of chunk c+1 / c-1 overlap the kernels of chunk c
// (the paper's copy/compute double buffering). Each chunk is one forward call over
// B = 1, H = units * H/H_kv, H_kv = units (flattened heads; bit-identical to the one-call result:
// every (b, h) problem is independent). One host call at a time (the call is synchronous).
constexpr int kSlots = 3;
struct HostPipe {
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev_in[kSlots], ev_comp[kSlots], ev_out[kSlots];
  void* stage = nullptr;
  size_t bytes = 0;
};
std::mutex g_host_mu;
std::map<int, HostPipe> g_host;

int forward_host(const void* q, const void* k, const void* v, void* out, const da_params* p, cudaStream_t st) {
  Plan P;
  if (int s = validate(p, true, &P)) return s;
  if (!q || !k || !v || !out) return fail(DA_ERR_INVALID, "null tensor pointer");
  int dev;
  if (int s = current_device(&dev)) return s;
  std::lock_guard<std::mutex> lk(g_host_mu);
  HostPipe& hp = g_host[dev];
  if (!hp.s_in) {
    DA_CUDA(cudaStreamCreateWithFlags(&hp.s_in, cudaStreamNonBlocking));
    DA_CUDA(cudaStreamCreateWithFlags(&hp.s_out, cudaStreamNonBlocking));
    for (int i = 0; i < kSlots; ++i) {
      DA_CUDA(cudaEventCreateWithFlags(&hp.ev_in[i], cudaEventDisableTiming));
      DA_CUDA(cudaEventCreateWithFlags(&hp.ev_comp[i], cudaEventDisableTiming));
      DA_CUDA(cudaEventCreateWithFlags(&hp.ev_out[i], cudaEventDisableTiming));
    }
  }
  const size_t es = P.f32 ? 4 : 2, g = (size_t)(P.H / P.Hkv), N = P.N, d = P.d;
  const size_t U = (size_t)P.B * P.Hkv;  // KV units
  // per-unit bytes of every buffer
  const size_t uq = g * N * d * es, ukv = N * d * es, ulse = p->lse ? g * N * 4 : 0;
  const size_t uexp = g * P.nqb * d, ub = p->bucket_ids ? uexp * 2 : 0, up = p->perm ? uexp : 0;
  // chunking: ~16 chunks for large jobs (copy/compute overlap), at least 8 MB of inputs per chunk
  const size_t total_in = U * (uq + 2 * ukv);
  size_t cu = (U + 15) / 16;
  const size_t min_units = (8u << 20) / (uq + 2 * ukv) + 1;
  if (cu < min_units) cu = min_units;
  if (const char* e = getenv("DA_HOST_CHUNK_UNITS")) cu = (size_t)atoll(e) > 0 ? (size_t)atoll(e) : cu;  // tests
  if (cu > U) cu = U;
  const size_t nchunks = (U + cu - 1) / cu;
  const int slots = nchunks < (size_t)kSlots ? (int)nchunks : kSlots;
  // slot layout: q, k, v, out, lse, buckets, perm of cu units
  const size_t o_q = 0, o_k = al256(o_q + cu * uq), o_v = al256(o_k + cu * ukv), o_o = al256(o_v + cu * ukv),
               o_l = al256(o_o + cu * uq), o_b = al256(o_l + cu * ulse), o_p = al256(o_b + cu * ub),
               slot_bytes = al256(o_p + cu * up);
  (void)total_in;
  if (hp.bytes < slot_bytes * slots) {
    if (hp.stage) {
      DA_CUDA(cudaDeviceSynchronize());
      DA_CUDA(cudaFree(hp.stage));
      hp.stage = nullptr;
      hp.bytes = 0;
    }
    DA_CUDA(cudaMalloc(&hp.stage, slot_bytes * slots));
    hp.bytes = slot_bytes * slots;
  }
  // Q-tile-pair shard: the 256-row pairs this call computes (kernel slot -> pair mapping)
  std::vector<std::pair<int, int>> rows;  // [r0, r1)
  const int npairs = (P.nqt + 1) / 2;
  if (P.pair_stride > 1) {
    for (int x = 0; x * P.pair_stride < npairs; ++x) {
      const int slot = x * P.pair_stride + ((x & 1) ? P.pair_stride - 1 - P.pair_off : P.pair_off);
      if (slot >= npairs) continue;
      const int pair = P.causal ? npairs - 1 - slot : slot;
      rows.emplace_back(pair * 256, std::min(P.N, pair * 256 + 256));
    }
  }
  const auto* qh = static_cast<const uint8_t*>(q);
  const auto* kh = static_cast<const uint8_t*>(k);
  const auto* vh = static_cast<const uint8_t*>(v);
  auto* oh = static_cast<uint8_t*>(out);
  auto* lh = reinterpret_cast<uint8_t*>(p->lse);
  auto* bh_ = reinterpret_cast<uint8_t*>(p->bucket_ids);
  auto* ph = reinterpret_cast<uint8_t*>(p->perm);
  uint8_t* S = static_cast<uint8_t*>(hp.stage);
  // D2H of [heads][rows_per_head][w] with only the shard's rows (or everything)
  auto d2h = [&](uint8_t* dst, const uint8_t* src, size_t heads, size_t per_head, size_t row_w, int row_div,
                 int nrows_total) -> cudaError_t {
    if (rows.empty() || row_div == 0)
      return cudaMemcpyAsync(dst, src, heads * per_head, cudaMemcpyDeviceToHost, hp.s_out);
    for (auto& rr : rows) {
      const int r0 = rr.first / row_div, r1 = std::min(nrows_total, (rr.second + row_div - 1) / row_div);
      cudaError_t e = cudaMemcpy2DAsync(dst + r0 * row_w, per_head, src + r0 * row_w, per_head, (r1 - r0) * row_w,
                                        heads, cudaMemcpyDeviceToHost, hp.s_out);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  };
  int launches = 0;
  for (size_t c = 0; c < nchunks; ++c) {
    const int sl = (int)(c % slots);
    const size_t u0 = c * cu, nu = std::min(cu, U - u0);
    uint8_t* base = S + sl * slot_bytes;
    if (c >= (size_t)slots) DA_CUDA(cudaStreamWaitEvent(hp.s_in, hp.ev_comp[sl], 0));  // inputs of c - slots consumed
    DA_CUDA(cudaMemcpyAsync(base + o_q, qh + u0 * uq, nu * uq, cudaMemcpyHostToDevice, hp.s_in));
    DA_CUDA(cudaMemcpyAsync(base + o_k, kh + u0 * ukv, nu * ukv, cudaMemcpyHostToDevice, hp.s_in));
    DA_CUDA(cudaMemcpyAsync(base + o_v, vh + u0 * ukv, nu * ukv, cudaMemcpyHostToDevice, hp.s_in));
    DA_CUDA(cudaEventRecord(hp.ev_in[sl], hp.s_in));
    DA_CUDA(cudaStreamWaitEvent(st, hp.ev_in[sl], 0));
    if (c >= (size_t)slots) DA_CUDA(cudaStreamWaitEvent(st, hp.ev_out[sl], 0));  // outputs of c - slots copied out
    da_params dp = *p;
    dp.B = 1;
    dp.H = (int)(nu * g);
    dp.H_kv = (int)nu;
    dp.workspace = nullptr;
    dp.workspace_bytes = 0;
    dp.lse = p->lse ? reinterpret_cast<float*>(base + o_l) : nullptr;
    dp.bucket_ids = p->bucket_ids ? reinterpret_cast<unsigned short*>(base + o_b) : nullptr;
    dp.perm = p->perm ? base + o_p : nullptr;
    if (int s = forward(base + o_q, base + o_k, base + o_v, base + o_o, &dp, st, true)) return s;
    launches += g_last_launches;
    DA_CUDA(cudaEventRecord(hp.ev_comp[sl], st));
    DA_CUDA(cudaStreamWaitEvent(hp.s_out, hp.ev_comp[sl], 0));
    const size_t heads = nu * g;
    DA_CUDA(d2h(oh + u0 * uq, base + o_o, heads, N * d * es, d * es, 1, P.N));
    if (p->lse) DA_CUDA(d2h(lh + u0 * ulse, base + o_l, heads, N * 4, 4, 1, P.N));
    if (p->bucket_ids) DA_CUDA(d2h(bh_ + u0 * ub, base + o_b, heads, P.nqb * d * 2, d * 2, P.l, P.nqb));
    if (p->perm) DA_CUDA(d2h(ph + u0 * up, base + o_p, heads, P.nqb * d, d, P.l, P.nqb));
    DA_CUDA(cudaEventRecord(hp.ev_out[sl], hp.s_out));
  }
  DA_CUDA(cudaStreamSynchronize(hp.s_out));
  DA_CUDA(cudaStreamSynchronize(st));
  DA_CUDA(cudaStreamSynchronize(hp.s_in));
  g_last_launches = launches;
  return DA_OK;
}

}  // namespace

extern "C" {

int distr_attn_init_params(da_params* p, int B, int H, int N, int d, int block_l, int group_size,
                           unsigned long long seed) {
  if (!p) return fail(DA_ERR_INVALID, "params is NULL");
  std::memset(p, 0, sizeof(*p));
  p->B = B; p->H = H; p->H_kv = H; p->N = N; p->d = d; p->block_l = block_l; p->group_size = group_size;
  p->seed = seed;
  p->causal = 0;
  p->scale = 0.f;
  p->dtype = DA_BF16;
  return DA_OK;
}

int distr_attn_fwd(const void* q, const void* k, const void* v, void* out, int B, int H, int N, int d,
                   int block_l, int group_size, unsigned long long seed) {
  da_params p;
  distr_attn_init_params(&p, B, H, N, d, block_l, group_size, seed);
  return forward(q, k, v, out, &p, nullptr, true);
}

int distr_attn_fwd_ex(const void* q, const void* k, const void* v, void* out, const da_params* p,
                      void* cuda_stream) {
  return forward(q, k, v, out, p, static_cast<cudaStream_t>(cuda_stream), true);
}

int exact_attn_fwd_ex(const void* q, const void* k, const void* v, void* out, const da_params* p,
                      void* cuda_stream) {
  return forward(q, k, v, out, p, static_cast<cudaStream_t>(cuda_stream), false);
}

int distr_attn_bwd_ex(const void* q, const void* k, const void* v, const void* out, const void* dout,
                      const float* lse, void* dq, void* dk, void* dv, const da_params* p, void* cuda_stream) {
  return backward(q, k, v, out, dout, lse, dq, dk, dv, p, static_cast<cudaStream_t>(cuda_stream));
}

int distr_attn_global_fwd_ex(const void* q, const void* k, const void* v, void* out, const da_params* p,
                             void* cuda_stream) {
  return forward_global(q, k, v, out, p, static_cast<cudaStream_t>(cuda_stream));
}

int distr_attn_fwd_host(const void* q, const void* k, const void* v, void* out, const da_params* p,
                        void* cuda_stream) {
  return forward_host(q, k, v, out, p, static_cast<cudaStream_t>(cuda_stream));
}

int distr_attn_hash(const void* q, const da_params* p, void* cuda_stream) {
  Plan P;
  if (int s = validate(p, true, &P)) return s;
  if (!q) return fail(DA_ERR_INVALID, "null q");
  if (!p->bucket_ids && !p->perm) return fail(DA_ERR_INVALID, "no export buffer (bucket_ids / perm)");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  int dev;
  if (int s = current_device(&dev)) return s;
  const float* proj;
  if (int s = get_projection(dev, p->seed, P.l, st, &proj)) return s;
  da::PrepArgs a{};
  a.q = q; a.k = nullptr; a.in_f32 = P.f32;
  a.BH = P.B * P.H; a.BHkv = P.B * P.Hkv; a.N = P.N; a.d = P.d; a.block_l = P.l; a.G = P.G; a.HB = P.HB;
  a.DR = P.DR; a.nqb = P.nqb; a.N_pad = P.N_pad; a.proj = proj;
  a.bucket_out = p->bucket_ids;
  a.perm_out = p->perm;
  a.n_hash_ctas = P.B * P.H * P.nqb;
  a.n_kt_ctas = 0;
  DA_CUDA(da::launch_prep(a, st));
  g_last_launches = 1;
  return DA_OK;
}

size_t distr_attn_bwd_workspace_size(const da_params* p) {
  static char dummy;
  g_bwd_size_only = true;
  g_bwd_query = 0;
  const int s = backward(&dummy, &dummy, &dummy, &dummy, &dummy, reinterpret_cast<const float*>(&dummy), &dummy,
                         &dummy, &dummy, p, nullptr);
  g_bwd_size_only = false;
  return s == kSizeOnly ? g_bwd_query : 0;
}

int distr_attn_projection(unsigned long long seed, int block_l, float* host_out) {
  if (!host_out) return fail(DA_ERR_INVALID, "host_out is NULL");
  if (block_l <= 0) return fail(DA_ERR_INVALID, "block_l=%d", block_l);
  make_projection(seed, block_l, host_out);
  return DA_OK;
}

size_t distr_attn_workspace_size(const da_params* p) {
  Plan P;
  if (validate(p, true, &P)) return 0;
  Plan E;
  validate(p, false, &E);
  size_t a, b;
  const size_t gl = P.f32 ? 0 : global_ws_bytes(P, &a, &b);
  size_t m = P.total > E.total ? P.total : E.total;
  return m > gl ? m : gl;
}

int distr_attn_plan(int N, int d, int block_l, int group_size, int distr, da_plan* out) {
  g_last_error.clear();
  if (!out) return fail(DA_ERR_INVALID, "out is NULL");
  da_params p;
  distr_attn_init_params(&p, 1, 1, N, d, block_l, distr ? group_size : 1, 0);
  Plan P;
  if (int s = validate(&p, distr != 0, &P)) return s;
  da::AttnConfig c;
  if (!da::attn_config(P.d, P.G, distr ? P.KHB : 1, distr ? 1 : 0, &c))
    return fail(DA_ERR_PRECONDITION, "no kernel for d=%d G*=%d block_l=%d", P.d, P.G, P.l);
  *out = da_plan{};
  out->tile_m = 128;
  out->tiles_per_cta = 2;
  out->tile_n = 128;
  out->s_width = c.dr;
  out->kv_stages = c.ns;
  out->khat_stages = c.nkh;
  out->threads = c.threads;
  out->smem_bytes = c.smem;
  out->tmem_cols = 512;  // 2 tiles x (O: d + S: m), rounded up to the allocation granule
  // Eq. 5 analogue: the largest m with tiles * (d + m) <= 512 TMEM columns
  int m_max = (512 / out->tiles_per_cta - P.d) / 16 * 16;
  out->m_max_tmem = m_max > 256 ? 256 : m_max;
  out->ctas = (P.N + 255) / 256;
  const double m = out->tile_n;
  out->mma_clk_per_tile = 2.0 * 128 * m * (c.dr + P.d) / 8192.0;
  out->exp_clk_per_tile = 128.0 * m / 16.0;
  // block_l = 256: one K̂ per key tile serves both Q tiles of the CTA
  out->fusion_smem_bytes_per_tile =
      distr ? ((double)P.d * m * 2 + (double)c.dr * m * 2) / (P.KHB == 0 ? 2.0 : 1.0) : 0.0;
  const double Nd = (double)P.N * P.d, l = P.l;
  out->hbm_bytes_paper = 2.0 * ((double)P.N / l) * (l * P.d + 2.0 * Nd + l * P.d);
  out->hbm_bytes_b200 = 2.0 * 4.0 * Nd + (distr ? 2.0 * 2.0 * Nd : 0.0);
  return DA_OK;
}

// Cost-model constants (clk on one SM at the 1800 MHz reference clock). d = 128: the CTA prologue
// (distr: Q landed + in-CTA hash + rank + Q̂ build + first S) and the steady clk per 128-key step
// of a CTA (two Q tiles), least-squares fits (tools/fit_planner.py) to the C4 N sweep of the
// ping-pong kernels (profiles/r02_v6/sweep*.json); d = 64 from the round-2 CTA timelines
// (tools/calibrate.sh, profiles/r02_v1/calib.txt).
struct StepCost {
  int d, l, G;
  double step, prologue;
};
constexpr StepCost kDistrCost[] = {
    {64, 64, 2, 3169, 13342},  {64, 128, 2, 3100, 11030}, {64, 128, 4, 3190, 11367},
    {64, 256, 2, 3045, 14314}, {64, 256, 4, 3112, 16459}, {128, 64, 2, 4625, 27688},
    {128, 128, 2, 3141, 14446}, {128, 128, 4, 3075, 18445}, {128, 256, 2, 3013, 15872},
    {128, 256, 4, 2847, 19427},
};
constexpr double kExactStep64 = 3268, kExactStep128 = 3349, kExactPrologue = 6000;

// Predicted kernel time (us) of one flavour: CTAs (Q tile pairs) list-scheduled over 148 SMs.
double predict_attn_us(int BH, int N, int causal, double step, double prologue, double mhz) {
  const int nqt = (N + 127) / 128, npairs = (nqt + 1) / 2, nkt = nqt;
  double total = 0, longest = 0;
  for (int p = 0; p < npairs; ++p) {
    const int steps = causal ? std::min(2 * p + 2, nkt) : nkt;
    const double t = prologue + steps * step;
    total += t;
    longest = std::max(longest, t);
  }
  total *= BH;
  const double sms = 148.0;
  const double clk = std::max(total / sms, longest) + std::ceil(BH * (double)npairs / sms) * 400.0;
  return clk / mhz;
}

const char* distr_attn_status_string(int status) {
  switch (status) {
    case DA_OK: return "ok";
    case DA_ERR_INVALID: return "invalid argument";
    case DA_ERR_PRECONDITION: return "unsupported configuration / precondition violated";
    case DA_ERR_CUDA: return "CUDA error";
    default: return "unknown status";
  }
}

int distr_attn_choose(int B, int H, int H_kv, int N, int d, int causal, int max_group_size, double clk_mhz,
                      da_choice* out) {
  g_last_error.clear();
  if (!out) return fail(DA_ERR_INVALID, "out is NULL");
  if (B <= 0 || H <= 0 || H_kv <= 0 || N <= 0 || H % H_kv) return fail(DA_ERR_INVALID, "bad shape");
  if (d != 32 && d != 64 && d != 128) return fail(DA_ERR_PRECONDITION, "d=%d unsupported", d);
  const double mhz = clk_mhz > 0 ? clk_mhz : 1800.0;
  const int BH = B * H;
  const double launch_us = 4.0;
  const double dc = d == 128 ? 128 : 64;  // d = 32 runs the d = 64 schedule (fewer K-steps, same softmax)
  *out = da_choice{};
  out->predicted_exact_us =
      launch_us + predict_attn_us(BH, N, causal, dc == 128 ? kExactStep128 : kExactStep64, kExactPrologue, mhz);
  // K^T layout pass: read K + write K^T (HBM, ~5.1 TB/s measured) + its launch
  const double kt_us = launch_us + 2.0 * 2.0 * B * H_kv * (double)N * d / 5.1e6;
  out->predicted_distr_us = 1e300;
  for (const StepCost& c : kDistrCost) {
    if (c.d != (int)dc || c.G > max_group_size) continue;
    if (d / c.G < 16) continue;
    const double t = launch_us + kt_us + predict_attn_us(BH, N, causal, c.step, c.prologue, mhz);
    if (t < out->predicted_distr_us) {
      out->predicted_distr_us = t;
      out->block_l = c.l;
      out->group_size = c.G;
    }
  }
  // the approximation is taken only when it is predicted clearly faster than exact attention
  // (more accurate by definition): by more than the model's spread against the sweeps, 2 %
  out->distr = out->predicted_distr_us < 0.98 * out->predicted_exact_us;
  out->predicted_us = out->distr ? out->predicted_distr_us : out->predicted_exact_us;
  if (!out->distr) {
    out->block_l = 0;
    out->group_size = 1;
  }
  return DA_OK;
}

const char* distr_attn_last_error(void) { return g_last_error.c_str(); }

int distr_attn_last_launch_count(void) { return g_last_launches; }

int distr_attn_set_trace(void* device_buf) {
  g_trace = static_cast<long long*>(device_buf);
  return DA_OK;
}

int distr_attn_set_profile_events(void* ev_start, void* ev_attn, void* ev_end) {
  g_ev[0] = static_cast<cudaEvent_t>(ev_start);
  g_ev[1] = static_cast<cudaEvent_t>(ev_attn);
  g_ev[2] = static_cast<cudaEvent_t>(ev_end);
  return DA_OK;
}

}  // extern "C"
