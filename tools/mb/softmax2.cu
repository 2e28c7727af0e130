// Microbenchmark: the exp phase of one 128-key row per thread with ONE warp per SM sub-partition
// (4 warps per SM; the FA4-style layout) vs two (8 warps), for several instruction schedules of
// the same work (per pair: FFMA2 affine, exp2 on MUFU or the FMA-pipe polynomial, FADD2 row sum,
// F2FP pack). Cycles per 128x128 tile (= per 4 warps' worth of rows).
//   V0 straight loop (as attn.cu), EMU of every 8 pairs on the polynomial
//   V1 batches of 8 pairs: 8 FFMA2, then the exps, then packs/sums
//   V2 MUFU pairs first, polynomial pairs afterwards (two passes over the row)
//   V3 polynomial pairs first, MUFU pairs afterwards
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2507_17245_b200/csrc/ptx.cuh"
using namespace da;
template <int EMU, int V>
__global__ void k(float* out, long long* cyc, int iters, float sl2) {
  float s[128];
#pragma unroll
  for (int e = 0; e < 128; ++e) s[e] = out[e * 1024 + threadIdx.x];
  float l = 0.f;
  uint32_t sink = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float m = l * 1e-30f + 3.0f;
    const float2 sl2x2 = make_float2(sl2, sl2), nm2 = make_float2(-m, -m);
    float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    uint32_t pr[64];
    if (V == 0) {
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        const float2 x = fma2(make_float2(s[2 * e], s[2 * e + 1]), sl2x2, nm2);
        float2 p;
        if ((e & 7) >= 8 - EMU) p = exp2_poly2(x); else p = make_float2(ex2(x.x), ex2(x.y));
        acc[e & 3] = fadd2(acc[e & 3], p);
        pr[e] = pack_bf16x2(p.x, p.y);
      }
    } else if (V == 1) {
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        float2 x[8], p[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma2(make_float2(s[16 * b + 2 * j], s[16 * b + 2 * j + 1]), sl2x2, nm2);
#pragma unroll
        for (int j = 0; j < 8; ++j) p[j] = j >= 8 - EMU ? exp2_poly2(x[j]) : make_float2(ex2(x[j].x), ex2(x[j].y));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc[j & 3] = fadd2(acc[j & 3], p[j]);
          pr[8 * b + j] = pack_bf16x2(p[j].x, p[j].y);
        }
      }
    } else {
      // two passes: pass A handles pairs with (e & 7) < 8 - EMU (MUFU), pass B the rest (poly)
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        const bool mufu_pass = (pass == 0) == (V == 2);
#pragma unroll
        for (int e = 0; e < 64; ++e) {
          const bool is_poly = (e & 7) >= 8 - EMU;
          if (is_poly == mufu_pass) continue;
          const float2 x = fma2(make_float2(s[2 * e], s[2 * e + 1]), sl2x2, nm2);
          const float2 p = is_poly ? exp2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
          acc[e & 3] = fadd2(acc[e & 3], p);
          pr[e] = pack_bf16x2(p.x, p.y);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 64; ++e) sink ^= pr[e];
    const float2 a = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
    l += a.x + a.y;
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = l + (float)sink;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int EMU, int V>
void run(float* out, long long* cyc, int warps) {
  const int iters = 200;
  k<EMU, V><<<148, warps * 32>>>(out, cyc, iters, 0.18f);
  cudaDeviceSynchronize();
  k<EMU, V><<<148, warps * 32>>>(out, cyc, iters, 0.18f);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("warps=%d V%d EMU=%d: clk per 128x128 tile %.0f  (%.1f exp/clk/SM)\n", warps, V, EMU, (double)c / iters * 4 / warps,
         128.0 * 128 / ((double)c / iters * 4 / warps));
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 128 * 4); cudaMemset(out, 0, 148 * 1024 * 128 * 4); cudaMalloc(&cyc, 148 * 8);
  for (int warps : {4, 8}) {
    run<0, 0>(out, cyc, warps); run<2, 0>(out, cyc, warps); run<3, 0>(out, cyc, warps);
    run<2, 1>(out, cyc, warps); run<3, 1>(out, cyc, warps);
    run<2, 2>(out, cyc, warps); run<3, 2>(out, cyc, warps);
    run<2, 3>(out, cyc, warps); run<3, 3>(out, cyc, warps);
  }
  return 0;
}
