// Microbenchmark: the softmax exp phase of one 128-key row per thread (like attn.cu), with EMU/8
// pairs on the FMA-pipe polynomial. One CTA per SM with W warps; cycles per tile via clock64.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2507_17245_b200/csrc/ptx.cuh"
using namespace da;
template <int EMU>
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
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t pr[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const int col = 64 * c + 2 * e;
        const float2 x = fma2(make_float2(s[col], s[col + 1]), sl2x2, nm2);
        float2 p;
        if ((e & 7) >= 8 - EMU) p = exp2_poly2(x); else p = make_float2(ex2(x.x), ex2(x.y));
        acc[e & 3] = fadd2(acc[e & 3], p);
        pr[e] = pack_bf16x2(p.x, p.y);
      }
#pragma unroll
      for (int e = 0; e < 32; ++e) sink ^= pr[e];
    }
    const float2 a = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
    l += a.x + a.y;
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = l + (float)sink;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 128 * 4); cudaMemset(out, 0, 148 * 1024 * 128 * 4); cudaMalloc(&cyc, 148 * 8);
  for (int warps : {4, 8}) {
    for (int emu : {0, 2, 3, 4}) {
      int iters = 200;
      auto launch = [&]() {
        if (emu == 0) k<0><<<148, warps * 32>>>(out, cyc, iters, 0.18f);
        if (emu == 2) k<2><<<148, warps * 32>>>(out, cyc, iters, 0.18f);
        if (emu == 3) k<3><<<148, warps * 32>>>(out, cyc, iters, 0.18f);
        if (emu == 4) k<4><<<148, warps * 32>>>(out, cyc, iters, 0.18f);
      };
      launch(); cudaDeviceSynchronize(); launch(); cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("warps=%d EMU=%d cycles/iter=%.0f  (per 128 rows x 128 keys: %.0f)\n", warps, emu, (double)c / iters, (double)c / iters * 4 / warps);
    }
  }
  return 0;
}
