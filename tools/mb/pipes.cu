// Microbenchmark: per-SM throughput of MUFU.EX2, FFMA2, FADD2 and the FMA-pipe exp2 polynomial.
// One CTA per SM, W warps; each thread runs 8 independent chains; cycles via clock64.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2507_17245_b200/csrc/ptx.cuh"
using namespace da;
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float2 x[8];
  for (int j = 0; j < 8; ++j) x[j] = make_float2(-0.001f * (threadIdx.x + j), -0.002f * j);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) { x[j].x = ex2(x[j].x) - 1.5f; x[j].y = ex2(x[j].y) - 1.5f; }       // 2 MUFU + 2 FADD
      if (MODE == 1) { x[j] = fma2(x[j], make_float2(0.999f, 0.999f), make_float2(-0.01f, -0.01f)); }  // 1 FFMA2
      if (MODE == 2) { float2 p = exp2_poly2(x[j]); x[j] = fadd2(p, make_float2(-1.5f, -1.5f)); }  // poly pair
      if (MODE == 3) { x[j].x = fmaf(x[j].x, 0.999f, -0.01f); x[j].y = fmaf(x[j].y, 0.999f, -0.01f); } // 2 FFMA
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int j = 0; j < 8; ++j) s += x[j].x + x[j].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"MUFU.EX2 pair(+FADD)", "FFMA2", "poly exp2 pair", "2x FFMA"};
  for (int warps : {4, 8, 16}) {
    for (int mode = 0; mode < 4; ++mode) {
      int iters = 2000;
      auto launch = [&]() {
        if (mode == 0) k<0><<<148, warps * 32>>>(out, cyc, iters);
        if (mode == 1) k<1><<<148, warps * 32>>>(out, cyc, iters);
        if (mode == 2) k<2><<<148, warps * 32>>>(out, cyc, iters);
        if (mode == 3) k<3><<<148, warps * 32>>>(out, cyc, iters);
      };
      launch(); cudaDeviceSynchronize(); launch(); cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double pairs = (double)iters * 8 * warps * 32;   // pairs processed per SM
      printf("warps=%2d %-22s cycles=%lld  pairs/clk/SM=%.2f  elem/clk/SM=%.2f\n", warps, names[mode], c, pairs / c, 2 * pairs / c);
    }
  }
  return 0;
}
