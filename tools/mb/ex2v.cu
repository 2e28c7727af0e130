// Microbenchmark: MUFU exp2 element throughput per SM for ex2.approx.ftz.f32, ex2.approx.f16x2
// and ex2.approx.ftz.bf16x2 (two exps per lane per instruction), at 4/8/16 warps per SM (148
// CTAs). 16 independent chains per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  uint32_t x[16];
  for (int j = 0; j < 16; ++j) {
    const float f = -0.001f * (threadIdx.x + j);
    x[j] = MODE == 0 ? __float_as_uint(f) : 0xBC00BC00u ^ (threadIdx.x + j);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      uint32_t y;
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=r"(y) : "r"(x[j]));
      if (MODE == 1) asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x[j]));
      if (MODE == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x[j]));
      x[j] = y ^ 0x80008000u;  // keep the argument negative (one ALU op per exp instruction)
    }
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t acc = 0;
  for (int j = 0; j < 16; ++j) acc ^= x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"ex2.ftz.f32", "ex2.f16x2", "ex2.ftz.bf16x2"};
  for (int warps : {4, 8, 16}) for (int mode = 0; mode < 3; ++mode) {
    int iters = 2000;
    auto launch = [&]() {
      if (mode == 0) k<0><<<148, warps * 32>>>(out, cyc, iters);
      if (mode == 1) k<1><<<148, warps * 32>>>(out, cyc, iters);
      if (mode == 2) k<2><<<148, warps * 32>>>(out, cyc, iters);
    };
    launch(); cudaDeviceSynchronize(); launch(); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double inst = (double)iters * 16 * warps * 32;
    const double elems = inst * (mode == 0 ? 1 : 2);
    printf("warps=%2d %-16s lane-instr/clk/SM = %6.2f  exps/clk/SM = %6.2f\n", warps, names[mode], inst / c, elems / c);
  }
  return 0;
}
