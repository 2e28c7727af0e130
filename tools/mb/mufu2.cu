// MUFU throughput: ex2.approx.ftz.f32 vs ex2.approx.ftz.bf16x2 vs ex2.approx.f16x2 (elements/clk/SM)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  uint32_t x[8];
  for (int j = 0; j < 8; ++j) x[j] = 0xBF80BF00u + threadIdx.x + j;  // small negative bf16/f16 pairs
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) {
        float a = __uint_as_float(x[j] | 0xBF000000u), b;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(a));
        float c;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(b));
        x[j] = __float_as_uint(c) ^ 0x80000000u;
      } else if (MODE == 1) {
        uint32_t y;
        asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x[j]));
        x[j] = y ^ 0x80008000u;
      } else {
        uint32_t y;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x[j]));
        x[j] = y ^ 0x80008000u;
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t s = 0; for (int j = 0; j < 8; ++j) s ^= x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"ex2.f32 (2 per elem pair)", "ex2.bf16x2", "ex2.f16x2"};
  for (int mode = 0; mode < 3; ++mode) {
    int iters = 2000, warps = 16;
    auto launch = [&]() {
      if (mode == 0) k<0><<<148, warps * 32>>>(out, cyc, iters);
      if (mode == 1) k<1><<<148, warps * 32>>>(out, cyc, iters);
      if (mode == 2) k<2><<<148, warps * 32>>>(out, cyc, iters);
    };
    launch(); cudaDeviceSynchronize(); launch(); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double elems = (double)iters * 8 * warps * 32 * 2;
    printf("%-28s elems/clk/SM = %.2f\n", names[mode], elems / c);
  }
  return 0;
}
