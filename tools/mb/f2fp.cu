// Does F2FP (cvt.rn.bf16x2.f32) share the MUFU (XU) pipe? Per-SM throughput of: EX2 only,
// EX2 + one F2FP per pair, EX2 + PRMT-based truncating pack per pair.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float x[16];
  for (int j = 0; j < 16; ++j) x[j] = -0.001f * (threadIdx.x + j);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      float a, b;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(x[j]));
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(x[j + 1]));
      uint32_t p;
      if (MODE == 1) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(b), "f"(a));
      if (MODE == 2) asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(p) : "r"(__float_as_uint(a)), "r"(__float_as_uint(b)));
      if (MODE == 0) p = __float_as_uint(a) ^ __float_as_uint(b);
      acc ^= p;
      x[j] = a - 1.5f;
      x[j + 1] = b - 1.5f;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc + x[0];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"EX2 x2 + LOP", "EX2 x2 + F2FP", "EX2 x2 + PRMT"};
  for (int warps : {8, 16}) for (int mode = 0; mode < 3; ++mode) {
    int iters = 2000;
    auto launch = [&]() {
      if (mode == 0) k<0><<<148, warps * 32>>>(out, cyc, iters);
      if (mode == 1) k<1><<<148, warps * 32>>>(out, cyc, iters);
      if (mode == 2) k<2><<<148, warps * 32>>>(out, cyc, iters);
    };
    launch(); cudaDeviceSynchronize(); launch(); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double ex = (double)iters * 16 * warps * 32;
    printf("warps=%d %-16s ex2/clk/SM = %.2f\n", warps, names[mode], ex / c);
  }
  return 0;
}
