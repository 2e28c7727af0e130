// Which pipe does the P pack (fp32 pair -> bf16x2) use, and what does it cost next to MUFU.EX2?
// Per-SM throughput (results per clk per SM) of: EX2 alone, F2FP alone, EX2 + F2FP at the
// softmax's 2:1 ratio, the integer round-and-permute pack (IADD3 + PRMT) alone and with EX2,
// and EX2.F16x2. 148 CTAs x W warps, 16 independent chains per thread, clock64 per CTA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb/pack tools/mb/pack.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float x[16];
  uint32_t u[16];
  for (int j = 0; j < 16; ++j) {
    x[j] = -0.001f * (threadIdx.x + j);
    u[j] = threadIdx.x * 77u + j;
  }
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      float a = x[j], b = x[j + 1];
      uint32_t p = 0;
      if (MODE == 0 || MODE == 2 || MODE == 4) {  // two EX2
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(x[j]));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(x[j + 1]));
      }
      if (MODE == 1 || MODE == 2) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(b), "f"(a));
      if (MODE == 3 || MODE == 4) {  // round half up on the bit pattern, then keep the high halves
        const uint32_t ra = __float_as_uint(a) + 0x8000u, rb = __float_as_uint(b) + 0x8000u;
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(p) : "r"(ra), "r"(rb));
      }
      if (MODE == 5) {  // EX2 on an f16x2 pair (one instruction for two results)
        uint32_t h;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(h) : "r"(u[j]));
        u[j] = h ^ 0x1u;
        p = h;
      }
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
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"EX2 x2", "F2FP", "EX2 x2 + F2FP", "IADD x2 + PRMT", "EX2 x2 + IADD/PRMT", "EX2.F16x2"};
  for (int warps : {8, 16})
    for (int mode = 0; mode < 6; ++mode) {
      const int iters = 2000;
      auto launch = [&]() {
        switch (mode) {
          case 0: k<0><<<148, warps * 32>>>(out, cyc, iters); break;
          case 1: k<1><<<148, warps * 32>>>(out, cyc, iters); break;
          case 2: k<2><<<148, warps * 32>>>(out, cyc, iters); break;
          case 3: k<3><<<148, warps * 32>>>(out, cyc, iters); break;
          case 4: k<4><<<148, warps * 32>>>(out, cyc, iters); break;
          default: k<5><<<148, warps * 32>>>(out, cyc, iters); break;
        }
      };
      launch();
      cudaDeviceSynchronize();
      launch();
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double pairs = (double)iters * 8 * warps * 32;
      printf("warps=%2d %-20s pairs/clk/SM = %6.2f  (elements %6.2f)\n", warps, names[mode], pairs / c, 2 * pairs / c);
    }
  return 0;
}
