// Microbenchmark: tcgen05.ld / tcgen05.st cost as seen by softmax-like warps. One CTA per SM,
// W warps (warp w owns TMEM lanes 32*(w%4)); each iteration loads 64 fp32 columns per thread
// (2 x 32x32b.x32) and waits, optionally stores 32 columns back; clock64 cycles per iteration.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2507_17245_b200/csrc/ptx.cuh"
using namespace da;

template <int MODE>  // 0: ld x32 x2 + wait; 1: ld + wait + st x32 + wait; 2: ld x16 x4 + wait
__global__ void k(float* out, long long* cyc, int iters) {
  __shared__ uint32_t tptr;
  const int warp = threadIdx.x / 32;
  if (warp == 0) { tmem_alloc(&tptr, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tptr + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 64);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t a[32], b[32];
    if (MODE == 2) {
      tmem_ld16(tmem, *reinterpret_cast<uint32_t(*)[16]>(&a[0]));
      tmem_ld16(tmem + 16, *reinterpret_cast<uint32_t(*)[16]>(&a[16]));
      tmem_ld16(tmem + 32, *reinterpret_cast<uint32_t(*)[16]>(&b[0]));
      tmem_ld16(tmem + 48, *reinterpret_cast<uint32_t(*)[16]>(&b[16]));
    } else {
      tmem_ld32(tmem, a);
      tmem_ld32(tmem + 32, b);
    }
    tmem_ld_wait();
#pragma unroll
    for (int e = 0; e < 32; ++e) acc += a[e] ^ b[e];
    if (MODE == 1) {
      tmem_st32(tmem, a);
      tmem_st_wait();
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tptr, 512); }
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  for (int warps : {4, 8}) {
    for (int mode = 0; mode < 3; ++mode) {
      const int iters = 1000;
      auto launch = [&]() {
        if (mode == 0) k<0><<<148, warps * 32>>>(out, cyc, iters);
        if (mode == 1) k<1><<<148, warps * 32>>>(out, cyc, iters);
        if (mode == 2) k<2><<<148, warps * 32>>>(out, cyc, iters);
      };
      launch(); cudaDeviceSynchronize(); launch();
      cudaError_t e = cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("warps=%d mode=%d (%s) cycles/iter=%.1f  TMEM read B/clk/SM=%.0f  %s\n", warps, mode,
             mode == 0 ? "ld 2x32 + wait" : mode == 1 ? "ld 2x32 + wait + st x32 + wait" : "ld 4x16 + wait",
             (double)c / iters, warps * 32 * 64 * 4.0 / ((double)c / iters), cudaGetErrorString(e));
    }
  }
  return 0;
}
