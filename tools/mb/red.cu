// Microbenchmark: fp32 reduction-into-global throughput on B200 for the single-pass backward's dQ
// accumulation. 148 CTAs (one per SM, 256 threads); CTA c adds a [128 rows x W] fp32 tile into
// tile (c + it) mod NT of a [NT*128 x W] buffer per iteration (staggered: CTAs of one head never
// hit the same tile at once). Modes: 0 = red.global.add.v4.f32 from registers, 1 = red.global.add.f32
// scalar, 2 = cp.reduce.async.bulk (1-D bulk add from shared memory, one 32 KB/64 KB request).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE, int W>
__global__ void __launch_bounds__(256) k(float* buf, int NT, int iters, long long* cyc) {
  extern __shared__ __align__(128) float sm[];
  for (int i = threadIdx.x; i < 128 * W; i += 256) sm[i] = 1.0f;
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int tile = (blockIdx.x + it * 7) % NT;
    float* dst = buf + (size_t)tile * 128 * W;
    if (MODE == 0) {
      for (int i = threadIdx.x; i < 128 * W / 4; i += 256) {
        float* p = dst + 4 * i;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
      }
    } else if (MODE == 3) {
      // row per lane (the 32x32b TMEM layout): warp w, lane = row (w%4)*32+lane, 16 B per lane
      // per instruction, W/4 instructions per thread for its row's W/2 columns (2 warps per row)
      const int w = threadIdx.x / 32, row = (w % 4) * 32 + (threadIdx.x & 31), half = w / 4;
      float* p = dst + (size_t)row * W + half * (W / 2);
#pragma unroll 4
      for (int i = 0; i < W / 8; ++i)
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p + 4 * i), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
    } else if (MODE == 4) {
      // 16x256b-like: 4 lanes cover 8 consecutive columns (32 B) of one row, 8 rows per instruction
      const int w = threadIdx.x / 32, l = threadIdx.x & 31;
      for (int rb = w; rb < 16; rb += 8)
        for (int cg = 0; cg < W / 8; ++cg)
          for (int hh = 0; hh < 2; ++hh) {
            float* p = dst + (size_t)(rb * 8 + (l >> 2)) * W + cg * 8 + (l & 3) * 2;
            (void)hh;
            asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(1.f), "f"(1.f) : "memory");
          }
    } else if (MODE == 1) {
      for (int i = threadIdx.x; i < 128 * W; i += 256) atomicAdd(dst + i, 1.0f);
    } else {
      if (threadIdx.x == 0) {
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
                     "r"((uint32_t)__cvta_generic_to_shared(sm)), "r"(128 * W * 4) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      }
    }
  }
  if (MODE == 2 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE, int W>
void run(const char* name, float* buf, long long* cyc, int NT) {
  const int iters = 200;
  cudaFuncSetAttribute(k<MODE, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * W * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE, W><<<148, 256, 128 * W * 4>>>(buf, NT, 5, cyc);
  cudaEventRecord(e0);
  k<MODE, W><<<148, 256, 128 * W * 4>>>(buf, NT, iters, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = 148.0 * iters * 128 * W * 4;
  printf("%-22s W=%3d NT=%4d: %.3f ms, %.2f TB/s of fp32 reductions (%s)\n", name, W, NT, ms, bytes / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  float* buf; long long* cyc;
  const size_t n = (size_t)2048 * 128 * 128;
  cudaMalloc(&buf, n * 4); cudaMemset(buf, 0, n * 4); cudaMalloc(&cyc, 148 * 8);
  for (int NT : {128, 2048}) {
    run<0, 64>("red.v4 regs", buf, cyc, NT);
    run<0, 128>("red.v4 regs", buf, cyc, NT);
    run<1, 64>("atomicAdd scalar", buf, cyc, NT);
    run<3, 64>("red.v4 row/lane", buf, cyc, NT);
    run<3, 128>("red.v4 row/lane", buf, cyc, NT);
    run<4, 128>("red.v2 4 lanes/sector", buf, cyc, NT);
    run<2, 64>("bulk reduce smem", buf, cyc, NT);
    run<2, 128>("bulk reduce smem", buf, cyc, NT);
  }
  return 0;
}
