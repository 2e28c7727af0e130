// Microbenchmark: how the single-thread tcgen05.mma issue behaves for the half-split pipeline's
// "serve" = PV (4 x M128 N128 K16, TS) + S half (4 x M128 N64 K16, SS) + commits. One CTA per
// SM (148 CTAs). Reports, per mode, the issue time (clock after the last issue) and the
// completion time (mbarrier observed), best over reps, for 1 serve and for 32 back-to-back
// serves (throughput), with and without commits between serves, and the N=128 S variant.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2507_17245_b200/csrc/ptx.cuh"
using namespace da;

__global__ void k(long long* cyc, int mode, int nserve, int reps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;          // 128 x 64 bf16 K-major SW128 (16 KB)
  uint8_t* sB = smem + 16384;  // 128 x 64 bf16 (MN-major K̂ for N=64/128 or K-major)
  uint8_t* sV = smem + 32768;  // 128 keys x 128 d bf16, MN-major SW128 (2 boxes of 16 KB)
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tptr;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc(&tptr, 512); tmem_relinquish(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tptr;
  if (warp == 1) {
    constexpr uint32_t IS64 = make_idesc_bf16(128, 64, false, true);
    constexpr uint32_t IS128 = make_idesc_bf16(128, 128, false, true);
    constexpr uint32_t IPV = make_idesc_bf16(128, 128, false, true);
    uint64_t ad[4], bd[4], vd[4];
    for (int kk = 0; kk < 4; ++kk) {
      ad[kk] = make_sdesc(smem_u32(sA) + kk * 32, 16, 1024, kSw128);
      bd[kk] = make_sdesc(smem_u32(sB) + kk * 2048, 64 * 128, 1024, kSw128);
      vd[kk] = make_sdesc(smem_u32(sV) + kk * 16 * 128, 128 * 128, 1024, kSw128);
    }
    uint32_t ph = 0;
    long long bi = 1LL << 60, bc = 1LL << 60;
    for (int r = 0; r < reps; ++r) {
      __syncwarp();
      long long t0 = clock64(), t1 = 0;
      if (elect_one()) {
        for (int j = 0; j < nserve; ++j) {
          const int t = j & 1;
          if (mode != 2) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) mma_ts(tmem + t * 128, tmem + 256 + 128 * t + kk * 8, vd[kk], IPV, 1);
            if (mode == 0 || mode == 3) mma_commit(&bar[1 + t]);
          }
          if (mode == 3) {  // N=128 S, 4 K-steps
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) mma_ss(tmem + 256 + 128 * t, ad[kk], bd[kk], IS128, kk > 0);
          } else {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) mma_ss(tmem + 256 + 128 * t + 64, ad[kk], bd[kk], IS64, kk > 0);
          }
          if (mode == 0 || mode == 3) mma_commit(&bar[3]);
        }
        t1 = clock64();
        mma_commit(&bar[0]);
      }
      mbar_wait(&bar[0], ph);
      ph ^= 1;
      long long t2 = clock64();
      t1 = __shfl_sync(0xffffffffu, t1, 0);
      if (lane_id() == 0) { bi = min(bi, t1 - t0); bc = min(bc, t2 - t0); }
    }
    if (lane_id() == 0) { cyc[blockIdx.x * 2] = bi; cyc[blockIdx.x * 2 + 1] = bc; }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  long long* cyc; cudaMalloc(&cyc, 148 * 16);
  const char* names[] = {"PV4+S4(N64)+commits", "PV4+S4(N64) no commits", "S4(N64) only", "PV4+S4(N128)+commits"};
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int mode = 0; mode < 4; ++mode)
    for (int ns : {1, 2, 32}) {
      k<<<148, 64, 80 * 1024>>>(cyc, mode, ns, 20);
      cudaError_t e = cudaDeviceSynchronize();
      long long c[2]; cudaMemcpy(c, cyc, 16, cudaMemcpyDeviceToHost);
      const double fl = ns * 2.0 * 128 * ((mode == 2 ? 0 : 128 * 64) + (mode == 3 ? 128 : 64) * 64);
      printf("%-26s serves=%2d  issue-return %6lld clk  complete %6lld clk  -> %.0f FLOP/clk/SM (%.0f clk/serve) %s\n",
             names[mode], ns, c[0], c[1], fl / c[1], (double)c[1] / ns, cudaGetErrorString(e));
    }
  return 0;
}
