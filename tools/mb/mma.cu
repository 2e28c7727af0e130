// Microbenchmark: tcgen05.mma latency and throughput for the attention kernel's shapes, one CTA
// per SM (148 CTAs, all SMs busy like the real kernel). Shapes per 128x128 tile:
//   S  = A·Bᵀ  M=128 N=128 K=KS (SS: A K-major SW128, B K-major SW128), KS = 64 (distr) or 128
//   PV = P·V   M=128 N=128 K=128 (TS: A = P from TMEM, B = V MN-major SW128)
// Modes: latency of one S, one PV, PV then S (the chain S_t(i+1) waits on); throughput of 64
// back-to-back (PV + S) groups. Operand contents are zero (timing only).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2507_17245_b200/csrc/ptx.cuh"
using namespace da;

template <int KS>
__global__ void k(long long* cyc, int mode, int reps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;              // 128 x KS bf16, K-major SW128 (KS/64 boxes of 16 KB)
  uint8_t* sB = smem + 32768;      // 128 x KS bf16
  uint8_t* sV = smem + 65536;      // 128 keys x 128 d bf16, MN-major SW128 (2 boxes of 16 KB)
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 98304 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc(&tptr, 512); tmem_relinquish(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tptr;
  if (threadIdx.x == 0) {
    constexpr uint32_t IS = make_idesc_bf16(128, 128, false, false);
    constexpr uint32_t IPV = make_idesc_bf16(128, 128, false, true);
    auto issue_s = [&]() {
#pragma unroll
      for (int kk = 0; kk < KS / 16; ++kk) {
        const uint64_t a = make_sdesc(smem_u32(sA) + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024, 2);
        const uint64_t b = make_sdesc(smem_u32(sB) + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024, 2);
        mma_ss(tmem + 256, a, b, IS, kk > 0);
      }
    };
    auto issue_pv = [&]() {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t v = make_sdesc(smem_u32(sV) + kk * 2048, 128 * 128, 1024, 2);
        mma_ts(tmem, tmem + 384 + kk * 8, v, IPV, 1);
      }
    };
    uint32_t ph = 0;
    long long best = 1LL << 60, tot = 0;
    for (int r = 0; r < reps; ++r) {
      long long t0 = clock64();
      if (mode == 0) issue_s();
      if (mode == 1) issue_pv();
      if (mode == 2) { issue_pv(); issue_s(); }
      if (mode == 3) for (int j = 0; j < 64; ++j) { issue_pv(); issue_s(); }
      if (mode == 4) for (int j = 0; j < 64; ++j) issue_pv();
      if (mode == 5) for (int j = 0; j < 64; ++j) issue_s();
      mma_commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
      long long t1 = clock64();
      tot += t1 - t0;
      best = min(best, t1 - t0);
    }
    cyc[blockIdx.x * 2] = best;
    cyc[blockIdx.x * 2 + 1] = tot / reps;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  long long* cyc; cudaMalloc(&cyc, 148 * 16);
  const char* names[] = {"S", "PV", "PV then S", "64 x (PV+S)", "64 x PV", "64 x S"};
  for (int ks : {64, 128}) {
    for (int mode = 0; mode < 6; ++mode) {
      auto kern = ks == 64 ? k<64> : k<128>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
      kern<<<148, 128, 100 * 1024>>>(cyc, mode, 20);
      cudaError_t e = cudaDeviceSynchronize();
      long long c[2]; cudaMemcpy(c, cyc, 16, cudaMemcpyDeviceToHost);
      const double flop = 2.0 * 128 * 128 * (mode == 0 ? ks : mode == 1 ? 128 : mode == 2 ? ks + 128 :
                                              mode == 3 ? 64.0 * (ks + 128) : mode == 4 ? 64.0 * 128 : 64.0 * ks);
      printf("KS=%3d %-12s best %7lld clk  avg %7lld clk  -> %.0f FLOP/clk/SM (peak 8192)  %s\n", ks, names[mode], c[0],
             c[1], flop / c[0], cudaGetErrorString(e));
    }
  }
  return 0;
}
