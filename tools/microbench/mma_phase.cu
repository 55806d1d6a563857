// Latency of one "MMA phase" of the BSFA kernel on one SM, nothing else running:
// 8 PV MMAs (TS, 128x128x16) + 8 QK MMAs (SS, 128x128x16) + commit -> mbarrier,
// observed by a second warp.  Also the commit->wake latency and single-MMA latency.
#include "../../paper_2512_07011_b200/csrc/ptx.cuh"
#include <cstdio>
using namespace bsfa;

__global__ void __launch_bounds__(128, 1) k(long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = base;             // 32 KB
  uint8_t* sK = base + 32768;     // 32 KB
  uint8_t* sV = base + 65536;     // 32 KB
  const uint32_t bar = smem_u32(base + 98304);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(base + 98304 + 64);
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbarrier_init(); }
  if (warp == 0) { tmem_alloc(tptr, 512); tmem_relinquish(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tptr;
  constexpr uint32_t IQK = make_idesc_bf16(128, 128, 0, 0);
  constexpr uint32_t IPV = make_idesc_bf16(128, 128, 0, 1);
  const uint64_t dq = make_sdesc_sw128(smem_u32(sQ), 16, 1024);
  const uint64_t dk = make_sdesc_sw128(smem_u32(sK), 16, 1024);
  const uint64_t dv = make_sdesc_sw128(smem_u32(sV), 64 * 128, 1024);
  if (warp == 0) {
    for (int it = 0; it < reps; ++it) {
      long long t0 = clock64();
      // mode A: PV (8) + QK (8)
      umma_pv64_w(tmem + 0, tmem + 256, dv, IPV, 0);
      umma_pv64_w(tmem + 0, tmem + 256 + 32, dv + 512, IPV, 1);
      umma_qk_tile_w<128, 128>(tmem + 256, dq, dk, IQK);
      long long t1 = clock64();
      umma_commit_w(bar);
      mbar_wait(bar, it & 1);
      long long t2 = clock64();
      // mode B: a single QK MMA tile (8 MMAs)
      umma_qk_tile_w<128, 128>(tmem + 384, dq, dk, IQK);
      umma_commit_w(bar);
      mbar_wait(bar, (it & 1) ^ 1);
      long long t3 = clock64();
      if (threadIdx.x == 0 && it == reps - 1) {
        out[0] = t1 - t0; out[1] = t2 - t0; out[2] = t3 - t2;
      }
    }
    // mode C: 64 back-to-back QK tiles, throughput
    long long t4 = clock64();
    for (int it = 0; it < 64; ++it) umma_qk_tile_w<128, 128>(tmem + 256 + (it & 1) * 128, dq, dk, IQK);
    long long t5 = clock64();
    umma_commit_w(bar);
    mbar_wait(bar, reps & 1);
    long long t6 = clock64();
    // mode E: 64 back-to-back QK tiles at N=64 (8 MMAs each, K tile 64 rows)
    {
      constexpr uint32_t IQ64 = make_idesc_bf16(128, 64, 0, 0);
      long long a0 = clock64();
      for (int it = 0; it < 64; ++it) umma_qk_tile_w<128, 64>(tmem + 256 + (it & 3) * 64, dq, dk, IQ64);
      umma_commit_w(bar);
      mbar_wait(bar, (reps & 1) ^ 1);
      long long a1 = clock64();
      if (threadIdx.x == 0) out[7] = a1 - a0;
    }
    // mode D: 64 back-to-back PV halves (4 MMAs each)
    for (int it = 0; it < 64; ++it) umma_pv64_w(tmem + (it & 1) * 128, tmem + 256, dv, IPV, 1);
    long long t7 = clock64();
    umma_commit_w(bar);
    mbar_wait(bar, reps & 1);
    long long t8 = clock64();
    if (threadIdx.x == 0) { out[3] = t5 - t4; out[4] = t6 - t4; out[5] = t7 - t6; out[6] = t8 - t6; }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<1, 128, 100 * 1024>>>(d, 16);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[8]; cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  printf("64 QK tiles N=64: %lld cyc -> %.1f cyc/MMA (ideal 32)\n", h[7], h[7] / 512.0);
  printf("err=%s\n", cudaGetErrorString(e));
  printf("phase: issue 16 MMAs %lld cyc, issue->commit observed %lld cyc (ideal 1024)\n", h[0], h[1]);
  printf("single QK tile (8 MMAs) issue->observed %lld cyc (ideal 512)\n", h[2]);
  printf("64 QK tiles: issue %lld, done %lld cyc -> %.1f cyc/MMA (ideal 64)\n", h[3], h[4], h[4] / 512.0);
  printf("64 PV halves: issue %lld, done %lld cyc -> %.1f cyc/MMA (ideal 64)\n", h[5], h[6], h[6] / 256.0);
  return 0;
}
