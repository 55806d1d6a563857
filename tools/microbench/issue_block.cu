// Which instructions of the MMA-issuing warp stall behind queued tcgen05.mma
// work?  One warp issues 8 back-to-back 128x128x16 SS MMAs (512 cycles of
// tensor work) and then, one per run, a single probe instruction; clock64
// brackets every step.  Reports cycles: MMA issue, probe, and the probe's
// start relative to the first MMA.
#include "../../paper_2512_07011_b200/csrc/ptx.cuh"
#include <cstdio>
using namespace bsfa;

template <int PROBE>
__global__ void __launch_bounds__(128, 1) k(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const uint32_t bar = smem_u32(base + 131072), bar2 = bar + 8, bar3 = bar + 16;
  uint32_t* tptr = reinterpret_cast<uint32_t*>(base + 131072 + 64);
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar2, 1);
    mbar_init(bar3, 1);
    fence_mbarrier_init();
  }
  if (warp == 0) { tmem_alloc(tptr, 512); tmem_relinquish(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tptr;
  if (threadIdx.x == 0) mbar_arrive(bar2);  // bar2 phase 0 complete: a try_wait on it succeeds at once
  __syncthreads();
  const uint64_t dA = make_sdesc_sw128(smem_u32(base), 16, 1024);
  const uint64_t dB = make_sdesc_sw128(smem_u32(base + 65536), 16, 1024);
  constexpr uint32_t ID = make_idesc_bf16(128, 128, 0, 0);
  if (warp == 0) {
    uint32_t ph = 0;
    for (int rep = 0; rep < 4; ++rep) {
      const long long t0 = clock64();
      umma_qk_chunk_w(tmem, dA, dB, ID, 0u);
      umma_qk_chunk_w(tmem, dA + 1024, dB + 1024, ID, 1u);
      const long long t1 = clock64();
      if constexpr (PROBE == 1) tc_fence_after();
      if constexpr (PROBE == 2) mbar_wait(bar2, 0);
      if constexpr (PROBE == 3) umma_commit_w(bar3);
      if constexpr (PROBE == 4) umma_qk_chunk_w(tmem + 128, dA, dB, ID, 0u);
      if constexpr (PROBE == 5) { tc_fence_after(); mbar_wait(bar2, 0); }
      if constexpr (PROBE == 6) tc_fence_before();
      const long long t2 = clock64();
      umma_commit_w(bar);
      mbar_wait(bar, ph);
      ph ^= 1;
      if constexpr (PROBE == 3) {
        mbar_wait(bar3, rep & 1);
      }
      const long long t3 = clock64();
      if (threadIdx.x == 0 && rep == 3) {
        out[0] = t1 - t0;
        out[1] = t2 - t1;
        out[2] = t3 - t0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int P>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  k<P><<<1, 128, 140 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[3];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-40s %s  issue 8 MMAs %5lld  probe %5lld  total %5lld\n", name, cudaGetErrorString(e), h[0], h[1], h[2]);
  cudaFree(d);
}

int main() {
  run<0>("none");
  run<1>("tcgen05.fence::after_thread_sync");
  run<2>("mbarrier try_wait (complete)");
  run<3>("tcgen05.commit");
  run<4>("4 more MMAs (other accumulator)");
  run<5>("fence::after + try_wait");
  run<6>("tcgen05.fence::before_thread_sync");
  return 0;
}
