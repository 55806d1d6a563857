// Warp-to-warp hand-off latency inside one CTA: two warps (different SMSPs)
// ping-pong N times; cycles per one-way hand-off.  Modes:
//   0 mbarrier arrive / try_wait loop        1 mbarrier arrive / test_wait spin
//   2 named barrier (bar.arrive / bar.sync)  3 shared-memory flag (st / volatile ld spin)
//   4 tcgen05.commit (no MMA outstanding) -> mbarrier -> try_wait
#include "../../paper_2512_07011_b200/csrc/ptx.cuh"
#include <cstdio>
using namespace bsfa;

__device__ __forceinline__ bool test_wait(uint32_t bar, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
  return ok != 0;
}

template <int MODE>
__global__ void k(long long* out, int n) {
  __shared__ __align__(8) uint64_t barmem[2];
  __shared__ volatile uint32_t flag[2];
  __shared__ uint32_t tptr;
  const uint32_t bar0 = smem_u32(&barmem[0]), bar1 = smem_u32(&barmem[1]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(bar0, 1); mbar_init(bar1, 1); fence_mbarrier_init(); flag[0] = flag[1] = 0; }
  if (MODE == 4 && warp == 0) { tmem_alloc(&tptr, 32); tmem_relinquish(); }
  __syncthreads();
  if (warp > 1) return;
  const uint32_t mine = warp == 0 ? bar0 : bar1, other = warp == 0 ? bar1 : bar0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const uint32_t ph = i & 1;
    if (warp == 0) {
      // signal, then wait for the reply
      if (MODE == 0 || MODE == 1) { __syncwarp(); if (lane == 0) mbar_arrive(other); }
      if (MODE == 2) named_bar_arrive(1, 64);
      if (MODE == 3) { __syncwarp(); if (lane == 0) flag[1] = i + 1; }
      if (MODE == 4) umma_commit_w(other);
      if (MODE == 0 || MODE == 4) { while (!mbar_try_wait(mine, ph)) {} }
      if (MODE == 1) { while (!test_wait(mine, ph)) {} }
      if (MODE == 2) named_bar_sync(2, 64);
      if (MODE == 3) { while (flag[0] != uint32_t(i + 1)) {} }
    } else {
      if (MODE == 0 || MODE == 4) { while (!mbar_try_wait(mine, ph)) {} }
      if (MODE == 1) { while (!test_wait(mine, ph)) {} }
      if (MODE == 2) named_bar_sync(1, 64);
      if (MODE == 3) { while (flag[1] != uint32_t(i + 1)) {} }
      if (MODE == 0 || MODE == 1) { __syncwarp(); if (lane == 0) mbar_arrive(other); }
      if (MODE == 2) named_bar_arrive(2, 64);
      if (MODE == 3) { __syncwarp(); if (lane == 0) flag[0] = i + 1; }
      if (MODE == 4) umma_commit_w(other);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (MODE == 4) { __syncwarp(); }
  if (MODE == 4 && warp == 0) { tmem_dealloc(tptr, 32); }
}

int main() {
  long long* d; cudaMalloc(&d, 8);
  const char* nm[] = {"mbarrier try_wait", "mbarrier test_wait spin", "named barrier", "smem flag spin", "tcgen05.commit->mbarrier"};
  const int n = 10000;
  for (int m = 0; m < 5; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      if (m == 0) k<0><<<1, 64>>>(d, n);
      if (m == 1) k<1><<<1, 64>>>(d, n);
      if (m == 2) k<2><<<1, 64>>>(d, n);
      if (m == 3) k<3><<<1, 64>>>(d, n);
      if (m == 4) k<4><<<1, 64>>>(d, n);
    }
    cudaError_t e = cudaDeviceSynchronize();
    long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %7.1f cycles per one-way hand-off (%s)\n", nm[m], h / (2.0 * n), cudaGetErrorString(e));
  }
  return 0;
}
