// Issue-slot cost of warps waiting on an mbarrier while a compute warp on the
// same SMSP runs: warp 0 does a fixed MUFU+FFMA workload, warps 4, 8 (same
// SMSP) wait on a barrier warp 0 completes at the end.
#include "../../paper_2512_07011_b200/csrc/ptx.cuh"
#include <cstdio>
using namespace bsfa;

template <int MODE>
__device__ __forceinline__ void wait_mode(uint32_t bar, uint32_t ph) {
  if (MODE == 0) { while (!mbar_try_wait(bar, ph)) {} }
  if (MODE == 1) { while (!mbar_try_wait_sleep(bar, ph, 10000000u)) {} }
  if (MODE == 2) { while (!mbar_try_wait_sleep(bar, ph, 1000u)) {} }
  if (MODE == 3) {
    uint32_t ok;
    do {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
      if (!ok) __nanosleep(256);
    } while (!ok);
  }
}

template <int MODE>
__global__ void k(long long* out, int nwait, float seed) {
  __shared__ __align__(8) uint64_t barmem;
  const uint32_t bar = smem_u32(&barmem);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbarrier_init(); }
  __syncthreads();
  if (warp == 0) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = seed + threadIdx.x * 1e-3f + i;
    long long t0 = clock64();
    for (int it = 0; it < 2000; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float y = ex2_approx(a[i] * -0.01f);
        a[i] = fmaf(y, 0.5f, a[i]);
      }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; mbar_arrive(bar); }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    if (s == 12345.f) out[1] = 1;
  } else if ((warp & 3) == 0 && warp / 4 <= nwait) {
    wait_mode<MODE>(bar, 0);
  }
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  const char* nm[] = {"try_wait spin", "try_wait hint 10ms", "try_wait hint 1us", "test_wait+nanosleep256"};
  for (int mode = 0; mode < 4; ++mode)
    for (int nw = 0; nw <= 2; ++nw) {
      auto f = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : k<3>;
      f<<<1, 384>>>(d, nw, 1.f);
      f<<<1, 384>>>(d, nw, 1.f);
      cudaDeviceSynchronize();
      long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("%-24s waiters on SMSP %d: compute warp %lld cycles\n", nm[mode], nw, h);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
