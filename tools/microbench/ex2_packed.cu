#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
__global__ void k(uint32_t* out, long long* cyc, uint32_t seed, int mode) {
  uint32_t a[16];
  for (int i = 0; i < 16; ++i) a[i] = seed + threadIdx.x * 3 + i * 0x00010001u;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < 2000; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      uint32_t y;
      if (mode == 0) asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(a[i]));
      else asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(a[i]));
      a[i] = y ^ 0x80008000u;
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  uint32_t* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
  for (int mode = 0; mode < 2; ++mode) for (int th : {128, 512}) {
    k<<<148, th>>>(o, c, 0x3f803f80u, mode); k<<<148, th>>>(o, c, 0x3f803f80u, mode); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%s threads %d: %.2f instr/clk/SM (%.2f exps/clk/SM)\n", mode ? "f16x2" : "bf16x2", th, 2000.0 * 16 * th / h, 2 * 2000.0 * 16 * th / h);
  }
  // accuracy check on host-visible values
  return 0;
}
