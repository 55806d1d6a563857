// MUFU exp2 throughput on one SM-full of warps: f32 vs packed f16x2 / bf16x2.
// Reports exponentials per clock per SM (each packed instruction = 2 exps).
#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t* out, long long* cyc, uint32_t seed, int mode) {
  uint32_t a[16];
  for (int i = 0; i < 16; ++i) a[i] = seed + threadIdx.x * 3 + i * 0x00010001u;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < 2000; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      uint32_t y;
      if (mode == 0) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=r"(y) : "r"(a[i]));
      else if (mode == 1) asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(a[i]));
      else asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(a[i]));
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
  const char* nm[] = {"f32", "f16x2", "bf16x2"};
  for (int mode = 0; mode < 3; ++mode) for (int th : {128, 256, 512}) {
    k<<<148, th>>>(o, c, 0x3f003f00u, mode); k<<<148, th>>>(o, c, 0x3f003f00u, mode); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double ipc = 2000.0 * 16 * th / h;
    printf("%-7s threads %3d: %.2f instr/clk/SM = %.2f exps/clk/SM\n", nm[mode], th, ipc, ipc * (mode ? 2 : 1));
  }
  return 0;
}
