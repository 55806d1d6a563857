// Per-SM throughput of the softmax instruction mix on sm_100a (lanes per clock per SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu && ./pipes
#include <cstdio>
#include <cuda_bf16.h>
#include <cstdint>

constexpr int ITERS = 4096;

template <int OP>
__global__ void k(float* out, long long* cyc, float seed) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-3f + i * 0.1f;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i])); a[i] = y * -0.5f; }
      if (OP == 1) { uint64_t x = (uint64_t(__float_as_uint(a[i])) << 32) | __float_as_uint(a[i]); uint64_t d;
                     asm volatile("fma.rn.f32x2 %0, %1, %1, %1;" : "=l"(d) : "l"(x)); a[i] = __uint_as_float(uint32_t(d)); }
      if (OP == 2) { __nv_bfloat162 v = __floats2bfloat162_rn(a[i], a[i] + 1.f); acc += *reinterpret_cast<uint32_t*>(&v);
                     a[i] = a[i] * 1.0001f; }
      if (OP == 3) { float y; asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(y) : "f"(a[i]), "f"(a[(i + 1) & 7]), "f"(a[(i + 2) & 7])); a[i] = y; }
      if (OP == 4) { a[i] = fmaf(a[i], 0.999f, 0.001f); }
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"MUFU.EX2 (+FMUL)", "FFMA2", "F2FP bf16x2 (+FMUL)", "FMNMX3", "FFMA"};
  for (int op = 0; op < 5; ++op) {
    for (int threads : {128, 512, 1024}) {
      void (*f)(float*, long long*, float) = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : op == 3 ? k<3> : k<4>;
      f<<<148, threads>>>(out, cyc, 0.5f);
      f<<<148, threads>>>(out, cyc, 0.5f);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double ops = double(ITERS) * 8 * threads;
      printf("%-22s threads/SM %5d: %7.2f ops/clk/SM\n", names[op], threads, ops / c);
    }
  }
  return 0;
}
