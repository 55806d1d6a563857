// tcgen05.mma kind::f16 throughput by operand source / major-ness / N and the
// number of independent accumulation chains, one CTA on one SM: cycles per
// 128xNx16 MMA over 512 MMAs issued round-robin over NCH accumulators
// (NCH = 1: every MMA accumulates onto the previous one's result).
//   A: T = TMEM, K = SMEM K-major SW128, M = SMEM MN-major SW128
//   B: K = SMEM K-major SW128, M = SMEM MN-major SW128
// Ideal (floor) = N / 2 cycles per MMA (8192 bf16 FLOP/clk/SM).
// Everything is a template parameter: the issue loop is a straight line of
// UTCHMMAs on uniform registers.
#include "../../paper_2512_07011_b200/csrc/ptx.cuh"
#include <cstdio>
using namespace bsfa;

template <char A>
__device__ __forceinline__ void mma1(uint32_t d, uint64_t a, uint32_t at, uint64_t b, uint32_t idesc) {
  if constexpr (A == 'T')
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t}" ::"r"(d),
                 "r"(at), "l"(b), "r"(idesc) : "memory");
  else
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc) : "memory");
}

template <char A, char B, int N, int NCH>
__device__ long long run(uint32_t tmem, uint32_t sA, uint32_t sB, uint32_t bar, uint32_t& ph) {
  constexpr uint32_t idesc = make_idesc_bf16(128, N, A == 'M' ? 1 : 0, B == 'M' ? 1 : 0);
  // K-major SW128: SBO 1024 (8-row groups), +32 B per K16 (= +2)
  // MN-major SW128: LBO 8192 (next 64-element MN atom), SBO 1024, +2048 B per K16 (= +128)
  const uint64_t dA = A == 'M' ? make_sdesc_sw128(sA, 8192, 1024) : make_sdesc_sw128(sA, 16, 1024);
  const uint64_t dB = B == 'M' ? make_sdesc_sw128(sB, 8192, 1024) : make_sdesc_sw128(sB, 16, 1024);
  constexpr int AST = A == 'M' ? 128 : 2, BST = B == 'M' ? 128 : 2;
  long long best = 1LL << 60;
  for (int rep = 0; rep < 3; ++rep) {
    const long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < 512 / (4 * NCH); ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int c = 0; c < NCH; ++c)
          mma1<A>(tmem + c * N, dA + kk * AST, tmem + 448 + kk * 8, dB + kk * BST, idesc);
    }
    umma_commit_w(bar);
    mbar_wait(bar, ph);
    ph ^= 1;
    const long long t = clock64() - t0;
    if (t < best) best = t;
  }
  return best;
}

template <char A, char B, int N, int NCH>
__device__ void one(long long* out, int& i, uint32_t tmem, uint32_t sA, uint32_t sB, uint32_t bar, uint32_t& ph) {
  const long long t = run<A, B, N, NCH>(tmem, sA, sB, bar, ph);
  if (threadIdx.x == 0) {
    out[4 * i] = A;
    out[4 * i + 1] = B;
    out[4 * i + 2] = N * 16 + NCH;
    out[4 * i + 3] = t;
  }
  ++i;
}

template <char A, char B>
__device__ void ab(long long* out, int& i, uint32_t tmem, uint32_t sA, uint32_t sB, uint32_t bar, uint32_t& ph) {
  one<A, B, 64, 1>(out, i, tmem, sA, sB, bar, ph);
  one<A, B, 64, 2>(out, i, tmem, sA, sB, bar, ph);
  one<A, B, 64, 4>(out, i, tmem, sA, sB, bar, ph);
  one<A, B, 128, 1>(out, i, tmem, sA, sB, bar, ph);
  one<A, B, 128, 2>(out, i, tmem, sA, sB, bar, ph);
  one<A, B, 128, 3>(out, i, tmem, sA, sB, bar, ph);
  one<A, B, 256, 1>(out, i, tmem, sA, sB, bar, ph);
}

__global__ void __launch_bounds__(128, 1) k(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const uint32_t bar = smem_u32(base + 196608);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(base + 196608 + 64);
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbarrier_init(); }
  if (warp == 0) { tmem_alloc(tptr, 512); tmem_relinquish(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tptr;
  const uint32_t sA = smem_u32(base), sB = smem_u32(base + 65536);
  uint32_t ph = 0;
  int i = 0;
  if (warp == 0) {
    ab<'T', 'K'>(out, i, tmem, sA, sB, bar, ph);
    ab<'T', 'M'>(out, i, tmem, sA, sB, bar, ph);
    ab<'K', 'K'>(out, i, tmem, sA, sB, bar, ph);
    ab<'K', 'M'>(out, i, tmem, sA, sB, bar, ph);
    ab<'M', 'K'>(out, i, tmem, sA, sB, bar, ph);
    ab<'M', 'M'>(out, i, tmem, sA, sB, bar, ph);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 4 * 64);
  cudaMemset(d, 0, 8 * 4 * 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<1, 128, 200 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long r[4 * 64];
  cudaMemcpy(r, d, sizeof(r), cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(e));
  printf("A B    N chains  cyc/MMA  ideal  frac\n");
  for (int i = 0; i < 42; ++i) {
    const int n = int(r[4 * i + 2] / 16), nch = int(r[4 * i + 2] % 16);
    const double c = r[4 * i + 3] / 512.0;
    printf("%c %c %4d %4d    %7.1f  %5d  %.2f\n", char(r[4 * i]), char(r[4 * i + 1]), n, nch, c, n / 2, (n / 2) / c);
  }
  return 0;
}
