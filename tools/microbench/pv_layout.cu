// Sustained PV MMA rate (128 x d=128 x 16, A = P from TMEM) for the two V
// layouts the kernel could stage: V [keys][d] (B MN-major, what TMA loads from
// the natural layout) vs V^T [d][keys] (B K-major, needs a transposed copy).
// Also QK (SS, K-major) for reference.  4 MMAs per asm block, one elect.
#include "../../paper_2512_07011_b200/csrc/ptx.cuh"
#include <cstdio>
using namespace bsfa;

#define TS4(BSTEP)                                                                                     \
  asm volatile(                                                                                        \
      "{\n\t.reg .pred e;\n\t.reg .b64 b1;\n\t.reg .b32 a1;\n\telect.sync _|e, 0xffffffff;\n\t"       \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"                               \
      "add.s32 a1, %1, 8; add.s64 b1, %2, " #BSTEP ";\n\t"                                             \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, 1;\n\t"                              \
      "add.s32 a1, %1, 16; add.s64 b1, %2, 2*" #BSTEP ";\n\t"                                          \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, 1;\n\t"                              \
      "add.s32 a1, %1, 24; add.s64 b1, %2, 3*" #BSTEP ";\n\t"                                          \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, 1;\n\t}" ::"r"(d_tmem),              \
      "r"(a_tmem), "l"(bdesc), "r"(idesc)                                                               \
      : "memory")

__global__ void __launch_bounds__(128, 1) k(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
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
  const uint32_t a_tmem = tmem + 256;
  uint32_t ph = 0;
  if (warp == 0) {
    // (a) V [keys][d]: MN-major, two 64-col d chunks 8 KB apart (LBO), 16 key rows = +128
    {
      const uint64_t bdesc = make_sdesc_sw128(smem_u32(base), 64 * 128, 1024);
      const uint32_t idesc = make_idesc_bf16(128, 128, 0, 1);
      for (int rep = 0; rep < 2; ++rep) {
        long long t0 = clock64();
        for (int it = 0; it < 64; ++it) {
          const uint32_t d_tmem = tmem + (it & 1) * 128;
          TS4(128);
        }
        umma_commit_w(bar);
        mbar_wait(bar, ph);
        ph ^= 1;
        if (threadIdx.x == 0) out[0] = clock64() - t0;
      }
    }
    // (b) V^T [d][keys]: K-major, 128 d rows x 64 keys (128 B rows), 16 keys = +32 B = +2
    {
      const uint64_t bdesc = make_sdesc_sw128(smem_u32(base + 32768), 16, 1024);
      const uint32_t idesc = make_idesc_bf16(128, 128, 0, 0);
      for (int rep = 0; rep < 2; ++rep) {
        long long t0 = clock64();
        for (int it = 0; it < 64; ++it) {
          const uint32_t d_tmem = tmem + (it & 1) * 128;
          TS4(2);
        }
        umma_commit_w(bar);
        mbar_wait(bar, ph);
        ph ^= 1;
        if (threadIdx.x == 0) out[1] = clock64() - t0;
      }
    }
    // (c) QK SS N=128 (8 MMAs per tile) for reference
    {
      const uint64_t dq = make_sdesc_sw128(smem_u32(base), 16, 1024);
      const uint64_t dk = make_sdesc_sw128(smem_u32(base + 32768), 16, 1024);
      const uint32_t idesc = make_idesc_bf16(128, 128, 0, 0);
      for (int rep = 0; rep < 2; ++rep) {
        long long t0 = clock64();
        for (int it = 0; it < 32; ++it) umma_qk_tile_w<128, 128>(tmem + (it & 1) * 128, dq, dk, idesc);
        umma_commit_w(bar);
        mbar_wait(bar, ph);
        ph ^= 1;
        if (threadIdx.x == 0) out[2] = clock64() - t0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<1, 128, 100 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(e));
  printf("PV TS, V MN-major : %.1f cyc/MMA (ideal 64)\n", h[0] / 256.0);
  printf("PV TS, V K-major  : %.1f cyc/MMA (ideal 64)\n", h[1] / 256.0);
  printf("QK SS N=128       : %.1f cyc/MMA (ideal 64)\n", h[2] / 256.0);
  return 0;
}
