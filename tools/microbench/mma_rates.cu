// Sustained tcgen05.mma rates (cycles per 128xNx16 bf16 MMA) for the operand
// layouts the BSFA kernel can use, one CTA on one SM, nothing else running.
#include "../../paper_2512_07011_b200/csrc/ptx.cuh"
#include <cstdio>
using namespace bsfa;

#define TS4(ADD_B) asm volatile("{\n\t.reg .pred e;\n\t.reg .b64 b1;\n\t.reg .b32 a1;\n\telect.sync _|e, 0xffffffff;\n\t" \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t" \
  "add.s32 a1, %1, 8; add.s64 b1, %2, " #ADD_B "*1;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, 1;\n\t" \
  "add.s32 a1, %1, 16; add.s64 b1, %2, " #ADD_B "*2;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, 1;\n\t" \
  "add.s32 a1, %1, 24; add.s64 b1, %2, " #ADD_B "*3;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, 1;\n\t}" \
  ::"r"(dcol), "r"(tmem + 256), "l"(B), "r"(ID) : "memory")
#define SS4(ADD_B) asm volatile("{\n\t.reg .pred e;\n\t.reg .b64 a1, b1;\n\telect.sync _|e, 0xffffffff;\n\t" \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t" \
  "add.s64 a1, %1, 2; add.s64 b1, %2, " #ADD_B "*1;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t" \
  "add.s64 a1, %1, 4; add.s64 b1, %2, " #ADD_B "*2;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t" \
  "add.s64 a1, %1, 6; add.s64 b1, %2, " #ADD_B "*3;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t}" \
  ::"r"(dcol), "l"(dA), "l"(B), "r"(ID) : "memory")

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(idesc) : "memory");
}

__global__ void __launch_bounds__(128, 1) k(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const uint32_t bar = smem_u32(base + 131072);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(base + 131072 + 64);
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbarrier_init(); }
  if (warp == 0) { tmem_alloc(tptr, 512); tmem_relinquish(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tptr;
  const uint64_t dA = make_sdesc_sw128(smem_u32(base), 16, 1024);             // K-major A (128 rows)
  const uint64_t dBk = make_sdesc_sw128(smem_u32(base + 32768), 16, 1024);    // K-major B
  const uint64_t dBm = make_sdesc_sw128(smem_u32(base + 65536), 64 * 128, 1024);  // MN-major B, 64-row K chunks
  uint32_t ph = 0;
  auto timeit = [&](int which) {
    long long t0 = clock64();
    for (int it = 0; it < 64; ++it) {
      const uint32_t dcol = tmem + (it & 1) * 128;
      switch (which) {
        case 0: { const uint64_t B = dBk; constexpr uint32_t ID = make_idesc_bf16(128, 128, 0, 0); SS4(2); } break;
        case 1: { const uint64_t B = dBk; constexpr uint32_t ID = make_idesc_bf16(128, 64, 0, 0); SS4(2); } break;
        case 2: { const uint64_t B = dBm; constexpr uint32_t ID = make_idesc_bf16(128, 128, 0, 1); TS4(128); } break;
        case 3: { const uint64_t B = dBk; constexpr uint32_t ID = make_idesc_bf16(128, 128, 0, 0); TS4(2); } break;
        case 4: { const uint64_t B = dBm; constexpr uint32_t ID = make_idesc_bf16(128, 128, 0, 1); SS4(128); } break;
        case 5: { const uint64_t B = dBk; constexpr uint32_t ID = make_idesc_bf16(128, 256, 0, 0); TS4(2); } break;
        case 6: { const uint64_t B = dBk; constexpr uint32_t ID = make_idesc_bf16(128, 256, 0, 0); SS4(2); } break;
      }
    }
    umma_commit_w(bar);
    mbar_wait(bar, ph);
    ph ^= 1;
    return clock64() - t0;
  };
  if (warp == 0) {
    for (int w = 0; w < 7; ++w) {
      timeit(w);
      long long c = timeit(w);
      if (threadIdx.x == 0) out[w] = c;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  k<<<1, 128, 140 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[8]; cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(e));
  const char* nm[] = {"QK SS N=128 K-major", "QK SS N=64", "PV TS N=128 V MN-major", "PV TS N=128 V K-major",
                      "PV SS N=128 V MN-major", "TS N=256 K-major", "SS N=256"};
  const double ideal[] = {64, 32, 64, 64, 64, 128, 128};
  for (int w = 0; w < 7; ++w) printf("%-26s %6.1f cyc/MMA (ideal %.0f)\n", nm[w], h[w] / 256.0, ideal[w]);
  return 0;
}
