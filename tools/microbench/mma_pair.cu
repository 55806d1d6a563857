// 2-SM tcgen05.mma (cta_group::2) throughput: one CTA pair (cluster of 2),
// CTA 0 issues 512 MMAs of 256xNx16 (128 rows per SM), cycles per MMA as seen
// by the issuing SM.  Ideal (each SM computes 128 x N x 16) = N / 2 cycles.
//   QK: A = SMEM K-major (each CTA's 128 rows), B = SMEM K-major (N/2 rows per CTA)
//   PV: A = TMEM (each CTA's 128 lanes), B = SMEM MN-major (N/2 columns per CTA)
// Also the single-SM cta_group::1 forms for reference.
#include "../../paper_2512_07011_b200/csrc/ptx.cuh"
#include <cstdio>
using namespace bsfa;

__device__ __forceinline__ uint32_t crank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int MODE, int N>
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint32_t at, uint64_t b, uint32_t idesc) {
  if constexpr (MODE == 0)  // 2-SM SS
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 1;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc) : "memory");
  else if constexpr (MODE == 1)  // 2-SM TS
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, 1;\n\t}" ::"r"(d),
                 "r"(at), "l"(b), "r"(idesc) : "memory");
  else if constexpr (MODE == 2)  // 2-SM TS with a disable-output-lane mask (all enabled)
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, {%4, %4, %4, %4, %4, %4, %4, %4}, 1;\n\t}" ::"r"(d),
                 "r"(at), "l"(b), "r"(idesc), "r"(0u) : "memory");
  else if constexpr (MODE == 3)  // 2-SM TS, CTA 1's lanes disabled
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, {%4, %4, %4, %4, %5, %5, %5, %5}, 1;\n\t}" ::"r"(d),
                 "r"(at), "l"(b), "r"(idesc), "r"(0u), "r"(0xffffffffu) : "memory");
}

template <int MODE, int N, int NCH>
__device__ long long run(uint32_t tmem, uint64_t dA, uint64_t dB, int ast, int bst, uint32_t bar, uint32_t& ph) {
  constexpr uint32_t idesc = make_idesc_bf16(256, N, 0, MODE == 0 ? 0 : 1);
  long long best = 1LL << 60;
  for (int rep = 0; rep < 3; ++rep) {
    const long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < 512 / (4 * NCH); ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int c = 0; c < NCH; ++c)
          mma2<MODE, N>(tmem + c * N, dA + kk * ast, tmem + 448 + kk * 8, dB + kk * bst, idesc);
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(bar),
        "h"((unsigned short)3)
        : "memory");
    mbar_wait(bar, ph);
    ph ^= 1;
    const long long t = clock64() - t0;
    if (t < best) best = t;
  }
  return best;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const uint32_t bar = smem_u32(base + 131072);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(base + 131072 + 64);
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = crank();
  if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init(bar + 8, 1); mbar_init(bar + 16, 1); fence_mbarrier_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tptr)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  csync();
  tc_fence_after();
  const uint32_t tmem = *tptr;
  const uint64_t dAk = make_sdesc_sw128(smem_u32(base), 16, 1024);
  const uint64_t dBk = make_sdesc_sw128(smem_u32(base + 65536), 16, 1024);
  const uint64_t dBm = make_sdesc_sw128(smem_u32(base + 65536), 8192, 1024);
  uint32_t ph = 0;
  if (warp < 2 && rank == 0) {
    // two issuing warps: warp 0 QK-style (SS into cols 0..127), warp 1 PV-style (TS into cols 256..383),
    // 256 MMAs each, interleaved in time; vs warp 0 issuing the same 512 alone
    __shared__ long long t2[3];
    if (warp == 0) {
      // one thread, alternating 4 QK + 4 PV
      constexpr uint32_t IQ = make_idesc_bf16(256, 128, 0, 0), IP = make_idesc_bf16(256, 128, 0, 1);
      for (int rep = 0; rep < 2; ++rep) {
        const long long t0 = clock64();
#pragma unroll 1
        for (int it = 0; it < 64; ++it) {
          if (rep == 0) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) mma2<0, 128>(tmem, dAk + kk * 2, 0, dBk + kk * 2, IQ);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) mma2<1, 128>(tmem + 256, 0, tmem + 448 + kk * 8, dBm + kk * 128, IP);
          } else {  // alternate every single MMA
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              mma2<0, 128>(tmem, dAk + kk * 2, 0, dBk + kk * 2, IQ);
              mma2<1, 128>(tmem + 256, 0, tmem + 448 + kk * 8, dBm + kk * 128, IP);
            }
          }
        }
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(bar),
            "h"((unsigned short)3)
            : "memory");
        mbar_wait(bar, ph);
        ph ^= 1;
        t2[rep] = clock64() - t0;
      }
    }
    __syncwarp();
    asm volatile("bar.sync 1, 64;" ::: "memory");
    {
      // two threads: warp 0 the QKs, warp 1 the PVs, each commits its own stream
      const uint32_t bar2 = bar + 8 + 8 * warp;
      constexpr uint32_t IQ = make_idesc_bf16(256, 128, 0, 0), IP = make_idesc_bf16(256, 128, 0, 1);
      const long long t0 = clock64();
#pragma unroll 1
      for (int it = 0; it < 64; ++it) {
        if (warp == 0) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma2<0, 128>(tmem, dAk + kk * 2, 0, dBk + kk * 2, IQ);
        } else {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma2<1, 128>(tmem + 256, 0, tmem + 448 + kk * 8, dBm + kk * 128, IP);
        }
      }
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(bar2),
          "h"((unsigned short)3)
          : "memory");
      mbar_wait(bar2, 0);
      const long long t = clock64() - t0;
      asm volatile("bar.sync 1, 64;" ::: "memory");
      if (warp == 1 && lane_id() == 0) t2[2] = t;
      asm volatile("bar.sync 1, 64;" ::: "memory");
      if (warp == 0 && lane_id() == 0) { out[8] = t2[0]; out[9] = t > t2[2] ? t : t2[2]; out[10] = t2[1]; }
    }
  }
  if (warp == 0 && rank == 0) {
    long long t[8];
    t[0] = run<0, 128, 1>(tmem, dAk, dBk, 2, 2, bar, ph);
    t[1] = run<0, 128, 2>(tmem, dAk, dBk, 2, 2, bar, ph);
    t[2] = run<0, 256, 1>(tmem, dAk, dBk, 2, 2, bar, ph);
    t[3] = run<1, 128, 1>(tmem, dAk, dBm, 2, 128, bar, ph);
    t[4] = run<1, 128, 2>(tmem, dAk, dBm, 2, 128, bar, ph);
    t[5] = run<2, 128, 1>(tmem, dAk, dBm, 2, 128, bar, ph);
    t[6] = run<3, 128, 1>(tmem, dAk, dBm, 2, 128, bar, ph);
    t[7] = run<1, 256, 1>(tmem, dAk, dBm, 2, 128, bar, ph);
    if (threadIdx.x == 0)
      for (int i = 0; i < 8; ++i) out[i] = t[i];
  } else if (warp == 0) {
    // the peer's barrier receives the multicast commits: consume its phases
    for (int i = 0; i < 26; ++i) { mbar_wait(bar, ph); ph ^= 1; }
  }
  tc_fence_before();
  __syncthreads();
  csync();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 128);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  k<<<2, 128, 140 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[11];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(e));
  const char* nm[] = {"2SM SS N=128 (QK) 1 chain", "2SM SS N=128 2 chains", "2SM SS N=256", "2SM TS N=128 (PV) 1 chain",
                      "2SM TS N=128 2 chains", "2SM TS N=128 + lane mask", "2SM TS N=128 CTA1 masked", "2SM TS N=256"};
  const int n[] = {128, 128, 256, 128, 128, 128, 128, 256};
  for (int i = 0; i < 8; ++i)
    printf("%-28s %7.1f cyc/MMA  ideal %4d  frac %.2f\n", nm[i], h[i] / 512.0, n[i] / 2, (n[i] / 2) / (h[i] / 512.0));
  printf("512 MMAs (256 QK SS + 256 PV TS, N=128): one issuing thread, 4+4 groups %.1f cyc/MMA; one thread, alternating "
         "every MMA %.1f; two issuing threads %.1f (ideal 64)\n", h[8] / 512.0, h[10] / 512.0, h[9] / 512.0);
  return 0;
}
