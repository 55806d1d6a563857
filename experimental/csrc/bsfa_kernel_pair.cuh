// BSFA forward (K1) on CTA pairs (cta_group::2): the "pair" kernel, b_n = 64,
// d = 128, GQA groups of 4 (or a multiple).
//
// A cluster of two CTAs (the two SMs of a TPC) owns one kv head x one query
// block i x four q heads of the group: CTA r holds query tiles of heads
// 4p + 2r + {0, 1}.  Every MMA is a 2-SM MMA issued by CTA 0 alone:
//   QK_s :  M = 256 (tile s of both CTAs) x N = 128 keys x K = 128;
//           each CTA stages only its 64 keys of the step (B is split on N)
//   PV_s :  M = 256 x N = d = 128 x K = 64 keys per gate tile;
//           each CTA stages only its 64 d-columns of V (B split on N); a CTA
//           whose head skipped the gate tile is masked out of the output
//           (disable-output-lane), so skipping stays per head
// Halving the K/V bytes each SM stages frees the shared memory for ALL of P:
// P_{s,h} (bf16, 128 rows x 64 keys) lives in SMEM, S_s holds nothing once
// the softmax has loaded it, and QK_s(j+1) is issued right then -- the S/P
// chain of the one-CTA kernel is gone; each query tile's step is bounded by
// its softmax alone.
//
// TMEM per CTA (512 columns): O_0, O_1 (fp32, 128 cols, zeroed at start,
// always accumulated) and S_0, S_1 (fp32, 128 cols).
// SMEM per CTA: Q_0, Q_1 (64 KB) | K ring 3 x 16 KB | V ring 6 x 8 KB (slot of
// gate tile (j, h) = (2j + h) mod 6) | P_{s,h} 4 x 16 KB.
//
// Cross-CTA protocol (barriers live at the same offsets in both CTAs; "L" =
// only CTA 0's copy is used):
//   bar_q, k_full, v_full (L): both CTAs' producers arrive.expect_tx; their
//        TMAs (cta_group::2) complete on CTA 0's barrier
//   k_empty, v_empty, s_full, pv_done, o_full: 2-SM commits multicast to both
//   s_free[s] (L, 8 warps), p0_full[s][j&1] (L, 8 warps: P of keys 0-63
//        written, decisions posted), p1_full[s][r] (L, 4 warps of CTA r, only
//        when CTA r kept keys 64-127)
//   decisions: CTA r's tile lead stores its bits into CTA 0's decm slots and
//        into both CTAs' V-producer rings (st.shared::cluster + remote arrive)
#pragma once

#include "bsfa_kernel.cuh"

namespace bsfa {

// ---------------------------------------------------------------- CTA-pair PTX
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// Cross-CTA signalling without cluster-scope fences (a release.cluster arrive
// compiles to MEMBAR.ALL.GPU, an acquire.cluster wait to an L1 invalidate):
// barriers are arrived with the default (CTA-scope) semantics, and the only
// generic data one CTA hands to the other -- the gate decisions -- travels as
// st.async, whose completion is counted on the consumer's mbarrier (like TMA).
__device__ __forceinline__ void mbar_arrive_cl(uint32_t cl) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cl) : "memory");
}
// single-thread arrive that also expects `bytes` of st.async / TMA data on that phase
__device__ __forceinline__ void mbar_arrive_expect_tx_cl(uint32_t cl, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;" ::"r"(cl), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_cl_w(uint32_t cl, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;\n\t}" ::"r"(cl),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ bool mbar_test_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// 4-byte store into another CTA's shared memory, completing on that CTA's barrier
__device__ __forceinline__ void st_async_u32(uint32_t cl_addr, uint32_t v, uint32_t cl_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(cl_addr), "r"(v),
               "r"(cl_bar)
               : "memory");
}
// TMA whose completion lands on the pair leader's barrier (bar = CTA 0's address)
__device__ __forceinline__ void tma_load_4d_2sm_w(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0,
                                                  int c1, int c2, int c3, uint64_t policy) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;\n\t}" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar), "l"(policy)
      : "memory");
}
// 2-SM commit, arriving on the barrier at `bar` in both CTAs of the pair
__device__ __forceinline__ void umma_commit2_w(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::
          "r"(bar),
      "h"((unsigned short)3)
      : "memory");
}
// S = Q K^T, M = 256 (both CTAs' tile), N = 128 keys (64 staged per CTA), K = 128
#define BSFA_QK2_STEP(A, B, ACC) \
  "add.s64 a1, %1, " #A "; add.s64 b1, %2, " #B ";\n\t@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, " #ACC ";\n\t"
__device__ __forceinline__ void umma2_qk_w(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred e;\n\t.reg .b64 a1, b1;\n\telect.sync _|e, 0xffffffff;\n\t"
               BSFA_QK2_STEP(0, 0, 0) BSFA_QK2_STEP(2, 2, 1) BSFA_QK2_STEP(4, 4, 1) BSFA_QK2_STEP(6, 6, 1)
               BSFA_QK2_STEP(1024, 512, 1) BSFA_QK2_STEP(1026, 514, 1) BSFA_QK2_STEP(1028, 516, 1)
               BSFA_QK2_STEP(1030, 518, 1) "}" ::"r"(d_tmem), "l"(a), "l"(b), "r"(idesc)
               : "memory");
}
#undef BSFA_QK2_STEP
// O += P V over one 64-key gate tile, M = 256, N = d = 128 (64 staged per CTA),
// always accumulating (O zeroed at start); lanes of a CTA that skipped the tile
// are disabled (m0: CTA 0's 128 rows, m1: CTA 1's)
#define BSFA_PV2_STEP(A, B) \
  "add.s64 a1, %1, " #A "; add.s64 b1, %2, " #B ";\n\t"                                          \
  "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, {%4, %4, %4, %4, %5, %5, %5, %5}, 1;\n\t"
__device__ __forceinline__ void umma2_pv64_w(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t m0,
                                             uint32_t m1) {
  asm volatile("{\n\t.reg .pred e;\n\t.reg .b64 a1, b1;\n\telect.sync _|e, 0xffffffff;\n\t"
               BSFA_PV2_STEP(0, 0) BSFA_PV2_STEP(2, 128) BSFA_PV2_STEP(4, 256) BSFA_PV2_STEP(6, 384) "}" ::"r"(d_tmem),
               "l"(a), "l"(b), "r"(idesc), "r"(m0), "r"(m1)
               : "memory");
}
#undef BSFA_PV2_STEP

struct PairCfg {
  static constexpr int D = 128, NQ = 2, GT = 2;
  static constexpr int Q_TILE = 128 * D * 2;  // 32 KB
  static constexpr int K_HALF = 64 * D * 2;   // this CTA's 64 keys of a 128-key step: 16 KB
  static constexpr int V_HALF = 64 * 64 * 2;  // 64 keys x this CTA's 64 d-columns: 8 KB
  static constexpr int P_TILE = 128 * 64 * 2; // 128 rows x 64 keys: 16 KB
  static constexpr int KS = 3, VS = 6, DQ = 4;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + NQ * Q_TILE;
  static constexpr int OFF_V = OFF_K + KS * K_HALF;
  static constexpr int OFF_P = OFF_V + VS * V_HALF;
  static constexpr int OFF_BAR = OFF_P + NQ * 2 * P_TILE;
  // bar_q, k_full/empty, v_full/empty, s_full, s_free, p0_full[2], p1_full[2], pv_done, o_full,
  // dec_full/empty
  static constexpr int NUM_BARS = 1 + 2 * KS + 2 * VS + NQ * 8 + 2 * DQ;
  static constexpr int OFF_DEC = (OFF_BAR + NUM_BARS * 8 + 15) / 16 * 16;  // u32 [DQ][2 ranks][NQ]
  static constexpr int OFF_DECM = OFF_DEC + DQ * 2 * NQ * 4;              // u32 [2 parities][2 ranks][NQ]
  static constexpr int OFF_TMEMPTR = OFF_DECM + 2 * 2 * NQ * 4;
  static constexpr int SMEM_BYTES = OFF_TMEMPTR + 16 + 1024;
  static constexpr int O_COL = 0, S_COL = NQ * D;
  static constexpr int TMEM_COLS = 512;
  static constexpr int SOFTMAX_WARPS = 8, KPROD_WARP = 8, MMA_WARP = 9, VPROD_WARP = 10;
  static constexpr int NUM_THREADS = 12 * 32;
  static constexpr int REG_LAUNCH = 168, REG_OTHER = 56, REG_SOFT = 224;
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
  static_assert(NUM_THREADS * REG_LAUNCH >= 256 * REG_SOFT + 128 * REG_OTHER, "register pool");
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PairCfg::NUM_THREADS, 1)
    bsfa_kernel_pair(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const KernelParams p) {
  using C = PairCfg;
  constexpr int D = C::D, NQ = C::NQ, GT = C::GT, KS = C::KS, VS = C::VS, DQ = C::DQ;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = opaque_u32((sraw + 1023u) & ~1023u);
  uint8_t* smem = smem_raw + (sbase - sraw);
  const uint32_t sQ = sbase + C::OFF_Q;
  const uint32_t sK = sbase + C::OFF_K;
  const uint32_t sV = sbase + C::OFF_V;
  const uint32_t sP = sbase + C::OFF_P;
  const uint32_t bar_q = sbase + C::OFF_BAR;
  const uint32_t k_full = bar_q + 8;              // [KS]      L
  const uint32_t k_empty = k_full + 8 * KS;       // [KS]
  const uint32_t v_full = k_empty + 8 * KS;       // [VS]      L
  const uint32_t v_empty = v_full + 8 * VS;       // [VS]
  const uint32_t s_full = v_empty + 8 * VS;       // [NQ]
  const uint32_t s_free = s_full + 8 * NQ;        // [NQ]      L
  const uint32_t p0_full = s_free + 8 * NQ;       // [NQ][2]   L (step parity)
  const uint32_t p1_full = p0_full + 16 * NQ;     // [NQ][2]   L (rank)
  const uint32_t pv_done = p1_full + 16 * NQ;     // [NQ]
  const uint32_t o_full = pv_done + 8 * NQ;       // [NQ]
  const uint32_t dec_full = o_full + 8 * NQ;      // [DQ]
  const uint32_t dec_empty = dec_full + 8 * DQ;   // [DQ]
  const uint32_t dec_sm = sbase + C::OFF_DEC;
  const uint32_t decm_sm = sbase + C::OFF_DECM;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEMPTR);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const uint32_t peer = rank ^ 1u;
  auto lead = [&](uint32_t a) { return mapa_u32(a, 0); };  // CTA 0's copy
  auto other = [&](uint32_t a) { return mapa_u32(a, peer); };

  // ---- work unit: (batch, kv head) major, heaviest query block first, quads of q heads minor
  const int quads = p.group / 4;
  const int per_bg = p.num_q_tiles * quads;
  const int unit = blockIdx.x >> 1;
  const int bg = unit / per_bg;
  const int rem = unit - bg * per_bg;
  const int qi = p.num_q_tiles - 1 - rem / quads;
  const int pq = rem - (rem / quads) * quads;
  const int b = bg / p.heads_kv;
  const int g = bg - b * p.heads_kv;
  const int hq0 = g * p.group + pq * 4 + int(rank) * 2;  // this CTA's q heads hq0, hq0 + 1
  const int nsteps = p.causal ? qi + 1 : p.num_steps;
  const int gate_mode = p.gate_mode;
  const int window = p.gate_window;
  const bool causal = p.causal != 0;
  const int valid_len = p.valid_len;

  if (warp == C::KPROD_WARP && lane == 0) {
    mbar_init(bar_q, 2);
    for (int i = 0; i < KS; ++i) {
      mbar_init(k_full + 8 * i, 2);
      mbar_init(k_empty + 8 * i, 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(v_full + 8 * i, 2);
      mbar_init(v_empty + 8 * i, 1);
    }
    for (int s = 0; s < NQ; ++s) {
      mbar_init(s_full + 8 * s, 1);
      mbar_init(s_free + 8 * s, 8);
      mbar_init(p0_full + 16 * s, 8);
      mbar_init(p0_full + 16 * s + 8, 8);
      mbar_init(p1_full + 16 * s, 4);
      mbar_init(p1_full + 16 * s + 8, 4);
      mbar_init(pv_done + 8 * s, 1);
      mbar_init(o_full + 8 * s, 1);
    }
    for (int i = 0; i < DQ; ++i) {
      mbar_init(dec_full + 8 * i, 4);
      mbar_init(dec_empty + 8 * i, 2);
    }
    fence_mbarrier_init();
  }
  if (warp == C::MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_ptr)),
                 "r"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_arrive();
  cluster_wait();  // both CTAs' barriers initialised and TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;

  if (warp == C::KPROD_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
    // ======================= TMA producer: own Q tiles, own 64 keys of each K step
    if (nsteps > 0) {
      if (lane == 0) {
        tma_prefetch_desc(&tm_q);
        tma_prefetch_desc(&tm_k);
      }
      const uint32_t lq = lead(bar_q);
      mbar_arrive_expect_tx_cl_w(lq, NQ * C::Q_TILE);
#pragma unroll
      for (int s = 0; s < NQ; ++s)
#pragma unroll
        for (int c = 0; c < 2; ++c)
          tma_load_4d_2sm_w(sQ + s * C::Q_TILE + c * 128 * 128, &tm_q, lq, c * 64, qi * 128, hq0 + s, b, kEvictFirst);
      for (int j = 0; j < nsteps; ++j) {
        const int st = j % KS;
        mbar_wait(k_empty + 8 * st, ((j / KS) & 1) ^ 1);
        const uint32_t lk = lead(k_full + 8 * st);
        mbar_arrive_expect_tx_cl_w(lk, C::K_HALF);
#pragma unroll
        for (int c = 0; c < 2; ++c)
          tma_load_4d_2sm_w(sK + st * C::K_HALF + c * 64 * 128, &tm_k, lk, c * 64, j * 128 + int(rank) * 64, g, b,
                            kEvictLast);
      }
    }
    __syncwarp();
    cluster_arrive();
    return;
  } else if (warp == C::VPROD_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
    // ======================= TMA producer: own 64 d-columns of every gate tile some head keeps
    if (nsteps > 0) {
      if (lane == 0) tma_prefetch_desc(&tm_v);
      uint32_t use_par = 0;  // bit slot: v_empty phase of the slot
      unsigned dn = 0, loads = 0;
      for (int j = 0; j < nsteps; ++j) {
        const int sb = step_static_bits<GT>(gate_mode, window, j, qi);
        uint32_t u;
        if (sb >= 0) {
          u = uint32_t(sb);
        } else {
          const int di = int(dn % DQ);
          mbar_wait(dec_full + 8 * di, (dn / DQ) & 1);
          u = 0;
#pragma unroll
          for (int x = 0; x < 2 * NQ; ++x) u |= lds_u32(dec_sm + (di * 2 * NQ + x) * 4);
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(dec_empty + 8 * di);
            mbar_arrive_cl(other(dec_empty + 8 * di));
          }
          ++dn;
        }
#pragma unroll
        for (int h = 0; h < GT; ++h) {
          if (!((u >> h) & 1u)) continue;
          const int slot = (2 * j + h) % VS;
          mbar_wait(v_empty + 8 * slot, ((use_par >> slot) & 1u) ^ 1u);
          use_par ^= 1u << slot;
          const uint32_t lv = lead(v_full + 8 * slot);
          mbar_arrive_expect_tx_cl_w(lv, C::V_HALF);
          tma_load_4d_2sm_w(sV + slot * C::V_HALF, &tm_v, lv, int(rank) * 64, j * 128 + h * 64, g, b, kEvictLast);
          ++loads;
        }
      }
      if (rank == 0 && lane == 0 && p.counters) {
        atomicAdd(&p.counters[2], (unsigned long long)loads);
        atomicAdd(&p.counters[3], (unsigned long long)nsteps * GT);
      }
    }
    __syncwarp();
    cluster_arrive();
    return;
  } else if (warp == C::MMA_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
    // ======================= 2-SM MMA issuer (CTA 0 only)
    if (rank == 0 && nsteps > 0) {
      constexpr uint32_t IDESC_QK = make_idesc_bf16(256, 128, 0, 0);
      constexpr uint32_t IDESC_PV = make_idesc_bf16(256, D, 0, 1);
      const uint64_t dq0 = make_sdesc_sw128(sQ, 16, 1024);
      const uint64_t dk0 = make_sdesc_sw128(sK, 16, 1024);
      const uint64_t dv0 = make_sdesc_sw128(sV, 64 * 128, 1024);
      const uint64_t dp0 = make_sdesc_sw128(sP, 16, 1024);
      mbar_wait(bar_q, 0);

      // In-order issue (an event-driven loop that polls every barrier measured
      // 10.4 ms vs 7.1: the spinning warp takes issue slots from two softmax warps)
      auto issue_qk = [&](int s, int j) {
        const int st = j % KS;
        if (s == 0) mbar_wait(k_full + 8 * st, (j / KS) & 1);
        tc_fence_after();
        umma2_qk_w(tmem + C::S_COL + s * 128, dq0 + uint64_t((s * C::Q_TILE) >> 4),
                   dk0 + uint64_t((st * C::K_HALF) >> 4), IDESC_QK);
        if (s == NQ - 1) umma_commit2_w(k_empty + 8 * st);
        umma_commit2_w(s_full + 8 * s);
      };
#pragma unroll
      for (int s = 0; s < NQ; ++s) issue_qk(s, 0);

      uint32_t vfull_par = 0;  // bit slot: v_full phase
      uint32_t p1_par = 0;     // bit 2s + r: p1_full phase
      for (int j = 0; j < nsteps; ++j) {
        // the next QK of each tile as soon as both CTAs' softmax read S_s(j)
        if (j + 1 < nsteps) {
#pragma unroll
          for (int s = 0; s < NQ; ++s) {
            mbar_wait(s_free + 8 * s, j & 1);
            issue_qk(s, j + 1);
          }
        }
        const int sb = step_static_bits<GT>(gate_mode, window, j, qi);
        uint32_t used = 0;    // gate tiles of this step kept by some head
        uint32_t waited = 0;  // V slots already waited for this step
#pragma unroll
        for (int s = 0; s < NQ; ++s) {
          mbar_wait(p0_full + 16 * s + 8 * (j & 1), (j >> 1) & 1);
          tc_fence_after();
          const uint32_t b0 = sb >= 0 ? uint32_t(sb) : lds_u32(decm_sm + (((j & 1) * 2 + 0) * NQ + s) * 4);
          const uint32_t b1 = sb >= 0 ? uint32_t(sb) : lds_u32(decm_sm + (((j & 1) * 2 + 1) * NQ + s) * 4);
#pragma unroll
          for (int h = 0; h < GT; ++h) {
            if (h == 1) {
              // P_{s,1} of every CTA that kept keys 64-127
              if ((b0 >> 1) & 1u) {
                mbar_wait(p1_full + 16 * s, (p1_par >> (2 * s)) & 1u);
                p1_par ^= 1u << (2 * s);
              }
              if ((b1 >> 1) & 1u) {
                mbar_wait(p1_full + 16 * s + 8, (p1_par >> (2 * s + 1)) & 1u);
                p1_par ^= 1u << (2 * s + 1);
              }
              tc_fence_after();
            }
            const uint32_t k0 = (b0 >> h) & 1u, k1 = (b1 >> h) & 1u;
            if (!(k0 | k1)) continue;
            const int slot = (2 * j + h) % VS;
            if (!((waited >> slot) & 1u)) {
              mbar_wait(v_full + 8 * slot, (vfull_par >> slot) & 1u);
              waited |= 1u << slot;
              tc_fence_after();
            }
            used |= 1u << h;
            umma2_pv64_w(tmem + C::O_COL + s * D, dp0 + uint64_t(((2 * s + h) * C::P_TILE) >> 4),
                         dv0 + uint64_t((slot * C::V_HALF) >> 4), IDESC_PV, k0 ? 0u : 0xffffffffu,
                         k1 ? 0u : 0xffffffffu);
          }
          umma_commit2_w(pv_done + 8 * s);  // one completion per step: P_s buffers free, O_s current
          if (j == nsteps - 1) umma_commit2_w(o_full + 8 * s);
        }
#pragma unroll
        for (int h = 0; h < GT; ++h)
          if ((used >> h) & 1u) {
            const int slot = (2 * j + h) % VS;
            umma_commit2_w(v_empty + 8 * slot);
            vfull_par ^= 1u << slot;
          }
      }
    }
    __syncwarp();
    cluster_arrive();
    cluster_wait();  // every role of both CTAs is done with TMEM
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS) : "memory");
    return;
  } else if (warp < C::SOFTMAX_WARPS) {
    setmaxnreg_inc<C::REG_SOFT>();
    // ======================= softmax of this CTA's query tile s, one thread per row
    const int s = warp >> 2;
    const int wq = warp & 3;
    const int r = wq * 32 + lane;
    const int hq = hq0 + s;
    const uint32_t lane_off = uint32_t(wq * 32) << 16;
    const uint32_t s_row = tmem + lane_off + C::S_COL + s * 128;
    const uint32_t o_row = tmem + lane_off + C::O_COL + s * D;
    const float sl2 = p.scale_log2;
    const float scale = p.scale;
    const float rescale_raw = p.rescale_raw;
    const float lam = p.gate_lambda;
    const uint32_t l_sfree = lead(s_free + 8 * s);
    const uint32_t l_p1 = lead(p1_full + 16 * s + 8 * rank);

    // O_s starts at zero: every PV accumulates (a skipping CTA is masked out, not "first")
    {
      uint32_t z[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) z[c] = 0u;
#pragma unroll
      for (int c = 0; c < D; c += 32) tmem_st32(o_row + c, z);
      tmem_wait_st();
    }

    float T = 0.f;
    if (gate_mode == kGateThreshold) {
      const int pos = qi < p.thr_positions - 1 ? qi : p.thr_positions - 1;
      T = p.thr[(long long)hq * p.thr_positions + pos];
    }
    float m_true = -INFINITY;
    float m_ref = -INFINITY;
    float l_sum = 0.f;
    bool o_valid = false;
    unsigned dn = 0;
    unsigned long long kept_tiles = 0;

    for (int j = 0; j < nsteps; ++j) {
      mbar_wait(s_full + 8 * s, j & 1);
      tc_fence_after();
      uint32_t sv[128];
#pragma unroll
      for (int c = 0; c < 128; c += 32) tmem_ld32(s_row + c, &sv[c]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cl(l_sfree);  // S_s may take QK_s(j+1) (after the peer's warps too)

      const int sb = step_static_bits<GT>(gate_mode, window, j, qi);
      if (j == qi && causal) {
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (c > r) sv[c] = __float_as_uint(-INFINITY);
      }
      if (!causal && (j + 1) * 128 > valid_len) {
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (j * 128 + c >= valid_len) sv[c] = __float_as_uint(-INFINITY);
      }
      float mh[2];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const uint32_t* x = sv + hh * 64;
        float a0 = fmax3(__uint_as_float(x[0]), __uint_as_float(x[1]), __uint_as_float(x[2]));
        float a1 = fmax3(__uint_as_float(x[3]), __uint_as_float(x[4]), __uint_as_float(x[5]));
        float a2 = fmax3(__uint_as_float(x[6]), __uint_as_float(x[7]), __uint_as_float(x[8]));
        float a3 = fmax3(__uint_as_float(x[9]), __uint_as_float(x[10]), __uint_as_float(x[11]));
#pragma unroll
        for (int c = 12; c < 60; c += 8) {
          a0 = fmax3(a0, __uint_as_float(x[c]), __uint_as_float(x[c + 1]));
          a1 = fmax3(a1, __uint_as_float(x[c + 2]), __uint_as_float(x[c + 3]));
          a2 = fmax3(a2, __uint_as_float(x[c + 4]), __uint_as_float(x[c + 5]));
          a3 = fmax3(a3, __uint_as_float(x[c + 6]), __uint_as_float(x[c + 7]));
        }
        a0 = fmax3(a0, __uint_as_float(x[60]), __uint_as_float(x[61]));
        a1 = fmax3(a1, __uint_as_float(x[62]), __uint_as_float(x[63]));
        mh[hh] = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3));
      }

      // ---- gate decision (OR over this tile's 128 rows in the barrier hardware)
      uint32_t bits;
      if (sb >= 0) {
        bits = uint32_t(sb);
      } else if (gate_mode == kGateThreshold) {
        bits = named_bar_red_or(1 + s, 128, mh[0] * scale > T ? 1u : 0u);
        bits |= named_bar_red_or(1 + s, 128, mh[1] * scale > T ? 1u : 0u) << 1;
      } else {
        bits = 0;
        float mrun = m_true;
#pragma unroll
        for (int x = 0; x < GT; ++x) {
          const uint32_t k = named_bar_red_or(1 + s, 128, (mh[x] - mrun) * scale >= lam ? 1u : 0u);
          bits |= k << x;
          if (k) mrun = fmaxf(mrun, mh[x]);
        }
      }
      if (gate_mode == kGateRunMax) {
#pragma unroll
        for (int x = 0; x < GT; ++x)
          if ((bits >> x) & 1u) m_true = fmaxf(m_true, mh[x]);
      }
      const uint32_t l_p0 = lead(p0_full + 16 * s + 8 * (j & 1));
      if (r == 0) {
        if (sb < 0) {  // both CTAs' V producers need every head's decision
          const int di = int(dn % DQ);
          mbar_wait(dec_empty + 8 * di, ((dn / DQ) & 1) ^ 1);
          const uint32_t slot = dec_sm + (di * 2 * NQ + rank * NQ + s) * 4;
          sts_u32(slot, bits);
          mbar_arrive(dec_full + 8 * di);
          const uint32_t pbar = other(dec_full + 8 * di);
          st_async_u32(other(slot), bits, pbar);
          mbar_arrive_expect_tx_cl(pbar, 4);
        }
        const uint32_t dslot = decm_sm + (((j & 1) * 2 + rank) * NQ + s) * 4;
        if (rank == 0)
          sts_u32(dslot, bits);
        else
          st_async_u32(lead(dslot), bits, l_p0);  // counted by warp 0's arrive.expect_tx below
        kept_tiles += __popc(bits);
        if (p.decisions) {
          int8_t* drow = p.decisions + (((long long)b * p.heads_q + hq) * p.num_q_tiles + qi) * p.gate_cols;
#pragma unroll
          for (int x = 0; x < GT; ++x)
            drow[j * GT + x] = j == qi ? int8_t(2) : (((bits >> x) & 1u) ? int8_t(3) : int8_t(1));
        }
      }
      if (sb < 0) ++dn;
      // P_{s,0} barrier: CTA 1's warp 0 arrival also expects its st.async decision
      auto arrive_p0 = [&]() {
        if (lane == 0) {
          if (rank == 1 && wq == 0)
            mbar_arrive_expect_tx_cl(l_p0, 4);
          else
            mbar_arrive_cl(l_p0);
        }
      };
      if (bits == 0) {
        __syncwarp();
        arrive_p0();
        continue;
      }

      float m_step = -INFINITY;
#pragma unroll
      for (int x = 0; x < GT; ++x)
        if ((bits >> x) & 1u) m_step = fmaxf(m_step, mh[x]);
      const float m_new = fmaxf(m_ref, m_step);
      float alpha = 1.f;
      bool rescale = false;
      if (!o_valid) {
        m_ref = m_new;
      } else if (m_new > m_ref + rescale_raw) {
        alpha = ex2_approx((m_ref - m_new) * sl2);
        m_ref = m_new;
        rescale = true;
      }
      // the previous step's PVs of this tile have landed: P buffers free, O_s current
      if (j > 0) mbar_wait(pv_done + 8 * s, (j - 1) & 1);
      if (__any_sync(0xffffffffu, rescale)) {
        tc_fence_after();
        const uint64_t ax2 = f2_pack(alpha, alpha);
#pragma unroll
        for (int c = 0; c < D; c += 32) {
          uint32_t ov[32];
          tmem_ld32(o_row + c, ov);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const uint64_t t = fmul2(f2_pack(__uint_as_float(ov[e]), __uint_as_float(ov[e + 1])), ax2);
            ov[e] = __float_as_uint(f2_lo(t));
            ov[e + 1] = __float_as_uint(f2_hi(t));
          }
          tmem_st32(o_row + c, ov);
        }
        tmem_wait_st();
        tc_fence_before();
      }

      const float neg = (m_ref == -INFINITY) ? 0.f : -m_ref * sl2;
      const uint64_t sl2x2 = f2_pack(sl2, sl2);
      const uint64_t negx2 = f2_pack(neg, neg);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const bool kept_h = ((bits >> hh) & 1u) != 0;
        if (kept_h) {
          uint32_t pk[32];
#pragma unroll
          for (int c = 0; c < 64; c += 4) {
            const int e = hh * 64 + c;
            const uint64_t x0 = ffma2(f2_pack(__uint_as_float(sv[e]), __uint_as_float(sv[e + 1])), sl2x2, negx2);
            const uint64_t x1 = ffma2(f2_pack(__uint_as_float(sv[e + 2]), __uint_as_float(sv[e + 3])), sl2x2, negx2);
            const float p0 = ex2_approx(f2_lo(x0)), p1 = ex2_approx(f2_hi(x0));
            const float p2 = ex2_approx(f2_lo(x1)), p3 = ex2_approx(f2_hi(x1));
            sv[e] = __float_as_uint(p0);
            sv[e + 1] = __float_as_uint(p1);
            sv[e + 2] = __float_as_uint(p2);
            sv[e + 3] = __float_as_uint(p3);
            pk[c / 2] = pack_bf16x2(p0, p1);
            pk[c / 2 + 1] = pack_bf16x2(p2, p3);
          }
          const uint32_t prow = sP + (2 * s + hh) * C::P_TILE + r * 128;
#pragma unroll
          for (int c16 = 0; c16 < 8; ++c16)
            sts_u128(prow + ((c16 ^ (r & 7)) << 4), pk[4 * c16], pk[4 * c16 + 1], pk[4 * c16 + 2], pk[4 * c16 + 3]);
          fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core
        }
        __syncwarp();
        if (hh == 0) {
          arrive_p0();  // decisions + P_{s,0}
        } else if (kept_h) {
          if (lane == 0) mbar_arrive_cl(l_p1);  // P_{s,1}, only when kept
        }
      }

      uint64_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        if ((bits >> hh) & 1u) {
#pragma unroll
          for (int c = 0; c < 64; c += 8) {
            const int e = hh * 64 + c;
            acc0 = fadd2(acc0, f2_pack(__uint_as_float(sv[e]), __uint_as_float(sv[e + 1])));
            acc1 = fadd2(acc1, f2_pack(__uint_as_float(sv[e + 2]), __uint_as_float(sv[e + 3])));
            acc2 = fadd2(acc2, f2_pack(__uint_as_float(sv[e + 4]), __uint_as_float(sv[e + 5])));
            acc3 = fadd2(acc3, f2_pack(__uint_as_float(sv[e + 6]), __uint_as_float(sv[e + 7])));
          }
        }
      }
      const uint64_t acc = fadd2(fadd2(acc0, acc1), fadd2(acc2, acc3));
      l_sum = l_sum * alpha + (f2_lo(acc) + f2_hi(acc));
      o_valid = true;
    }

    // ---- epilogue: O = O~ / l, lse = m * scale + ln l (engine.py:178-182)
    mbar_wait(o_full + 8 * s, 0);
    tc_fence_after();
    const float inv_l = 1.f / l_sum;
    bool bad = !(l_sum > 0.f);
    const int row = qi * 128 + r;
    const long long orow = (long long)b * p.o_sb + (long long)hq * p.o_sh + (long long)row * p.o_sn;
#pragma unroll
    for (int c = 0; c < D; c += 32) {
      uint32_t ov[32];
      tmem_ld32(o_row + c, ov);
      tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        float a0 = __uint_as_float(ov[e]) * inv_l, a1 = __uint_as_float(ov[e + 1]) * inv_l;
        if (p.inject_fault && qi == 0 && r == 0 && hq == 0 && c == 0 && e == 0) a0 += 1.0f;  // O[0][0] += 1
        bad |= !isfinite(a0) || !isfinite(a1);
        pk[e / 2] = pack_bf16x2(a0, a1);
      }
      store_o32(p, orow + c, pk);
    }
    p.lse[((long long)b * p.heads_q + hq) * p.seq_len + row] = m_ref * scale + logf(l_sum);
    if (bad && p.status) atomicOr(p.status, 1);
    if (r == 0 && p.counters) {
      atomicAdd(&p.counters[0], (unsigned long long)nsteps * GT);
      atomicAdd(&p.counters[1], kept_tiles);
    }
    tc_fence_before();
    cluster_arrive();
    return;
  } else {
    setmaxnreg_dec<C::REG_OTHER>();
    cluster_arrive();
    return;
  }
}

}  // namespace bsfa
