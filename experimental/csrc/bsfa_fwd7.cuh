// BSFA forward (K1) for sm_100a, v7: CTA pairs (cta_group::2), ONE query tile
// per CTA, double-buffered scores and P in tensor memory, two softmax threads
// per row.
//
// A cluster of two CTAs (the two SMs of a TPC) owns two q heads of one GQA
// group at query block i; CTA r holds the 128-row query tile of head
// g*group + 2*pair + r.  Every MMA is a 2-SM MMA issued by CTA 0:
//   QK(j) : M = 256 (both CTAs' tiles) x N = 128 keys x K = D;
//           each CTA stages only its 64 keys of the step (B split on N)
//   PV(j) : M = 256 x N = D x K = 64 keys per kept 64-key half; A = P from
//           each CTA's tensor memory, each CTA stages only its D/2 columns of
//           V (B split on N); a CTA whose head skipped the gate tile has its
//           output lanes disabled, so skipping stays per head (gates.py:77-78)
// Keys stream in steps of 128 (GT = 128 / b_n gate tiles of the reference,
// tiling.py:19-69).
//
// TMEM per CTA (512 columns): O (fp32, D = 128 columns), S[2] (fp32, 128
// columns each), P[2] (bf16 pairs, 64 columns each).  Step j uses S[j&1] and
// P[j&1].  QK(j+2) is issued as soon as both CTAs' softmax copied S(j) into
// registers (s_free), before their exponentials; the PVs trail by a step,
// so the tensor pipe runs, in issue order,
//   ... QK(j+2)  PV(j-1)  QK(j+3)  PV(j) ...
// and the V unit of step j-1 (requested after that step's vote) has had a
// whole step to land.  The softmax rewrites P[j&1] at step j+2 only after
// pv_done[j&1] says PV(j) read it, and rescales O only after PV(j-1) landed.
//
// Warp roles per CTA (384 threads):
//   warps 0-3 / 4-7  softmax, key half 0 / 1 of the step: thread (h, r) owns
//                    row r (TMEM lane r) and the 64 keys h*64..h*64+63; the
//                    two threads of a row share the running max through
//                    shared memory at the per-step vote barrier
//   warp 8           TMA: own Q tile once, own 64 keys of every K step
//   warp 9           CTA 0: 2-SM tcgen05 issuer; both CTAs: TMEM owner.  One
//                    thread issues every MMA (tools/microbench/mma_pair.cu:
//                    QKs and PVs from two issuing threads interleaved in the
//                    pipe run at 1/3 of the rate of the same stream from one)
//   warp 10          TMA: own D/2 columns of every 64-key V unit kept by
//                    either CTA's head (decisions exchanged through a ring)
//   warp 11          idle (completes the warpgroup for setmaxnreg)
// Cross-CTA protocol (barriers at the same offsets in both CTAs; "L" = only
// CTA 0's copy is used):
//   bar_q, k_full, v_full (L): both CTAs' producers arrive.expect_tx, their
//        TMAs (cta_group::2) complete on CTA 0's barrier
//   s_free[2], p_full[4] (L): 8 softmax warps of each CTA; CTA 1's gate bits
//        travel as st.async into CTA 0's decm words, counted on p_full.  A
//        warp can be up to three steps ahead of the slowest one at p_full
//        (QK(j+2) needs only the S(j) loads), hence four p_full / decm slots
//   k_empty, v_empty, s_full[2], pv_done[2], o_full: 2-SM commits multicast to both
//   dec ring: each CTA's bits into both CTAs' V-producer rings
#pragma once

#include "../../paper_2512_07011_b200/csrc/bsfa_common.cuh"

namespace bsfa {

// ---------------------------------------------------------------- CTA-pair PTX
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_rel() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acq() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_cta(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// arrive on a barrier of either CTA of the cluster (CTA-scope semantics)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cl) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cl) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_cluster(uint32_t cl, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;" ::"r"(cl), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_cluster_w(uint32_t cl, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;\n\t}" ::"r"(cl),
      "r"(bytes)
      : "memory");
}
// 4-byte store into the peer CTA's shared memory, completing on its barrier
__device__ __forceinline__ void st_async_b32(uint32_t cl_addr, uint32_t v, uint32_t cl_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(cl_addr), "r"(v),
               "r"(cl_bar)
               : "memory");
}
// TMA whose completion lands on the pair leader's barrier (bar = CTA 0's address)
__device__ __forceinline__ void tma_load_4d_pair_w(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                                   int c2, int c3, uint64_t policy) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;\n\t}" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar), "l"(policy)
      : "memory");
}
// 2-SM commit: arrives on the barrier at `bar` in both CTAs of the pair
__device__ __forceinline__ void umma_commit_pair_w(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::
          "r"(bar),
      "h"((unsigned short)3)
      : "memory");
}
// S = Q K^T over D = 128: M = 256, N = 128 keys (64 staged per CTA), 8 MMAs.
// A (Q): 128 rows x 128 B atoms, +32 B per K16, next atom +16 KB (+1024);
// B (this CTA's 64 keys): 64 rows x 128 B atoms, next atom +8 KB (+512).
#define BSFA_QKP_STEP(A, B, ACC) \
  "add.s64 a1, %1, " #A "; add.s64 b1, %2, " #B ";\n\t@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, " #ACC ";\n\t"
__device__ __forceinline__ void umma_pair_qk_w(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred e;\n\t.reg .b64 a1, b1;\n\telect.sync _|e, 0xffffffff;\n\t"
               BSFA_QKP_STEP(0, 0, 0) BSFA_QKP_STEP(2, 2, 1) BSFA_QKP_STEP(4, 4, 1) BSFA_QKP_STEP(6, 6, 1)
               BSFA_QKP_STEP(1024, 512, 1) BSFA_QKP_STEP(1026, 514, 1) BSFA_QKP_STEP(1028, 516, 1)
               BSFA_QKP_STEP(1030, 518, 1) "}" ::"r"(d_tmem), "l"(a), "l"(b), "r"(idesc)
               : "memory");
}
#undef BSFA_QKP_STEP
// O += P V over one 64-key half: M = 256, N = D (D/2 staged per CTA), K = 64
// as 4 MMAs; P (bf16) from TMEM (+8 columns per 16 keys), V MN-major SW128
// (+2 KB per 16 keys); always accumulating (O zeroed at start); lanes of a CTA
// that skipped the half are disabled (m0: CTA 0's rows, m1: CTA 1's).
#define BSFA_PVP_STEP(A, B) \
  "add.s32 a1, %1, " #A "; add.s64 b1, %2, " #B ";\n\t"                                           \
  "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a1], b1, %3, {%4, %4, %4, %4, %5, %5, %5, %5}, 1;\n\t"
__device__ __forceinline__ void umma_pair_pv64_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                                 uint32_t m0, uint32_t m1) {
  asm volatile("{\n\t.reg .pred e;\n\t.reg .b64 b1;\n\t.reg .b32 a1;\n\telect.sync _|e, 0xffffffff;\n\t"
               BSFA_PVP_STEP(0, 0) BSFA_PVP_STEP(8, 128) BSFA_PVP_STEP(16, 256) BSFA_PVP_STEP(24, 384) "}" ::"r"(d_tmem),
               "r"(a_tmem), "l"(b), "r"(idesc), "r"(m0), "r"(m1)
               : "memory");
}
#undef BSFA_PVP_STEP

template <int GT>
struct FCfg7 {
  static constexpr int D = 128;
  static constexpr int Q_TILE = 128 * D * 2;   // 32 KB: this CTA's query tile
  static constexpr int Q_ATOM = 128 * 128;     // 128 rows x 128 bytes
  static constexpr int K_HALF = 64 * D * 2;    // this CTA's 64 keys of a step: 16 KB
  static constexpr int V_HALF = 64 * 64 * 2;   // 64 keys x this CTA's 64 columns: 8 KB
  static constexpr int KS = 4, VS = 10, DQ = 8;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_TILE;
  static constexpr int OFF_V = OFF_K + KS * K_HALF;
  static constexpr int OFF_BAR = OFF_V + VS * V_HALF;
  // bar_q, k_full/empty[KS], v_full/empty[VS], s_full[2], s_free[2], p_full[4],
  // pv_done[2], o_full, dec_full/empty[DQ]
  static constexpr int NUM_BARS = 1 + 2 * KS + 2 * VS + 2 + 2 + 4 + 2 + 1 + 2 * DQ;
  static constexpr int OFF_VOTE = (OFF_BAR + NUM_BARS * 8 + 15) / 16 * 16;  // u32 [2 parity][8 warps]
  static constexpr int OFF_RMAX = OFF_VOTE + 2 * 8 * 4;                   // f32 [2 parity][2 halves][128]
  static constexpr int OFF_LSUM = OFF_RMAX + 2 * 2 * 128 * 4;             // f32 [2 halves][128]
  static constexpr int OFF_DEC = OFF_LSUM + 2 * 128 * 4;                  // u32 [DQ][2 ranks]
  static constexpr int OFF_DECM = OFF_DEC + DQ * 2 * 4;                   // u32 [4 slots][2 ranks]
  static constexpr int OFF_TMEMPTR = OFF_DECM + 4 * 2 * 4;
  static constexpr int SMEM_BYTES = OFF_TMEMPTR + 16 + 1024;
  static constexpr int O_COL = 0, S_COL = 128, P_COL = 384;  // S[b] at S_COL + 128 b, P[b] at P_COL + 64 b
  static constexpr int TMEM_COLS = 512;
  static constexpr int NUM_THREADS = 12 * 32;
  static constexpr int KPROD_WARP = 8, MMA_WARP = 9, VPROD_WARP = 10;
  static constexpr int REG_OTHER = 88;  // producers / issuer keep their descriptors in registers
  static constexpr int REG_LAUNCH = (65536 / NUM_THREADS) / 8 * 8;                            // 168
  static constexpr int REG_SOFT = (NUM_THREADS * REG_LAUNCH - 128 * REG_OTHER) / 256 / 8 * 8;  // 208
  static_assert(GT == 1 || GT == 2, "b_n in {64, 128}");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
};

// GM: gate class -- 0 ThresholdGate (voted), 1 statically known steps (DenseGate,
// FrontierOnlyGate, SlidingWindowGate), 2 RunningMaxGate (voted).
template <int GT, int GM, bool CAUSAL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(FCfg7<GT>::NUM_THREADS, 1)
    bsfa_fwd7_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const KernelParams p) {
  using C = FCfg7<GT>;
  constexpr int D = C::D, KS = C::KS, VS = C::VS, DQ = C::DQ;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = opaque_u32((sraw + 1023u) & ~1023u);
  uint8_t* smem = smem_raw + (sbase - sraw);
  const uint32_t sQ = sbase + C::OFF_Q;
  const uint32_t sK = sbase + C::OFF_K;
  const uint32_t sV = sbase + C::OFF_V;
  const uint32_t bar_q = sbase + C::OFF_BAR;     // L
  const uint32_t k_full = bar_q + 8;             // [KS] L
  const uint32_t k_empty = k_full + 8 * KS;      // [KS]
  const uint32_t v_full = k_empty + 8 * KS;      // [VS] L
  const uint32_t v_empty = v_full + 8 * VS;      // [VS]
  const uint32_t s_full = v_empty + 8 * VS;      // [2]  QK(j) landed in S[j&1]
  const uint32_t s_free = s_full + 16;           // [2]  L: both CTAs copied S(j) to registers (16 warps)
  const uint32_t p_full = s_free + 16;           // [4]  L: step j decided, P[j&1] written (16 warps)
  const uint32_t pv_done = p_full + 32;          // [2]  PV(j) landed (one phase per step of that parity)
  const uint32_t o_full = pv_done + 16;          //      last PV landed
  const uint32_t dec_full = o_full + 8;          // [DQ]
  const uint32_t dec_empty = dec_full + 8 * DQ;  // [DQ]
  const uint32_t vote_sm = sbase + C::OFF_VOTE;
  const uint32_t rmax_sm = sbase + C::OFF_RMAX;
  const uint32_t lsum_sm = sbase + C::OFF_LSUM;
  const uint32_t dec_sm = sbase + C::OFF_DEC;
  const uint32_t decm_sm = sbase + C::OFF_DECM;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEMPTR);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const uint32_t peer = rank ^ 1u;
  auto lead = [&](uint32_t a) { return mapa_cta(a, 0); };
  auto other = [&](uint32_t a) { return mapa_cta(a, peer); };

  // ---- work unit: (batch, kv head) major, heaviest query block first, head
  //      pairs of the group minor (the v3 order, one head per CTA)
  const int pairs = p.group / 2;
  const int per_bg = p.num_q_tiles * pairs;
  const int unit = int(blockIdx.x >> 1);
  const int bg = unit / per_bg;
  const int rem = unit - bg * per_bg;
  const int qi = p.num_q_tiles - 1 - rem / pairs;
  const int pr = rem - (rem / pairs) * pairs;
  const int b = bg / p.heads_kv;
  const int g = bg - b * p.heads_kv;
  const int hq = g * p.group + 2 * pr + int(rank);
  const int nsteps = CAUSAL ? qi + 1 : p.num_steps;
  const int gate_mode = p.gate_mode;
  const int window = p.gate_window;
  auto sbits = [&](int j) -> int {
    if constexpr (GM == 1) return step_static_bits<GT>(gate_mode, window, j, qi);
    return j == qi ? (1 << GT) - 1 : -1;  // frontier (tiling.py:50-60)
  };
  // debug timeline (-DBSFA_TRACE=1 builds only): clock64 per (event, rank, step)
  // of one cluster (p.trace_cta = cluster index)
  const bool tr_cta = BSFA_TRACE && p.trace && unit == p.trace_cta;
  auto trace = [&](int ev, int j) {
    if (BSFA_TRACE && tr_cta && j < kTraceSteps) p.trace[(ev * 2 + int(rank)) * kTraceSteps + j] = clock64();
  };

  // ---- setup (both CTAs), then a cluster barrier before any remote access
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
    for (int s = 0; s < 2; ++s) {
      mbar_init(s_full + 8 * s, 1);
      mbar_init(s_free + 8 * s, 16);
      mbar_init(p_full + 8 * s, 16);
      mbar_init(p_full + 16 + 8 * s, 16);
      mbar_init(pv_done + 8 * s, 1);
    }
    mbar_init(o_full, 1);
    for (int i = 0; i < DQ; ++i) {
      mbar_init(dec_full + 8 * i, 2);
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
  cluster_sync_all();  // both CTAs' barriers initialised and TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;

  if (warp == C::KPROD_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
    // ======================= TMA: own Q tile, own 64 keys of every K step =======
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
    }
    const uint32_t lq = lead(bar_q);
    mbar_arrive_expect_tx_cluster_w(lq, C::Q_TILE);
#pragma unroll
    for (int c = 0; c < 2; ++c)
      tma_load_4d_pair_w(sQ + c * C::Q_ATOM, &tm_q, lq, c * 64, qi * 128, hq, b, kEvictFirst);
    for (int j = 0; j < nsteps; ++j) {
      const int st = j % KS;
      mbar_wait(k_empty + 8 * st, ((j / KS) & 1) ^ 1);
      const uint32_t lk = lead(k_full + 8 * st);
      mbar_arrive_expect_tx_cluster_w(lk, C::K_HALF);
#pragma unroll
      for (int c = 0; c < 2; ++c)
        tma_load_4d_pair_w(sK + st * C::K_HALF + c * (C::K_HALF / 2), &tm_k, lk, c * 64, j * 128 + int(rank) * 64, g,
                           b, kEvictLast);
    }
    __syncwarp();
    named_bar_arrive(15, C::NUM_THREADS);
  } else if (warp == C::VPROD_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
    // ======================= TMA: own 64 columns of every V unit either head kept ==
    if (lane == 0) tma_prefetch_desc(&tm_v);
    unsigned dn = 0, vcount = 0;
    for (int j = 0; j < nsteps; ++j) {
      const int sb = sbits(j);
      uint32_t u;
      if (sb >= 0) {
        u = uint32_t(sb);
      } else {
        const int di = int(dn % DQ);
        mbar_wait(dec_full + 8 * di, (dn / DQ) & 1);
        u = lds_u32(dec_sm + di * 8) | lds_u32(dec_sm + di * 8 + 4);
        if (lane == 0) trace(13, j);
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(dec_empty + 8 * di);
          mbar_arrive_cluster(other(dec_empty + 8 * di));
        }
        ++dn;
      }
      const uint32_t hb = GT == 2 ? u : (u ? 3u : 0u);  // 64-key halves used by the pair
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        if (!((hb >> hh) & 1u)) continue;
        const int slot = int(vcount % VS);
        mbar_wait(v_empty + 8 * slot, ((vcount / VS) & 1) ^ 1);
        const uint32_t lv = lead(v_full + 8 * slot);
        mbar_arrive_expect_tx_cluster_w(lv, C::V_HALF);
        tma_load_4d_pair_w(sV + slot * C::V_HALF, &tm_v, lv, int(rank) * 64, j * 128 + hh * 64, g, b, kEvictLast);
        ++vcount;
        if (lane == 0) trace(14, j);
      }
    }
    if (rank == 0 && lane == 0 && p.counters) {
      // per pair: one fetch of a 64-key unit serves both heads (b_n = 128: two units per gate tile)
      atomicAdd(&p.counters[2], (unsigned long long)(vcount / (3 - GT)));
      atomicAdd(&p.counters[3], (unsigned long long)nsteps * GT);
    }
    __syncwarp();
    named_bar_arrive(15, C::NUM_THREADS);
  } else if (warp == C::MMA_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
    // ======================= 2-SM tcgen05 issuer (CTA 0 only) =====================
    if (rank == 0) {
      constexpr uint32_t IDESC_QK = make_idesc_bf16(256, 128, 0, 0);
      constexpr uint32_t IDESC_PV = make_idesc_bf16(256, D, 0, 1);
      const uint64_t dq0 = make_sdesc_sw128(sQ, 16, 1024);
      const uint64_t dk0 = make_sdesc_sw128(sK, 16, 1024);
      const uint64_t dv0 = make_sdesc_sw128(sV, C::V_HALF, 1024);
      mbar_wait(bar_q, 0);
      auto issue_qk = [&](int j) {  // into S[j&1]
        const int st = j % KS;
        mbar_wait(k_full + 8 * st, (j / KS) & 1);
        if (lane == 0) trace(10, j);
        tc_fence_after();
        umma_pair_qk_w(tmem + C::S_COL + (j & 1) * 128, dq0, dk0 + uint64_t((st * C::K_HALF) >> 4), IDESC_QK);
        umma_commit_pair_w(k_empty + 8 * st);
        umma_commit_pair_w(s_full + 8 * (j & 1));
        if (lane == 0) trace(5, j);
      };
      unsigned vcount = 0;
      auto issue_pv = [&](int j) {
        mbar_wait(p_full + 8 * (j & 3), (j >> 2) & 1);
        if (lane == 0) trace(6, j);
        tc_fence_after();
        const int sb = sbits(j);
        uint32_t b0, b1;
        if (sb >= 0) {
          b0 = b1 = uint32_t(sb);
        } else {
          b0 = lds_u32(decm_sm + (j & 3) * 8);
          b1 = lds_u32(decm_sm + (j & 3) * 8 + 4);
        }
        const uint32_t h0 = GT == 2 ? b0 : (b0 ? 3u : 0u), h1 = GT == 2 ? b1 : (b1 ? 3u : 0u);
        const uint32_t hu = h0 | h1;
        unsigned nunits = 0;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if (!((hu >> hh) & 1u)) continue;
          const unsigned uu = vcount + nunits++;
          mbar_wait(v_full + 8 * (uu % VS), (uu / VS) & 1);
          if (lane == 0) trace(11, j);
          tc_fence_after();
          umma_pair_pv64_w(tmem + C::O_COL, tmem + C::P_COL + (j & 1) * 64 + hh * 32,
                           dv0 + uint64_t(((uu % VS) * C::V_HALF) >> 4), IDESC_PV,
                           ((h0 >> hh) & 1u) ? 0u : 0xffffffffu, ((h1 >> hh) & 1u) ? 0u : 0xffffffffu);
        }
        umma_commit_pair_w(pv_done + 8 * (j & 1));
        if (lane == 0) trace(7, j);
        if (j == nsteps - 1) umma_commit_pair_w(o_full);
        for (unsigned x = 0; x < nunits; ++x) umma_commit_pair_w(v_empty + 8 * ((vcount + x) % VS));
        vcount += nunits;
      };
      issue_qk(0);
      if (nsteps > 1) issue_qk(1);
      for (int j = 0; j <= nsteps; ++j) {
        // the scores two steps ahead as soon as both CTAs read S(j), then the
        // previous step's PVs
        if (j + 2 < nsteps) {
          mbar_wait(s_free + 8 * (j & 1), (j >> 1) & 1);
          issue_qk(j + 2);
        }
        if (j >= 1) issue_pv(j - 1);
      }
    }
    __syncwarp();
    named_bar_sync(15, C::NUM_THREADS);
    cluster_sync_all();  // both CTAs are done with their tensor memory
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS) : "memory");
    return;
  } else if (warp < 8) {
    setmaxnreg_inc<C::REG_SOFT>();
    // ======================= softmax: thread (h, r) = row r, keys h*64 .. h*64+63 ====
    const int h = warp >> 2;
    const int wq = warp & 3;
    const int r = wq * 32 + lane;
    const uint32_t lane_off = uint32_t(wq * 32) << 16;
    const uint32_t o_row = tmem + lane_off + C::O_COL + h * 64;  // this thread's 64 output columns
    const float sl2 = p.scale_log2;
    const float scale = p.scale;
    const float rescale_raw = p.rescale_raw;
    const int valid_len = p.valid_len;
    const uint32_t lp_full = lead(p_full);
    const uint32_t ls_free = lead(s_free);

    // O starts at zero: every PV accumulates (a skipping CTA is masked out)
    {
      uint32_t z[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) z[c] = 0u;
      tmem_st32(o_row, z);
      tmem_st32(o_row + 32, z);
      tmem_wait_st();
    }
    float T = 0.f;
    if constexpr (GM == 0) {
      const int pos = qi < p.thr_positions - 1 ? qi : p.thr_positions - 1;
      T = p.thr[(long long)hq * p.thr_positions + pos];  // thresholds.py:87
    }
    const float lam = p.gate_lambda;
    float m_true = -INFINITY;  // exact running row max (RunningMaxGate), raw units
    float m_ref = -INFINITY;   // raw reference max of this row over its kept tiles
    float l_sum = 0.f;         // this thread's half of the row sum, relative to m_ref
    bool o_valid = false;
    unsigned dn = 0;
    unsigned nb = 0;  // vote barriers passed (double-buffers the vote words / row maxima)
    unsigned long long kept_tiles = 0;
    int8_t* drow = p.decisions ? p.decisions + (((long long)b * p.heads_q + hq) * p.num_q_tiles + qi) * p.gate_cols
                               : nullptr;

    for (int j = 0; j < nsteps; ++j) {
      const int par = j & 1;
      mbar_wait(s_full + 8 * par, (j >> 1) & 1);
      if (warp == 0 && lane == 0) trace(0, j);
      tc_fence_after();
      uint32_t sv[64];
      const uint32_t s_row = tmem + lane_off + C::S_COL + par * 128 + h * 64;
      tmem_ld32(s_row, &sv[0]);
      tmem_ld32(s_row + 32, &sv[32]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(ls_free + 8 * par);  // QK(j+2) may overwrite S[par]
      if (warp == 0 && lane == 0) trace(1, j);

      const int sb = sbits(j);
      if (CAUSAL && j == qi) {  // frontier step: key offset h*64 + c vs row r inside block i
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (h * 64 + c > r) sv[c] = __float_as_uint(-INFINITY);
      }
      if (!CAUSAL && (j + 1) * 128 > valid_len) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (j * 128 + h * 64 + c >= valid_len) sv[c] = __float_as_uint(-INFINITY);
      }
      float mh;
      {
        float a0 = fmax3(__uint_as_float(sv[0]), __uint_as_float(sv[1]), __uint_as_float(sv[2]));
        float a1 = fmax3(__uint_as_float(sv[3]), __uint_as_float(sv[4]), __uint_as_float(sv[5]));
        float a2 = fmax3(__uint_as_float(sv[6]), __uint_as_float(sv[7]), __uint_as_float(sv[8]));
        float a3 = fmax3(__uint_as_float(sv[9]), __uint_as_float(sv[10]), __uint_as_float(sv[11]));
#pragma unroll
        for (int c = 12; c < 60; c += 8) {
          a0 = fmax3(a0, __uint_as_float(sv[c]), __uint_as_float(sv[c + 1]));
          a1 = fmax3(a1, __uint_as_float(sv[c + 2]), __uint_as_float(sv[c + 3]));
          a2 = fmax3(a2, __uint_as_float(sv[c + 4]), __uint_as_float(sv[c + 5]));
          a3 = fmax3(a3, __uint_as_float(sv[c + 6]), __uint_as_float(sv[c + 7]));
        }
        a0 = fmax3(a0, __uint_as_float(sv[60]), __uint_as_float(sv[61]));
        a1 = fmax3(a1, __uint_as_float(sv[62]), __uint_as_float(sv[63]));
        mh = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3));
      }

      // ---- gate decision + the partner thread's half max, one barrier
      uint32_t bits;
      float mp = -INFINITY;  // partner's half max (valid when anything is kept)
      // shared words of a barrier are rewritten two barriers later: every warp
      // read them before arriving at the next one
      const int bp = int(nb & 1u);
      const uint32_t rm_mine = rmax_sm + ((bp * 2 + h) * 128 + r) * 4;
      const uint32_t rm_peer = rmax_sm + ((bp * 2 + (h ^ 1)) * 128 + r) * 4;
      if constexpr (GM == 0) {
        if (sb >= 0) {
          bits = uint32_t(sb);
          sts_f32(rm_mine, mh);
          named_bar_sync(1, 256);
          ++nb;
          mp = lds_f32(rm_peer);
        } else {
          // ThresholdGate: keep iff tile max (scaled) > T (gates.py:77-78)
          const uint32_t v = mh * scale > T ? (GT == 2 ? (1u << h) : 1u) : 0u;
          const uint32_t wv = __reduce_or_sync(0xffffffffu, v);
          if (lane == 0) sts_u32(vote_sm + (bp * 8 + warp) * 4, wv);
          sts_f32(rm_mine, mh);
          named_bar_sync(1, 256);
          ++nb;
          const uint4 w0 = lds_u128(vote_sm + bp * 32), w1 = lds_u128(vote_sm + bp * 32 + 16);
          bits = w0.x | w0.y | w0.z | w0.w | w1.x | w1.y | w1.z | w1.w;
          mp = lds_f32(rm_peer);
        }
      } else if constexpr (GM == 1) {
        bits = uint32_t(sb);
        if (bits) {
          sts_f32(rm_mine, mh);
          named_bar_sync(1, 256);
          ++nb;
          mp = lds_f32(rm_peer);
        }
      } else {
        sts_f32(rm_mine, mh);
        named_bar_sync(1, 256);
        ++nb;
        mp = lds_f32(rm_peer);
        if (sb >= 0) {
          bits = uint32_t(sb);
        } else {
          // RunningMaxGate (gates.py:101-118): gate tiles in key order, each judged
          // against the running max before it is merged
          const float mA = h == 0 ? mh : mp, mB = h == 0 ? mp : mh;
          if constexpr (GT == 2) {
            const uint32_t k0 = named_bar_red_or(2, 256, (mA - m_true) * scale >= lam ? 1u : 0u);
            const float mrun = k0 ? fmaxf(m_true, mA) : m_true;
            const uint32_t k1 = named_bar_red_or(2, 256, (mB - mrun) * scale >= lam ? 1u : 0u);
            bits = k0 | (k1 << 1);
          } else {
            bits = named_bar_red_or(2, 256, (fmaxf(mA, mB) - m_true) * scale >= lam ? 1u : 0u);
          }
        }
      }
      if (warp == 0 && lane == 0) trace(2, j);
      const float mA = h == 0 ? mh : mp, mB = h == 0 ? mp : mh;
      if constexpr (GM == 2) {
        if constexpr (GT == 2) {
          if (bits & 1u) m_true = fmaxf(m_true, mA);
          if (bits & 2u) m_true = fmaxf(m_true, mB);
        } else {
          if (bits) m_true = fmaxf(m_true, fmaxf(mA, mB));
        }
      }
      // ---- decisions out: the trace row, the V producers' rings, the MMA warp's masks
      if (warp == 0 && lane == 0) {
        kept_tiles += __popc(bits);
        if (drow) {
#pragma unroll
          for (int x = 0; x < GT; ++x)
            drow[j * GT + x] = j == qi ? int8_t(2) : (((bits >> x) & 1u) ? int8_t(3) : int8_t(1));
        }
        if (sb < 0) {
          const int di = int(dn % DQ);
          mbar_wait(dec_empty + 8 * di, ((dn / DQ) & 1) ^ 1);
          const uint32_t slot = dec_sm + (di * 2 + int(rank)) * 4;
          sts_u32(slot, bits);
          mbar_arrive(dec_full + 8 * di);
          const uint32_t pbar = other(dec_full + 8 * di);
          st_async_b32(other(slot), bits, pbar);
          mbar_arrive_expect_tx_cluster(pbar, 4);
          const uint32_t mslot = decm_sm + ((j & 3) * 2 + int(rank)) * 4;
          if (rank == 0)
            sts_u32(mslot, bits);
          else
            st_async_b32(lead(mslot), bits, lp_full + 8 * (j & 3));  // counted by this warp's arrival below
        }
      }
      if (sb < 0) ++dn;
      auto arrive_p = [&]() {
        __syncwarp();
        if (lane == 0) {
          if (rank == 1 && warp == 0 && sb < 0)
            mbar_arrive_expect_tx_cluster(lp_full + 8 * (j & 3), 4);
          else
            mbar_arrive_cluster(lp_full + 8 * (j & 3));
        }
      };
      if (bits == 0) {
        arrive_p();
        if (warp == 0 && lane == 0) {
          trace(3, j);
          trace(4, j);
        }
        continue;
      }

      float m_step;
      if constexpr (GT == 2)
        m_step = fmaxf((bits & 1u) ? mA : -INFINITY, (bits & 2u) ? mB : -INFINITY);
      else
        m_step = fmaxf(mA, mB);
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
      // lazy rescale (reference max moved by more than 2^8): O must be quiescent
      // -- PV(j-1) landed (rescale is decided identically by both threads of a row)
      if (__any_sync(0xffffffffu, rescale)) {
        if (j > 0) mbar_wait(pv_done + 8 * ((j - 1) & 1), ((j - 1) >> 1) & 1);
        tc_fence_after();
        const uint64_t ax2 = f2_pack(alpha, alpha);
#pragma unroll
        for (int c = 0; c < 64; c += 32) {
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
      }
      const bool kept_mine = GT == 2 ? ((bits >> h) & 1u) != 0 : true;
      float rsum = 0.f;
      if (kept_mine) {
        // P = exp2(s * scale*log2e - m * scale*log2e), bf16 pairs into P[par]
        // once PV(j-2) read it
        const float neg = (m_ref == -INFINITY) ? 0.f : -m_ref * sl2;
        const uint64_t sl2x2 = f2_pack(sl2, sl2);
        const uint64_t negx2 = f2_pack(neg, neg);
        uint64_t acc0 = 0, acc1 = 0;
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 64; c += 4) {
          const uint64_t x0 = ffma2(f2_pack(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])), sl2x2, negx2);
          const uint64_t x1 = ffma2(f2_pack(__uint_as_float(sv[c + 2]), __uint_as_float(sv[c + 3])), sl2x2, negx2);
          const float p0 = ex2_approx(f2_lo(x0)), p1 = ex2_approx(f2_hi(x0));
          const float p2 = ex2_approx(f2_lo(x1)), p3 = ex2_approx(f2_hi(x1));
          acc0 = fadd2(acc0, f2_pack(p0, p1));
          acc1 = fadd2(acc1, f2_pack(p2, p3));
          pk[c / 2] = pack_bf16x2(p0, p1);
          pk[c / 2 + 1] = pack_bf16x2(p2, p3);
        }
        if (warp == 0 && lane == 0) trace(3, j);
        if (j >= 2) mbar_wait(pv_done + 8 * par, ((j - 2) >> 1) & 1);
        tc_fence_after();
        tmem_st32(tmem + lane_off + C::P_COL + par * 64 + h * 32, pk);
        const uint64_t acc = fadd2(acc0, acc1);
        rsum = f2_lo(acc) + f2_hi(acc);
      }
      tmem_wait_st();
      tc_fence_before();
      arrive_p();
      if (warp == 0 && lane == 0) trace(4, j);
      l_sum = l_sum * alpha + rsum;
      o_valid = true;
    }

    // ---- epilogue: O = O~ / l, lse = m * scale + ln l (engine.py:178-182); the
    //      row sum is the two halves' sums
    sts_f32(lsum_sm + (h * 128 + r) * 4, l_sum);
    named_bar_sync(1, 256);
    const float l_tot = l_sum + lds_f32(lsum_sm + ((h ^ 1) * 128 + r) * 4);
    mbar_wait(o_full, 0);
    tc_fence_after();
    const float inv_l = 1.f / l_tot;
    bool bad = !(l_tot > 0.f);
    const int row = qi * 128 + r;
    const long long orow = (long long)b * p.o_sb + (long long)hq * p.o_sh + (long long)row * p.o_sn + h * 64;
#pragma unroll
    for (int c = 0; c < 64; c += 32) {
      uint32_t ov[32];
      tmem_ld32(o_row + c, ov);
      tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        float a0 = __uint_as_float(ov[e]) * inv_l, a1 = __uint_as_float(ov[e + 1]) * inv_l;
        if (p.inject_fault && qi == 0 && r == 0 && hq == 0 && h == 0 && c == 0 && e == 0) a0 += 1.0f;  // O[0][0] += 1
        bad |= !isfinite(a0) || !isfinite(a1);
        pk[e / 2] = pack_bf16x2(a0, a1);
      }
      store_o32(p, orow + c, pk);
    }
    if (h == 0) p.lse[((long long)b * p.heads_q + hq) * p.seq_len + row] = m_ref * scale + logf(l_tot);
    if (bad && p.status) atomicOr(p.status, 1);
    if (warp == 0 && lane == 0 && p.counters) {
      atomicAdd(&p.counters[0], (unsigned long long)nsteps * GT);
      atomicAdd(&p.counters[1], kept_tiles);
    }
    tc_fence_before();
    named_bar_arrive(15, C::NUM_THREADS);
  } else {
    setmaxnreg_dec<C::REG_OTHER>();
    named_bar_arrive(15, C::NUM_THREADS);
  }
  // every role but the MMA warp: the peer CTA may still signal this CTA's
  // barriers / write its shared memory until its own roles are done
  cluster_sync_all();
}

}  // namespace bsfa
