// BSFA forward (K1) for sm_100a, v3: one score buffer shared by the two query
// tiles, P in tensor memory.
//
// One CTA owns two query tiles (128 rows each) that read the same K/V: two q
// heads of one GQA group at query block i, or -- odd groups, MHA -- query
// blocks 2m+1 and 2m of one q head (`block_pair`).  Keys stream in steps of
// 128 (one QK^T MMA tile) holding GT = 128 / b_n gate tiles of the reference
// (tiling.py:19-69).
//
// TMEM (512 columns): O_0, O_1 (fp32, D columns each), ONE score buffer S
// (fp32, 128 columns) and P_0, P_1 (bf16, 64 columns each).  The softmax
// warps of a tile copy S into registers and release it at once (`s_free`),
// so the tensor core computes the other tile's scores while this tile votes,
// exponentiates and writes P_s; P never aliases S, so a tile's next QK never
// waits for its own exponentials (the chain S -> softmax -> PV -> next QK of
// a TMEM-aliased P is gone), and P stays in TMEM (tcgen05.st, TS-form PV:
// no shared-memory stores, no P reads from shared memory).
//
// Tensor-pipe order (in-order), iteration j:
//   QK_0(j+1)  PV_0(j)  QK_1(j+1)  PV_1(j)
// QK_1(j+1) waits until tile 0 has read S(j+1); while it waits the pipe runs
// PV_0(j), which hides the tcgen05.ld latency whenever tile 0 kept something.
// Every wait of the issuer is on an event the next item depends on anyway
// (tile 0 reads S(j+1) only after writing P_0(j)), so no tile blocks the other.
//
// Shared memory: Q 2 x 128 rows x D, K ring of KC 64-column chunks (128 keys),
// V ring of VS units of 64 keys x D (one unit per kept 64-key half).
//
// head_dim 256 (FCfg3::NQ = 1): one query tile per CTA, its O spanning both O
// slots (O 256 | S 128 | P 64 columns), tile 1 absent (qi = -1, as for the
// missing second block of an odd block pair).  b_m = 64 (BM): see the
// template comment below.
//
// Warp roles (384 threads):
//   warps 0-3 / 4-7  softmax of query tile 0 / 1, thread r owns row r (TMEM lane r)
//   warp 8           TMA: Q once, K chunks
//   warp 9           tcgen05 issuer (one elected lane) + TMEM owner
//   warp 10          TMA: V units, fetched only when some query tile kept them
//   warp 11          idle (completes the warpgroup for setmaxnreg)
// Per step and tile: QK = D/16 MMAs 128x128x16 (SS, K-major SW128); gate vote
// rowmax*scale > T OR-reduced over the 128 rows (gates.py:77-78: warp REDUX +
// shared vote words + a named barrier the V producer joins; RunningMaxGate:
// BAR.RED.OR per gate tile);
// skipped gate tiles get no V TMA, no exponentials, no PV (engine.py:172-174);
// kept ones run the lazily rescaled online softmax (engine.py:57-68) and
// O_s += P_h V_h as 4 MMAs 128xDx16 (TS: P from TMEM, V MN-major SW128) per
// 64-key half.
#pragma once

#include "bsfa_common.cuh"

#ifndef BSFA_FWD3_KC
#define BSFA_FWD3_KC 0  // 0: default per head_dim
#endif
#ifndef BSFA_FWD3_VS
#define BSFA_FWD3_VS 0
#endif
// 1: QKs issued by warp 9, PVs by warp 11 (each waits only on its own inputs;
// measured 20 % slower: PVs then queue behind QKs in the in-order tensor pipe);
// 0: one issuer in the order QK_0(j+1) PV_0(j) QK_1(j+1) PV_1(j)
// ThresholdGate vote at b_n = 64: 1 = one barrier for both gate tiles of a step
// (warp REDUX + shared words), 0 = one BAR.RED.OR per gate tile
// with BSFA_EXP_EMU: make each polynomial pair depend on the preceding MUFU pair
#ifndef BSFA_EXP_CHAIN
#define BSFA_EXP_CHAIN 1
#endif
#ifndef BSFA_PV_EVERY_PHASE
#define BSFA_PV_EVERY_PHASE 0
#endif
#ifndef BSFA_VOTE1
#define BSFA_VOTE1 1
#endif
// with BSFA_VOTE1 (ThresholdGate, b_n = 64): the V producer joins the vote
// barrier and reads the decision from the vote words itself (no decision ring)
#ifndef BSFA_VOTE_PRODUCER
#define BSFA_VOTE_PRODUCER 1
#endif
#ifndef BSFA_FWD3_SPLIT
#define BSFA_FWD3_SPLIT 0
#endif
// S release (softmax -> MMA warp) through a named barrier (bar.arrive by the
// tile's 128 threads, bar.sync by the issuer) instead of an mbarrier phase:
// 0 never, 1 always, 2 for the statically gated kernels (GM == 1: dense,
// frontier-only, sliding window), where it measured 2-4 % faster; the voted
// kernels measured 4-6 % slower with it
#ifndef BSFA_SFREE_NB
#define BSFA_SFREE_NB 2
#endif
// b_n = 128 ThresholdGate through the vote words + V producer in the barrier
// (as b_n = 64) instead of BAR.RED.OR + the decision ring: 128x128 BSFA 15 %
// faster at 32K, 10 % at 128K (profiles/r02_s3_ab_gt1vp.jsonl)
#ifndef BSFA_VOTE1_GT1
#define BSFA_VOTE1_GT1 1
#endif
#ifndef BSFA_MAXTREE
#define BSFA_MAXTREE 0
#endif
// the score row as one 32x32b.x128 tcgen05.ld (1) or four x32 loads (0)
#ifndef BSFA_LD128
#define BSFA_LD128 0
#endif

namespace bsfa {

// Ring depths per gate class (measured, profiles/r02_s3_ab_rings.jsonl): the
// voted kernels (GM 0 / 2) fetch V only after a vote, so a deeper K ring (6
// chunks = 3 steps) beats a deeper V ring (BSFA 1.1 % faster at 32K, 0.5 % at
// 128K); the statically gated ones (dense, frontier, window) prefetch V and
// keep the 6-unit V ring (dense 1.1-1.4 % faster with it).
// head_dim 256: ONE query tile per CTA whose O spans both O slots of the
// D = 128 layout (O 256 columns | S 128 | P 64 = 448 of 512), QK with K = 256
// and one N = 256 PV per 64-key unit; rings 6 K chunks (1.5 steps) + 2 V
// units (one step) so Q + K + V fit in 224 KB.
template <int D, int GT, int GM = 1>
struct FCfg3 {
  static constexpr int NQ = D == 256 ? 1 : 2;   // query tiles per CTA
  static constexpr int BN = 128 / GT;           // gate tile width (reference b_n)
  static constexpr int NCH = D / 64;            // 64-column swizzle atoms along head_dim
  static constexpr int Q_TILE = 128 * D * 2;
  static constexpr int Q_ATOM = 128 * 128;      // 128 rows x 128 bytes
  static constexpr int K_CHUNK = 128 * 128;     // 128 keys x 64 columns, bf16
  static constexpr int V_UNIT = 64 * D * 2;     // 64 keys of V
  static constexpr int V_ATOM = 64 * 128;       // 64 keys x 64 columns
  static constexpr int KC = BSFA_FWD3_KC ? BSFA_FWD3_KC : (D == 256 ? 6 : (GM == 1 ? 4 : 6));
  static constexpr int VS = BSFA_FWD3_VS ? BSFA_FWD3_VS : (D == 256 ? 2 : (D == 128 ? (GM == 1 ? 6 : 4) : 8));
  static constexpr int DQ = 8;                  // decision ring depth (V producer)
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + NQ * Q_TILE;
  static constexpr int OFF_V = OFF_K + KC * K_CHUNK;
  static constexpr int OFF_BAR = OFF_V + VS * V_UNIT;
  // bar_q, k_full/empty[KC], v_full/empty[VS], s_full[2], s_free,
  // p_full[2][2 parity], pv_done[2], o_full[2]
  static constexpr int NUM_BARS = 1 + 2 * KC + 2 * VS + 2 + 2 + 4 + 2 + 2;
  static constexpr int OFF_DEC = (OFF_BAR + NUM_BARS * 8 + 15) / 16 * 16;  // u32 [2][DQ] tagged decisions
  static constexpr int OFF_DECC = OFF_DEC + 2 * DQ * 4;                    // u32 [2] decisions consumed
  static constexpr int OFF_DECM = OFF_DECC + 2 * 4;                        // u32 [2][2 parity]
  static constexpr int OFF_VOTE = (OFF_DECM + 4 * 4 + 15) / 16 * 16;      // u32 [2][2 parity][4 warps]
  static constexpr int OFF_TMEMPTR = OFF_VOTE + 2 * 2 * 4 * 4;
  static constexpr int SMEM_BYTES = OFF_TMEMPTR + 16 + 1024;  // + alignment slack
  static constexpr int O_COL = 0;          // O_s at s * D
  static constexpr int S_COL = NQ * D;     // the shared score buffer
  static constexpr int P_COL = S_COL + 128;  // P_s (bf16 pairs) at P_COL + s * 64
  static constexpr int TMEM_COLS = 512;
  static constexpr int NUM_THREADS = 12 * 32;
  static constexpr int KPROD_WARP = 8, MMA_WARP = 9, VPROD_WARP = 10, PV_WARP = 11;
  static constexpr int REG_OTHER = 56;
  static constexpr int REG_LAUNCH = (65536 / NUM_THREADS) / 8 * 8;                       // 168
  static constexpr int REG_SOFT = (NUM_THREADS * REG_LAUNCH - 128 * REG_OTHER) / 256 / 8 * 8;  // 224
  static_assert(GT == 1 || GT == 2, "b_n in {64, 128}");
  static_assert(D == 64 || D == 128 || D == 256, "head_dim 64, 128 or 256");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
  static_assert(P_COL + 128 <= TMEM_COLS, "TMEM budget");
  static_assert(KC >= NCH + 1 || KC >= 2, "K ring");
  static_assert(VS >= 2, "V ring must hold one step");
};

// GM: gate class -- 0 ThresholdGate (voted), 1 statically known steps (DenseGate,
// FrontierOnlyGate, SlidingWindowGate: no vote), 2 RunningMaxGate (voted).  GM and
// CAUSAL are template parameters so the per-step softmax code carries no
// runtime gate/causality branches (smaller loop body, fewer taken branches).
// BM: the reference's query block b_m.  128: a query tile is one block.  64: a
// 128-row tile holds blocks 2t (rows 0-63, warps 0-1 of the tile) and 2t+1
// (rows 64-127, warps 2-3); each block has its own threshold, frontier and
// gate decisions (one vote word per warp, combined per block), a 64-key unit
// is fetched and multiplied when either block of either tile keeps it, and a
// block that skipped a unit the other block kept writes zeros into its P rows
// (its O, max and row sum are untouched).
template <int D, int GT, int GM, bool CAUSAL, int BM = 128>
__global__ void __launch_bounds__(FCfg3<D, GT, GM>::NUM_THREADS, 1)
    bsfa_fwd3_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const KernelParams p) {
  using C = FCfg3<D, GT, GM>;
  constexpr int KC = C::KC, VS = C::VS, DQ = C::DQ, NCH = C::NCH;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = opaque_u32((sraw + 1023u) & ~1023u);
  uint8_t* smem = smem_raw + (sbase - sraw);
  const uint32_t sQ = sbase + C::OFF_Q;
  const uint32_t sK = sbase + C::OFF_K;
  const uint32_t sV = sbase + C::OFF_V;
  const uint32_t bar_q = sbase + C::OFF_BAR;
  const uint32_t k_full = bar_q + 8;
  const uint32_t k_empty = k_full + 8 * KC;
  const uint32_t v_full = k_empty + 8 * KC;
  const uint32_t v_empty = v_full + 8 * VS;
  const uint32_t s_full = v_empty + 8 * VS;    // [2]  QK_s(j) landed in S
  const uint32_t s_free = s_full + 16;         // the tile that owned S copied it to registers (4 warps)
  const uint32_t p_full = s_free + 16;         // [2][2 parity]  P_s(j) written / step decided (4 warps)
  const uint32_t pv_done = p_full + 32;        // [2]  the PVs of tile s's last kept step landed
  const uint32_t o_full = pv_done + 16;        // [2]  last PV_s landed
  // decision hand-off to the V producer: tagged words ((n + 1) << 4 | bits) in a
  // DQ ring per tile, polled with volatile loads -- no mbarrier round trips on
  // the softmax's critical path; dec_cons[s] = decisions the producer consumed
  const uint32_t dec_sm = sbase + C::OFF_DEC;
  const uint32_t dec_cons = sbase + C::OFF_DECC;
  const uint32_t vote_sm = sbase + C::OFF_VOTE;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEMPTR);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- work unit (same order as the calibration kernel): (batch, kv head)
  //      major, heaviest query block first, head pairs of the group minor
  int qi_a[2], hq_a[2], ns_a[2];
  int b_, g_, qi_;
  {
    const int unit = blockIdx.x;
    if constexpr (C::NQ == 1) {
      // head_dim 256: one query tile per CTA, (batch, kv head) major, heaviest block first
      const int per_bg = p.num_q_tiles * p.group;
      const int bg = unit / per_bg;
      const int rem = unit - bg * per_bg;
      b_ = bg / p.heads_kv;
      g_ = bg - b_ * p.heads_kv;
      qi_ = p.num_q_tiles - 1 - rem / p.group;
      qi_a[0] = qi_;
      qi_a[1] = -1;  // no second tile
      hq_a[0] = hq_a[1] = g_ * p.group + rem % p.group;
    } else if (p.block_pair) {
      const int per_bg = ((p.num_q_tiles + 1) / 2) * p.group;
      const int bg = unit / per_bg;
      const int rem = unit - bg * per_bg;
      const int m = rem / p.group;
      b_ = bg / p.heads_kv;
      g_ = bg - b_ * p.heads_kv;
      qi_ = p.num_q_tiles - 1 - 2 * m;
      const int hq = g_ * p.group + (rem - m * p.group);
      qi_a[0] = qi_;
      qi_a[1] = qi_ - 1;  // -1: no second block (odd block count)
      hq_a[0] = hq_a[1] = hq;
    } else {
      const int pairs = p.group / 2;
      const int per_bg = p.num_q_tiles * pairs;
      const int bg = unit / per_bg;
      const int rem = unit - bg * per_bg;
      qi_ = p.num_q_tiles - 1 - rem / pairs;
      const int pr = rem - (rem / pairs) * pairs;
      b_ = bg / p.heads_kv;
      g_ = bg - b_ * p.heads_kv;
      qi_a[0] = qi_a[1] = qi_;
      hq_a[0] = g_ * p.group + 2 * pr;
      hq_a[1] = hq_a[0] + 1;
    }
  }
  const int b = b_, g = g_;
  constexpr bool causal = CAUSAL;
#pragma unroll
  for (int t = 0; t < 2; ++t) ns_a[t] = qi_a[t] < 0 ? 0 : (causal ? qi_a[t] + 1 : p.num_steps);
  const int nsteps = ns_a[0];  // tile 0 is never the shorter one
  const int gate_mode = p.gate_mode;
  const int window = p.gate_window;
  static_assert(BM == 128 || BM == 64, "b_m in {64, 128}");
  // b_m = 64: the reference grid is padded to lcm(64, b_n) <= 128, the kernel's
  // to 128; gate columns / query blocks past the reference grid are not counted
  constexpr int LCM = BM == 64 ? (GT == 1 ? 128 : 64) : 128;
  const int n_ref = (p.valid_len + LCM - 1) / LCM * LCM;
  const int kv_valid = n_ref / (128 / GT);
  const int q_valid = n_ref / BM;
  // b_m = 64: statics of both blocks of tile s at step j; the union of the two
  // blocks' keeps from the tile's four vote words
  auto bits64 = [&](int j, int qi, int hf) { return step_bits64<GT>(gate_mode, window, CAUSAL, j, 2 * qi + hf); };
  auto voted64 = [&](const StepBits64& a) { return a.reach & ~a.smask; };
  auto union64 = [&](const StepBits64& a0, const StepBits64& a1, const uint4 w) {
    return (a0.sval | (voted64(a0) & (w.x | w.y))) | (a1.sval | (voted64(a1) & (w.z | w.w)));
  };
  // statically known decision bits of step j for query block qi (-1: voted)
  // the V producer reads ThresholdGate decisions straight from the vote words
  // (BSFA_VOTE1_GT1 = 0: b_n = 128 keeps the BAR.RED.OR vote and the decision ring)
  constexpr bool VP = GM == 0 && (GT == 2 || BM == 64 || BSFA_VOTE1_GT1) && BSFA_VOTE1 && BSFA_VOTE_PRODUCER;
  constexpr bool SNB = !BSFA_FWD3_SPLIT && (BSFA_SFREE_NB == 1 || (BSFA_SFREE_NB == 2 && GM == 1));
  auto sbits = [&](int j, int qi) -> int {
    if constexpr (GM == 1) return step_static_bits<GT>(gate_mode, window, j, qi);
    return j == qi ? (1 << GT) - 1 : -1;  // frontier (tiling.py:50-60)
  };
  // debug timeline (-DBSFA_TRACE=1 builds only): clock64 per (event, tile, step) of one CTA
  const bool tr_cta = BSFA_TRACE && p.trace && (int)blockIdx.x == p.trace_cta;
  auto trace = [&](int ev, int s, int j) {
    if (BSFA_TRACE && tr_cta && j < kTraceSteps) p.trace[(ev * 2 + s) * kTraceSteps + j] = clock64();
  };

  // ---- setup
  if (warp == C::KPROD_WARP && lane == 0) {
    mbar_init(bar_q, 1);
    for (int i = 0; i < KC; ++i) {
      mbar_init(k_full + 8 * i, 1);
      mbar_init(k_empty + 8 * i, 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(v_full + 8 * i, 1);
      mbar_init(v_empty + 8 * i, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(s_full + 8 * s, 1);
      if (s == 0) mbar_init(s_free, 4);
      mbar_init(p_full + 16 * s, 4);
      mbar_init(p_full + 16 * s + 8, 4);
      mbar_init(pv_done + 8 * s, 1);
      mbar_init(o_full + 8 * s, 1);
    }
    fence_mbarrier_init();
  }
  if (warp == C::VPROD_WARP) {
    for (int i = lane; i < 2 * DQ + 2; i += 32) sts_u32(dec_sm + 4 * i, 0u);  // dec ring + dec_cons
  }
  if (warp == C::MMA_WARP) {
    tmem_alloc(tmem_ptr, C::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;
  if (threadIdx.x == 0) trace(12, 0, 0);  // (debug builds) CTA start, after setup

  if (warp == C::KPROD_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
    // ======================= TMA: Q once, K in 64-column chunks =======================
    if (nsteps > 0) {
      if (lane == 0) {
        tma_prefetch_desc(&tm_q);
        tma_prefetch_desc(&tm_k);
      }
      mbar_arrive_expect_tx_w(bar_q, C::NQ * C::Q_TILE);
#pragma unroll
      for (int s = 0; s < C::NQ; ++s)
#pragma unroll
        for (int c = 0; c < NCH; ++c)
          tma_load_4d_w(sQ + s * C::Q_TILE + c * C::Q_ATOM, &tm_q, bar_q, c * 64, (qi_a[s] < 0 ? 0 : qi_a[s]) * 128,
                        hq_a[s], b, kEvictFirst);
      unsigned u = 0;
      for (int j = 0; j < nsteps; ++j) {
#pragma unroll
        for (int c = 0; c < NCH; ++c, ++u) {
          const int slot = int(u % KC);
          mbar_wait(k_empty + 8 * slot, ((u / KC) & 1) ^ 1);
          mbar_arrive_expect_tx_w(k_full + 8 * slot, C::K_CHUNK);
          tma_load_4d_w(sK + slot * C::K_CHUNK, &tm_k, k_full + 8 * slot, c * 64, j * 128, g, b, kEvictLast);
        }
      }
    }
    __syncwarp();
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  } else if (warp == C::VPROD_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
    // ======================= TMA: V units kept by some query tile ======================
    if (nsteps > 0) {
      if (lane == 0) tma_prefetch_desc(&tm_v);
      unsigned vcount = 0;
      unsigned dn_a[2] = {0u, 0u};
      for (int j = 0; j < nsteps; ++j) {
        // tile 0's keeps as soon as its decision is known, then the units only
        // tile 1 keeps (the MMA warp numbers units in the same order)
        uint32_t prev = 0;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (j >= ns_a[s]) continue;
          const int sbs = BM == 64 ? 0 : sbits(j, qi_a[s]);
          uint32_t w;
          if constexpr (BM == 64) {
            const int qs = s ? qi_a[1] : qi_a[0];
            const StepBits64 a0 = bits64(j, qs, 0), a1 = bits64(j, qs, 1);
            if (GM == 1 || !(voted64(a0) | voted64(a1))) {
              w = a0.sval | a1.sval;
            } else if constexpr (VP) {
              named_bar_sync(1 + s, 160);
              w = union64(a0, a1, lds_u128(vote_sm + (s * 2 + int(dn_a[s] & 1u)) * 16));
              ++dn_a[s];  // (vote rounds of tile s)
            } else {
              const uint32_t slot_addr = dec_sm + (s * DQ + int(dn_a[s] % DQ)) * 4;
              const uint32_t tag = dn_a[s] + 1;
              uint32_t word = ld_volatile_u32(slot_addr);
              while ((word >> 4) != tag) word = ld_volatile_u32(slot_addr);
              w = word & 0xFu;
              ++dn_a[s];
              __syncwarp();
              if (lane == 0) st_volatile_u32(dec_cons + 4 * s, dn_a[s]);
            }
          } else if (sbs >= 0) {
            w = uint32_t(sbs);
          } else if constexpr (VP) {
            named_bar_sync(1 + s, 160);  // the tile's vote (128 softmax threads + this warp)
            const uint4 all = lds_u128(vote_sm + (s * 2 + (j & 1)) * 16);
            w = all.x | all.y | all.z | all.w;
            if (lane == 0) trace(13, s, j);
          } else {
            const uint32_t slot_addr = dec_sm + (s * DQ + int(dn_a[s] % DQ)) * 4;
            const uint32_t tag = dn_a[s] + 1;
            uint32_t word = ld_volatile_u32(slot_addr);
            while ((word >> 4) != tag) word = ld_volatile_u32(slot_addr);
            w = word & 0xFu;
            ++dn_a[s];
            __syncwarp();
            if (lane == 0) st_volatile_u32(dec_cons + 4 * s, dn_a[s]);
          }
          const uint32_t hb = GT == 2 ? w : (w ? 3u : 0u);  // 64-key halves kept
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            if (((hb & ~prev) >> hh) & 1u) {
              const int slot = int(vcount % VS);
              mbar_wait(v_empty + 8 * slot, ((vcount / VS) & 1) ^ 1);
              mbar_arrive_expect_tx_w(v_full + 8 * slot, C::V_UNIT);
#pragma unroll
              for (int c = 0; c < NCH; ++c)
                tma_load_4d_w(sV + slot * C::V_UNIT + c * C::V_ATOM, &tm_v, v_full + 8 * slot, c * 64,
                              j * 128 + hh * 64, g, b, kEvictLast);
              ++vcount;
              if (lane == 0) trace(14, s, j);
            }
          }
          prev |= hb;
        }
      }
      if (lane == 0 && p.counters) {
        // counters in gate tiles: a b_n = 128 gate tile is two 64-key units
        atomicAdd(&p.counters[2], (unsigned long long)(vcount / (3 - GT)));
        atomicAdd(&p.counters[3], (unsigned long long)nsteps * GT);
      }
    }
    __syncwarp();
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  } else if (warp == C::MMA_WARP || (BSFA_FWD3_SPLIT && warp == C::PV_WARP)) {
    setmaxnreg_dec<C::REG_OTHER>();
    // ======================= tcgen05 issuers (warp-convergent, one elected lane) ========
    // warp 9 issues the QKs (and owns TMEM), warp 11 the PVs: a QK is issued
    // as soon as S is free, never queued behind another tile's P hand-off
    const bool qk_role = warp == C::MMA_WARP;
    const bool pv_role = !BSFA_FWD3_SPLIT || warp == C::PV_WARP;
    if (nsteps > 0) {
      constexpr uint32_t IDESC_QK = make_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t IDESC_PV = make_idesc_bf16(128, D, 0, 1);
      const uint64_t dq0 = make_sdesc_sw128(sQ, 16, 1024);
      const uint64_t dk0 = make_sdesc_sw128(sK, 16, 1024);
      const uint64_t dv0 = make_sdesc_sw128(sV, C::V_ATOM, 1024);
      mbar_wait(bar_q, 0);

      // S is owned by one tile at a time: every QK after the first waits for
      // the previous owner's tcgen05.ld (one s_free phase per read, in order)
      uint32_t sfree_ph = 0;
      auto do_qk = [&](int s, int j) {
        const unsigned u0 = unsigned(j) * NCH;
        if (s != 0 || j != 0) ++sfree_ph;
        if (lane == 0) trace(10, s, j);
        tc_fence_after();
        const int last = j < ns_a[1] ? 1 : 0;  // last reader of K(j)
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const unsigned u = u0 + c;
          const int slot = int(u % KC);
          umma_qk_chunk_w(tmem + C::S_COL, dq0 + uint64_t((s * C::Q_TILE + c * C::Q_ATOM) >> 4),
                          dk0 + uint64_t((slot * C::K_CHUNK) >> 4), IDESC_QK, c > 0 ? 1u : 0u);
          if (s == last) umma_commit_w(k_empty + 8 * slot);
        }
        umma_commit_w(s_full + 8 * s);
        if (lane == 0) trace(5, s, j);
      };
      auto issue_qk = [&](int s, int j) {
        const unsigned u0 = unsigned(j) * NCH;
        const bool wait_s = s != 0 || j != 0;
        if (SNB) {
          // K(j) first (tile 0 is its first reader), then the S release
          if (s == 0)
            for (int c = 0; c < NCH; ++c) mbar_wait(k_full + 8 * int((u0 + c) % KC), ((u0 + c) / KC) & 1);
          if (wait_s) named_bar_sync(5, 160);
        } else if (s == 0) {
          // tile 0 is the first reader of K(j): S free + every chunk landed, tested together
          if (NCH == 2 && wait_s)
            mbar_wait3(s_free, sfree_ph & 1u, k_full + 8 * int(u0 % KC), (u0 / KC) & 1,
                       k_full + 8 * int((u0 + 1) % KC), ((u0 + 1) / KC) & 1);
          else if (NCH == 1 && wait_s)
            mbar_wait2(s_free, sfree_ph & 1u, k_full + 8 * int(u0 % KC), (u0 / KC) & 1);
          else {  // (head_dim 256: four chunks)
            if (wait_s) mbar_wait(s_free, sfree_ph & 1u);
            for (int c = 0; c < NCH; ++c) mbar_wait(k_full + 8 * int((u0 + c) % KC), ((u0 + c) / KC) & 1);
          }
        } else {
          mbar_wait(s_free, sfree_ph & 1u);
        }
        do_qk(s, j);
      };
      unsigned vbase = 0;      // V units consumed before this step
      unsigned nunits = 0;     // V units of the current step
      uint32_t prev = 0;       // 64-key halves of the current step already given a unit
      unsigned uidx[2] = {0u, 0u};
      uint32_t o_started = 0;  // bit s: O_s holds a partial sum
      unsigned dn_m[2] = {0u, 0u};                // voted decisions read, per tile
      unsigned long long kept_m = 0;              // processed gate tiles (counters[1])
      // PV_s(j), part 1 (after p_full): the tile's decision -> 64-key halves kept
      // and their V unit numbers (units numbered in the producer's fetch order)
      auto pv_decide = [&](int s, int j) -> uint32_t {
        const int sb = BM == 64 ? 0 : sbits(j, s ? qi_a[1] : qi_a[0]);  // (selects: s may be a runtime value)
        tc_fence_after();
        if (lane == 0) trace(6, s, j);
        uint32_t bits;
        if constexpr (BM == 64) {
          const int qs = s ? qi_a[1] : qi_a[0];
          const StepBits64 a0 = bits64(j, qs, 0), a1 = bits64(j, qs, 1);
          if (GM == 1 || !(voted64(a0) | voted64(a1))) {
            bits = a0.sval | a1.sval;
          } else if constexpr (VP) {
            const unsigned n = s ? dn_m[1] : dn_m[0];
            bits = union64(a0, a1, lds_u128(vote_sm + (s * 2 + int(n & 1u)) * 16));
            if (s) ++dn_m[1]; else ++dn_m[0];
          } else {
            const unsigned n = s ? dn_m[1] : dn_m[0];
            bits = ld_volatile_u32(dec_sm + (s * DQ + int(n % DQ)) * 4) & 0xFu;
            if (s) ++dn_m[1]; else ++dn_m[0];
          }
        } else if (sb >= 0) {
          bits = uint32_t(sb);
        } else if constexpr (VP) {
          // the vote words of step j: rewritten only at step j + 2, whose vote
          // needs QK_s(j+2), issued after this decision is read
          const uint4 all = lds_u128(vote_sm + (s * 2 + (j & 1)) * 16);
          bits = all.x | all.y | all.z | all.w;
        } else {
          // the tile's decision was posted to its tagged ring before its p_full
          // arrivals; the ring slot is reused only DQ voted steps later
          const unsigned n = s ? dn_m[1] : dn_m[0];
          bits = ld_volatile_u32(dec_sm + (s * DQ + int(n % DQ)) * 4) & 0xFu;
          if (s) ++dn_m[1]; else ++dn_m[0];
        }
        kept_m += __popc(bits);
        const uint32_t hb = GT == 2 ? bits : (bits ? 3u : 0u);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
          if (((hb & ~prev) >> hh) & 1u) uidx[hh] = vbase + nunits++;
        prev |= hb;
        return hb;
      };
      // part 2: per kept half, wait for its V unit and issue its MMAs; commits
      auto pv_mma = [&](int s, int j, uint32_t hb) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if ((hb >> hh) & 1u) {
            const unsigned uu = uidx[hh];
            mbar_wait(v_full + 8 * (uu % VS), (uu / VS) & 1);
            if (lane == 0) trace(11, s, j);
            tc_fence_after();
            umma_pv64_w(tmem + C::O_COL + s * D, tmem + C::P_COL + s * 64 + hh * 32,
                        dv0 + uint64_t(((uu % VS) * C::V_UNIT) >> 4), IDESC_PV, (o_started >> s) & 1u);
            o_started |= 1u << s;
          }
        }
        // P_s is free again once these PVs land.  Default: one pv_done phase per
        // step; the softmax waits only for the phase before a P write (a skipped
        // phase is provably complete by then: its commit precedes QK_s(j+1), whose
        // completion the softmax already waited for).  BSFA_PV_EVERY_PHASE: one
        // phase per step that issued PVs, each with a waiter (compute-sanitizer
        // synccheck reports skipped phases as "missing wait").
        if (!BSFA_PV_EVERY_PHASE || hb) umma_commit_w(pv_done + 8 * s);
        if (j == (s ? ns_a[1] : ns_a[0]) - 1) umma_commit_w(o_full + 8 * s);
        if (lane == 0) trace(7, s, j);
      };
      auto issue_pv = [&](int s, int j) {
        mbar_wait(p_full + 16 * s + 8 * (j & 1), (j >> 1) & 1);
        pv_mma(s, j, pv_decide(s, j));
      };
      auto end_pv_step = [&]() {
        for (unsigned x = 0; x < nunits; ++x) umma_commit_w(v_empty + 8 * ((vbase + x) % VS));
        vbase += nunits;
        prev = 0;
        nunits = 0;
      };

      if (qk_role) {
        issue_qk(0, 0);
        if (ns_a[1] > 0) issue_qk(1, 0);
      }
      for (int j = 0; j < nsteps; ++j) {
        if (qk_role && j + 1 < ns_a[0]) issue_qk(0, j + 1);
        if (pv_role) issue_pv(0, j);
        if (qk_role && j + 1 < ns_a[1]) issue_qk(1, j + 1);
        if (pv_role && j < ns_a[1]) issue_pv(1, j);
        if (pv_role) end_pv_step();
      }
      if (BM == 128 && pv_role && lane == 0 && p.counters) {  // (b_m = 64: counted per block by the softmax)
        atomicAdd(&p.counters[0], (unsigned long long)(ns_a[0] + ns_a[1]) * GT);
        atomicAdd(&p.counters[1], kept_m);
      }
    }
    __syncwarp();
    if (!qk_role) {
      named_bar_arrive(15, C::NUM_THREADS);
      return;
    }
    named_bar_sync(15, C::NUM_THREADS);
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
    return;
  } else if (warp < 8) {
    setmaxnreg_inc<C::REG_SOFT>();
    // ======================= softmax of query tile s =======================
    const int s = warp >> 2;
    const int wq = warp & 3;
    const int r = wq * 32 + lane;
    const int hq = s ? hq_a[1] : hq_a[0];  // (no dynamic indexing: keeps the arrays in registers)
    const int qi_s = s ? qi_a[1] : qi_a[0];
    const int nst = s ? ns_a[1] : ns_a[0];
    if (qi_s < 0) {  // a block pair's missing second block
      named_bar_arrive(15, C::NUM_THREADS);
      return;
    }
    const uint32_t lane_off = uint32_t(wq * 32) << 16;
    const uint32_t s_row = tmem + lane_off + C::S_COL;            // the shared score buffer
    const uint32_t p_row = tmem + lane_off + C::P_COL + s * 64;   // this tile's P (bf16 pairs)
    const uint32_t o_row = tmem + lane_off + C::O_COL + s * D;
    const float sl2 = p.scale_log2;
    const float scale = p.scale;
    const float rescale_raw = p.rescale_raw;
    const int valid_len = p.valid_len;

    // b_m = 64: this thread's query block (rows 0-63 / 64-127 of the tile)
    const int hf = BM == 64 ? (r >> 6) : 0;
    const int blk = BM == 64 ? 2 * qi_s + hf : qi_s;
    float T = 0.f;
    if constexpr (GM == 0) {
      const int pos = blk < p.thr_positions - 1 ? blk : p.thr_positions - 1;
      T = p.thr[(long long)hq * p.thr_positions + pos];  // thresholds.py:87
    }
    unsigned nb = 0;                          // b_m = 64: vote rounds of this tile
    unsigned long long reach_cnt = 0, kept_cnt = 0;  // b_m = 64: this block's counters
    const float lam = p.gate_lambda;
    float m_true = -INFINITY;  // exact running row max (RunningMaxGate), raw units
    float m_ref = -INFINITY;   // raw reference max of this row over its kept tiles
    float l_sum = 0.f;         // row sum relative to m_ref
    bool o_valid = false;      // tile-uniform: O_s holds data
    unsigned npv = 0;          // steps of this tile that issued PVs (pv_done phases)
    bool pv_pending = false;   // the last of them not yet waited on
    auto pv_wait = [&]() {
      if (pv_pending) {
        mbar_wait(pv_done + 8 * s, (npv - 1) & 1);
        pv_pending = false;
      }
    };
    unsigned dn = 0;
    int8_t* drow = p.decisions ? p.decisions + (((long long)b * p.heads_q + hq) * (p.num_q_tiles * (128 / BM)) + blk) *
                                                   p.gate_cols
                               : nullptr;

    for (int j = 0; j < nst; ++j) {
      if (!BSFA_PV_EVERY_PHASE) {  // default: phase j-1 (step j-1's commit) is the one to wait for
        npv = unsigned(j);
        pv_pending = j > 0;
      }
      mbar_wait(s_full + 8 * s, j & 1);
      if (r == 0) trace(0, s, j);
      tc_fence_after();
      uint32_t sv[128];
      if (BSFA_LD128) {
        tmem_ld128(s_row, sv);
      } else {
#pragma unroll
        for (int c = 0; c < 128; c += 32) tmem_ld32(s_row + c, &sv[c]);
      }
      tmem_wait_ld();
      tc_fence_before();
      if (SNB) {
        // the other tile's QK may overwrite S; no arrival after the CTA's last
        // S read (a named barrier has no phases to leave behind)
        if (s == 0 ? (j < ns_a[1] || j + 1 < ns_a[0]) : j + 1 < ns_a[0]) named_bar_arrive(5, 160);
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(s_free);  // the other tile's QK may overwrite S
      }
      if (r == 0) trace(1, s, j);

      const int sb = sbits(j, qi_s);
      if (CAUSAL && j == qi_s) {  // frontier step: key offset c vs row r inside block i
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (c > r) sv[c] = __float_as_uint(-INFINITY);
      }
      if (!CAUSAL && (j + 1) * 128 > valid_len) {
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (j * 128 + c >= valid_len) sv[c] = __float_as_uint(-INFINITY);
      }
      // row max per 64-key half (three-input FMNMX, four chains each; BSFA_MAXTREE:
      // a balanced ternary tree, 4 levels deep instead of 16)
      float mh[2];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const uint32_t* x = sv + hh * 64;
        if (BSFA_MAXTREE) {
          float l1[22];
#pragma unroll
          for (int t = 0; t < 21; ++t)
            l1[t] = fmax3(__uint_as_float(x[3 * t]), __uint_as_float(x[3 * t + 1]), __uint_as_float(x[3 * t + 2]));
          l1[21] = __uint_as_float(x[63]);
          float l2[8];
#pragma unroll
          for (int t = 0; t < 7; ++t) l2[t] = fmax3(l1[3 * t], l1[3 * t + 1], l1[3 * t + 2]);
          l2[7] = l1[21];
          const float l3a = fmax3(l2[0], l2[1], l2[2]), l3b = fmax3(l2[3], l2[4], l2[5]);
          mh[hh] = fmaxf(fmax3(l3a, l3b, l2[6]), l2[7]);
          continue;
        }
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
      float mx[GT];
      if constexpr (GT == 2) {
        mx[0] = mh[0];
        mx[1] = mh[1];
      } else {
        mx[0] = fmaxf(mh[0], mh[1]);
      }
      if (BSFA_TRACE && r == 0) {
        // keep the clock read after the maxima (a dependent no-op on them)
        asm volatile("" ::"f"(mx[0]));
        trace(8, s, j);
      }

      // ---- gate decision, OR over the tile's 128 rows in the barrier hardware
      uint32_t bits;   // this thread's query block's keeps (gate tiles of the step)
      uint32_t ubits;  // keeps of either block of the tile (b_m = 64; = bits otherwise)
      if constexpr (BM == 128) {
        if (GM == 1 || sb >= 0) {
          bits = uint32_t(sb);
        } else if constexpr (GM == 0) {
          // ThresholdGate: keep iff tile max (scaled) > T (gates.py:77-78)
          if constexpr ((GT == 2 || BSFA_VOTE1_GT1) && BSFA_VOTE1) {
            // both gate tiles in ONE barrier: OR within the warp (REDUX), one word
            // per warp in shared memory (parity double-buffered: a warp reaches
            // step j+2's store only after every warp passed step j+1's barrier,
            // i.e. read step j's words), bar.sync, OR of the four words
            uint32_t v = 0;
#pragma unroll
            for (int x = 0; x < GT; ++x) v |= (mx[x] * scale > T ? 1u : 0u) << x;
            const uint32_t wv = __reduce_or_sync(0xffffffffu, v);
            const uint32_t slot = vote_sm + (s * 2 + (j & 1)) * 16;
            if (lane == 0) sts_u32(slot + wq * 4, wv);
            named_bar_sync(1 + s, VP ? 160 : 128);
            const uint4 all = lds_u128(slot);
            bits = all.x | all.y | all.z | all.w;
          } else {
            bits = 0;
  #pragma unroll
            for (int x = 0; x < GT; ++x) bits |= named_bar_red_or(1 + s, 128, mx[x] * scale > T ? 1u : 0u) << x;
          }
        } else {
          // RunningMaxGate (gates.py:101-118): gate tiles in key order, each judged
          // against the running max before it is merged
          bits = 0;
          float mrun = m_true;
  #pragma unroll
          for (int x = 0; x < GT; ++x) {
            const uint32_t k = named_bar_red_or(1 + s, 128, (mx[x] - mrun) * scale >= lam ? 1u : 0u);
            bits |= k << x;
            if (k) mrun = fmaxf(mrun, mx[x]);
          }
        }
        if constexpr (GM == 2) {
  #pragma unroll
          for (int x = 0; x < GT; ++x)
            if ((bits >> x) & 1u) m_true = fmaxf(m_true, mx[x]);
        }
        if (BSFA_TRACE && r == 0) {
          asm volatile("" ::"r"(bits));
          trace(9, s, j);
        }
        // bookkeeping spread over the tile's warps (every thread holds `bits`), so
        // no single warp lags into the next vote
        if (GM != 1 && !VP && r == 64 && sb < 0) {
          // ring slot reuse: the producer consumed decision dn - DQ (it lags by a
          // few steps at most -- it gates the PVs -- so this never spins in practice)
          if (dn >= DQ)
            while (ld_volatile_u32(dec_cons + 4 * s) < dn - DQ + 1) {
            }
          st_volatile_u32(dec_sm + (s * DQ + int(dn % DQ)) * 4, ((dn + 1) << 4) | bits);
        }
        if (drow && r == 0) {
  #pragma unroll
          for (int x = 0; x < GT; ++x)
            drow[j * GT + x] = j == qi_s ? int8_t(2) : (((bits >> x) & 1u) ? int8_t(3) : int8_t(1));
        }
        if (GM != 1 && sb < 0) ++dn;
        ubits = bits;
      } else {
        // b_m = 64: statics per block; one vote round per gate class decision,
        // a word per warp (warps 0-1: block 2t, warps 2-3: block 2t+1)
        const StepBits64 a0 = bits64(j, qi_s, 0), a1 = bits64(j, qi_s, 1);
        const StepBits64 am = hf ? a1 : a0;
        const uint32_t v0 = voted64(a0), v1 = voted64(a1), vm = voted64(am);
        uint32_t b0 = a0.sval, b1 = a1.sval;
        const bool voted_step = GM != 1 && (v0 | v1) != 0;
        if constexpr (GM == 0) {
          if (voted_step) {
            uint32_t v = 0;
#pragma unroll
            for (int x = 0; x < GT; ++x)
              if (((vm >> x) & 1u) && mx[x] * scale > T) v |= 1u << x;  // gates.py:77-78
            const uint32_t wv = __reduce_or_sync(0xffffffffu, v);
            const uint32_t slot = vote_sm + (s * 2 + int(nb & 1u)) * 16;
            if (lane == 0) sts_u32(slot + wq * 4, wv);
            named_bar_sync(1 + s, VP ? 160 : 128);
            const uint4 all = lds_u128(slot);
            ++nb;
            b0 |= v0 & (all.x | all.y);
            b1 |= v1 & (all.z | all.w);
          }
        } else if constexpr (GM == 2) {
          // RunningMaxGate (gates.py:101-118): gate tiles in key order, each
          // judged against this row's running max before it is merged
          float mrun = m_true;
#pragma unroll
          for (int x = 0; x < GT; ++x) {
            if (((v0 | v1) >> x) & 1u) {
              const uint32_t pv = (((vm >> x) & 1u) && (mx[x] - mrun) * scale >= lam) ? (1u << x) : 0u;
              const uint32_t wv = __reduce_or_sync(0xffffffffu, pv);
              const uint32_t slot = vote_sm + (s * 2 + int(nb & 1u)) * 16;
              if (lane == 0) sts_u32(slot + wq * 4, wv);
              named_bar_sync(1 + s, 128);
              const uint4 all = lds_u128(slot);
              ++nb;
              b0 |= v0 & (all.x | all.y) & (1u << x);
              b1 |= v1 & (all.z | all.w) & (1u << x);
            }
            if ((((hf ? b1 : b0)) >> x) & 1u) mrun = fmaxf(mrun, mx[x]);
          }
        }
        bits = hf ? b1 : b0;
        ubits = b0 | b1;
        if constexpr (GM == 2) {
#pragma unroll
          for (int x = 0; x < GT; ++x)
            if ((bits >> x) & 1u) m_true = fmaxf(m_true, mx[x]);
        }
        if (GM != 1 && !VP && r == 64 && voted_step) {  // the union for the V producer and the MMA warp
          if (dn >= DQ)
            while (ld_volatile_u32(dec_cons + 4 * s) < dn - DQ + 1) {
            }
          st_volatile_u32(dec_sm + (s * DQ + int(dn % DQ)) * 4, ((dn + 1) << 4) | ubits);
        }
        if (voted_step) ++dn;
        if ((r & 63) == 0) {  // one thread per query block: trace row and counters
          if (drow) {
#pragma unroll
            for (int x = 0; x < GT; ++x)
              if ((am.reach >> x) & 1u)
                drow[j * GT + x] = ((am.front >> x) & 1u) ? int8_t(2) : (((bits >> x) & 1u) ? int8_t(3) : int8_t(1));
          }
          if (blk < q_valid) {  // the reference grid only
            const int cols = kv_valid - j * GT;
            const uint32_t cm = cols >= GT ? (1u << GT) - 1 : (cols > 0 ? (1u << cols) - 1 : 0u);
            reach_cnt += __popc(am.reach & cm);
            kept_cnt += __popc(bits & am.reach & cm);
          }
        }
      }
      if (r == 0) trace(2, s, j);
      const uint32_t p_bar = p_full + 16 * s + 8 * (j & 1);
      if (ubits == 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(p_bar);
        if (r == 0) {
          trace(3, s, j);
          trace(4, s, j);
        }
        continue;
      }
      const uint32_t hb = GT == 2 ? bits : (bits ? 3u : 0u);  // 64-key units this row keeps
      const uint32_t hbu = GT == 2 ? ubits : 3u;               // units the tile's PVs read (b_m = 64: either block)

      float m_step = -INFINITY;
#pragma unroll
      for (int x = 0; x < GT; ++x)
        if ((bits >> x) & 1u) m_step = fmaxf(m_step, mx[x]);
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
      // lazy rescale (reference max moved by more than 2^8): O_s must be
      // quiescent -- every PV_s up to step j-1 landed
      if (__any_sync(0xffffffffu, rescale)) {
        pv_wait();  // O_s quiescent
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
      }

      // P = exp2(s * scale*log2e - m * scale*log2e) per 64-key half, bf16 pairs
      // into P_s (TMEM lane r = row r, 32 columns per half)
      const float neg = (m_ref == -INFINITY) ? 0.f : -m_ref * sl2;
      const uint64_t sl2x2 = f2_pack(sl2, sl2);
      const uint64_t negx2 = f2_pack(neg, neg);
      uint64_t acc0 = 0, acc1 = 0;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const bool kept_h = ((hb >> hh) & 1u) != 0;
        if (kept_h) {
          uint32_t pk[32];
#pragma unroll
          for (int c = 0; c < 64; c += 4) {
            const int e = hh * 64 + c;
            const uint64_t x0 = ffma2(f2_pack(__uint_as_float(sv[e]), __uint_as_float(sv[e + 1])), sl2x2, negx2);
            const uint64_t x1 = ffma2(f2_pack(__uint_as_float(sv[e + 2]), __uint_as_float(sv[e + 3])), sl2x2, negx2);
            const float p0 = ex2_approx(f2_lo(x0)), p1 = ex2_approx(f2_hi(x0));
            float p2, p3;
            if (BSFA_EXP_EMU == 2 || (BSFA_EXP_EMU == 1 && ((c >> 2) & 1))) {
              // part of the exponentials on the FMA pipe (relieves the MUFU / MIO queue)
              const uint64_t e1 = exp2_poly_x2(BSFA_EXP_CHAIN ? ffma2(f2_pack(p0, p1), 0ull, x1) : x1);
              p2 = f2_lo(e1);
              p3 = f2_hi(e1);
            } else {
              p2 = ex2_approx(f2_lo(x1));
              p3 = ex2_approx(f2_hi(x1));
            }
            acc0 = fadd2(acc0, f2_pack(p0, p1));
            acc1 = fadd2(acc1, f2_pack(p2, p3));
            pk[c / 2] = pack_bf16x2(p0, p1);
            pk[c / 2 + 1] = pack_bf16x2(p2, p3);
          }
          pv_wait();  // the last PVs have read P_s
          tmem_st32(p_row + hh * 32, pk);
        } else if (BM == 64 && ((hbu >> hh) & 1u)) {
          // the other block of the tile kept this unit: zero rows for this block
          uint32_t z[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) z[c] = 0u;
          pv_wait();
          tmem_st32(p_row + hh * 32, z);
        }
        if (hh == 0 && r == 0) trace(3, s, j);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_bar);
      if (BSFA_PV_EVERY_PHASE) {  // this step issued PVs: one more pv_done phase
        ++npv;
        pv_pending = true;
      }
      const uint64_t acc = fadd2(acc0, acc1);
      l_sum = l_sum * alpha + (f2_lo(acc) + f2_hi(acc));
      if (BM == 128 || bits) o_valid = true;
      if (r == 0) trace(4, s, j);
    }

    // ---- epilogue: O = O~ / l, lse = m * scale + ln l (engine.py:178-182)
    if (BSFA_PV_EVERY_PHASE) pv_wait();  // (implied by o_full; gives the last phase a waiter)
    mbar_wait(o_full + 8 * s, 0);
    tc_fence_after();
    const float inv_l = 1.f / l_sum;
    bool bad = !(l_sum > 0.f);
    const int row = qi_s * 128 + r;
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
        if (p.inject_fault && qi_s == 0 && r == 0 && hq == 0 && c == 0 && e == 0) a0 += 1.0f;  // O[0][0] += 1
        bad |= !isfinite(a0) || !isfinite(a1);
        pk[e / 2] = pack_bf16x2(a0, a1);
      }
      store_o32(p, orow + c, pk);
    }
    p.lse[((long long)b * p.heads_q + hq) * p.seq_len + row] = m_ref * scale + logf(l_sum);
    if (r == 0) trace(12, 1, s);  // (debug builds) tile s's epilogue stores issued
    if (bad && p.status) atomicOr(p.status, 1);
    if (BM == 64 && (r & 63) == 0 && p.counters && (reach_cnt | kept_cnt)) {
      atomicAdd(&p.counters[0], reach_cnt);
      atomicAdd(&p.counters[1], kept_cnt);
    }
    tc_fence_before();
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  } else {
    setmaxnreg_dec<C::REG_OTHER>();
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  }
}

}  // namespace bsfa
