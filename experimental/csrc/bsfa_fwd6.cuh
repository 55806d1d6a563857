// BSFA forward (K1) for sm_100a, v6: one score buffer PER query tile, P written
// into the upper half of its own score buffer.
//
// One CTA owns two query tiles (128 rows each) that read the same K/V: two q
// heads of one GQA group at query block i, or -- odd groups, MHA -- query
// blocks 2m+1 and 2m of one q head (`block_pair`).  Keys stream in steps of
// 128 (one QK^T MMA tile) holding GT = 128 / b_n gate tiles of the reference
// (tiling.py:19-69).
//
// TMEM (512 columns): O_0, O_1 (fp32, D columns each), S_0, S_1 (fp32, 128
// columns each).  The softmax warps of tile s copy S_s into registers, vote,
// and write P_s (bf16 pairs, 64 columns) into columns 64..127 of S_s.  The
// MMA warp issues, per tile and step, PV_s(j) and then QK_s(j+1) into the same
// columns: the tensor pipe executes a thread's MMAs in issue order, so the QK
// overwrites P only after the PV read it.  Each tile's score chain
//   QK_s(j+1) -> tcgen05.ld -> vote [-> exp -> P] -> PV_s(j+1), QK_s(j+2)
// runs against the other tile's, so while one tile votes and exponentiates
// the pipe computes the other tile's QK and PV; an all-skipped step hands S
// back right after the vote (no exponentials, no PV).
//
// Tensor-pipe order (in-order), iteration j:
//   PV_0(j)  QK_0(j+1)  PV_1(j)  QK_1(j+1)
// s_full_s(j) is committed after QK_s(j), i.e. after every earlier MMA of the
// thread, so a softmax that saw it also knows PV_s(j-1) landed: O_s may be
// rescaled and P_s rewritten without a separate PV-done barrier.
//
// Shared memory: Q 2 x 128 rows x D, K ring of KC 64-column chunks (128 keys),
// V ring of VS units of 64 keys x D (one unit per kept 64-key half).
//
// Warp roles (384 threads):
//   warps 0-3 / 4-7  softmax of query tile 0 / 1, thread r owns row r (TMEM lane r)
//   warp 8           TMA: Q once, K chunks
//   warp 9           tcgen05 issuer (one elected lane) + TMEM owner
//   warp 10          TMA: V units, fetched only when some query tile kept them
//   warp 11          idle (completes the warpgroup for setmaxnreg)
// Per step and tile: QK = D/16 MMAs 128x128x16 (SS, K-major SW128); gate vote
// rowmax*scale > T OR-reduced over the 128 rows (gates.py:77-78); skipped gate
// tiles get no V TMA, no exponentials, no PV (engine.py:172-174); kept ones
// run the lazily rescaled online softmax (engine.py:57-68) and O_s += P_h V_h
// as 4 MMAs 128xDx16 (TS: P from TMEM, V MN-major SW128) per 64-key half.
#pragma once

#include "../../paper_2512_07011_b200/csrc/bsfa_common.cuh"

#ifndef BSFA_FWD6_KC
#define BSFA_FWD6_KC 0  // 0: default (4 chunks = 2 steps of K at D = 128)
#endif
#ifndef BSFA_FWD6_VS
#define BSFA_FWD6_VS 0
#endif
// ThresholdGate vote at b_n = 64: one barrier for both gate tiles of a step
// (warp REDUX + shared words); the V producer joins it and reads the vote
// words itself.  b_n = 128 and RunningMaxGate post decisions to a tagged ring.
#ifndef BSFA_VOTE1
#define BSFA_VOTE1 1
#endif
#ifndef BSFA_VOTE_PRODUCER
#define BSFA_VOTE_PRODUCER 1
#endif

namespace bsfa {

template <int D, int GT>
struct FCfg6 {
  static constexpr int BN = 128 / GT;           // gate tile width (reference b_n)
  static constexpr int NCH = D / 64;            // 64-column swizzle atoms along head_dim
  static constexpr int Q_TILE = 128 * D * 2;
  static constexpr int Q_ATOM = 128 * 128;      // 128 rows x 128 bytes
  static constexpr int K_CHUNK = 128 * 128;     // 128 keys x 64 columns, bf16
  static constexpr int V_UNIT = 64 * D * 2;     // 64 keys of V
  static constexpr int V_ATOM = 64 * 128;       // 64 keys x 64 columns
  static constexpr int KC = BSFA_FWD6_KC ? BSFA_FWD6_KC : 4;
  static constexpr int VS = BSFA_FWD6_VS ? BSFA_FWD6_VS : (D == 128 ? 6 : 8);
  static constexpr int DQ = 8;                  // decision ring depth (V producer)
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * Q_TILE;
  static constexpr int OFF_V = OFF_K + KC * K_CHUNK;
  static constexpr int OFF_BAR = OFF_V + VS * V_UNIT;
  // bar_q, k_full/empty[KC], v_full/empty[VS], s_full[2], p_full[2], o_full[2]
  static constexpr int NUM_BARS = 1 + 2 * KC + 2 * VS + 2 + 2 + 2;
  static constexpr int OFF_DEC = (OFF_BAR + NUM_BARS * 8 + 15) / 16 * 16;  // u32 [2][DQ] tagged decisions
  static constexpr int OFF_DECC = OFF_DEC + 2 * DQ * 4;                    // u32 [2] decisions consumed
  static constexpr int OFF_VOTE = (OFF_DECC + 2 * 4 + 15) / 16 * 16;      // u32 [2][2 parity][4 warps]
  static constexpr int OFF_TMEMPTR = OFF_VOTE + 2 * 2 * 4 * 4;
  static constexpr int SMEM_BYTES = OFF_TMEMPTR + 16 + 1024;  // + alignment slack
  static constexpr int O_COL = 0;          // O_s at s * D
  static constexpr int S_COL = 2 * D;      // S_s at S_COL + s * 128
  static constexpr int P_OFF = 64;         // P_s (bf16 pairs) at S_COL + s * 128 + P_OFF
  static constexpr int TMEM_COLS = 512;
  static constexpr int NUM_THREADS = 12 * 32;
  static constexpr int KPROD_WARP = 8, MMA_WARP = 9, VPROD_WARP = 10;
  static constexpr int REG_OTHER = 56;
  static constexpr int REG_LAUNCH = (65536 / NUM_THREADS) / 8 * 8;                       // 168
  static constexpr int REG_SOFT = (NUM_THREADS * REG_LAUNCH - 128 * REG_OTHER) / 256 / 8 * 8;  // 224
  static_assert(GT == 1 || GT == 2, "b_n in {64, 128}");
  static_assert(D == 64 || D == 128, "head_dim 64 or 128");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
  static_assert(S_COL + 256 <= TMEM_COLS, "TMEM budget");
  static_assert(KC >= NCH + 1 || KC >= 2, "K ring");
  static_assert(VS >= 2, "V ring must hold one step");
};

// GM: gate class -- 0 ThresholdGate (voted), 1 statically known steps (DenseGate,
// FrontierOnlyGate, SlidingWindowGate: no vote), 2 RunningMaxGate (voted).
template <int D, int GT, int GM, bool CAUSAL>
__global__ void __launch_bounds__(FCfg6<D, GT>::NUM_THREADS, 1)
    bsfa_fwd6_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const KernelParams p) {
  using C = FCfg6<D, GT>;
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
  const uint32_t s_full = v_empty + 8 * VS;    // [2]  QK_s(j) (and every earlier MMA) landed
  const uint32_t p_full = s_full + 16;         // [2]  tile s read S_s(j), decided, wrote P_s(j) (4 warps)
  const uint32_t o_full = p_full + 16;         // [2]  last PV_s landed
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
    if (p.block_pair) {
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
  constexpr bool VP = GM == 0 && GT == 2 && BSFA_VOTE1 && BSFA_VOTE_PRODUCER;
  // statically known decision bits of step j for query block qi (-1: voted)
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
      mbar_init(p_full + 8 * s, 4);
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
      mbar_arrive_expect_tx_w(bar_q, 2 * C::Q_TILE);
#pragma unroll
      for (int s = 0; s < 2; ++s)
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
          const int sbs = sbits(j, qi_a[s]);
          uint32_t w;
          if (sbs >= 0) {
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
  } else if (warp == C::MMA_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
    // ======================= tcgen05 issuer (warp-convergent, one elected lane) ========
    if (nsteps > 0) {
      constexpr uint32_t IDESC_QK = make_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t IDESC_PV = make_idesc_bf16(128, D, 0, 1);
      const uint64_t dq0 = make_sdesc_sw128(sQ, 16, 1024);
      const uint64_t dk0 = make_sdesc_sw128(sK, 16, 1024);
      const uint64_t dv0 = make_sdesc_sw128(sV, C::V_ATOM, 1024);
      mbar_wait(bar_q, 0);

      // QK_s(j) into S_s; tile 0 is the first reader of K(j) and waits for it
      auto issue_qk = [&](int s, int j) {
        const unsigned u0 = unsigned(j) * NCH;
        if (s == 0) {
          if (NCH == 2)
            mbar_wait2(k_full + 8 * int(u0 % KC), (u0 / KC) & 1, k_full + 8 * int((u0 + 1) % KC),
                       ((u0 + 1) / KC) & 1);
          else
            mbar_wait(k_full + 8 * int(u0 % KC), (u0 / KC) & 1);
        }
        if (lane == 0) trace(10, s, j);
        tc_fence_after();
        const int last = j < ns_a[1] ? 1 : 0;  // last reader of K(j)
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const unsigned u = u0 + c;
          const int slot = int(u % KC);
          umma_qk_chunk_w(tmem + C::S_COL + s * 128, dq0 + uint64_t((s * C::Q_TILE + c * C::Q_ATOM) >> 4),
                          dk0 + uint64_t((slot * C::K_CHUNK) >> 4), IDESC_QK, c > 0 ? 1u : 0u);
          if (s == last) umma_commit_w(k_empty + 8 * slot);
        }
        umma_commit_w(s_full + 8 * s);
        if (lane == 0) trace(5, s, j);
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
        const int sb = sbits(j, s ? qi_a[1] : qi_a[0]);
        tc_fence_after();
        if (lane == 0) trace(6, s, j);
        uint32_t bits;
        if (sb >= 0) {
          bits = uint32_t(sb);
        } else if constexpr (VP) {
          // the vote words of step j: rewritten only at step j + 2, whose vote
          // needs QK_s(j+2), issued after this decision is read
          const uint4 all = lds_u128(vote_sm + (s * 2 + (j & 1)) * 16);
          bits = all.x | all.y | all.z | all.w;
        } else {
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
      // part 2: per kept half, wait for its V unit and issue its MMAs (P_s from
      // the upper half of S_s)
      auto pv_mma = [&](int s, int j, uint32_t hb) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if ((hb >> hh) & 1u) {
            const unsigned uu = uidx[hh];
            mbar_wait(v_full + 8 * (uu % VS), (uu / VS) & 1);
            if (lane == 0) trace(11, s, j);
            tc_fence_after();
            umma_pv64_w(tmem + C::O_COL + s * D, tmem + C::S_COL + s * 128 + C::P_OFF + hh * 32,
                        dv0 + uint64_t(((uu % VS) * C::V_UNIT) >> 4), IDESC_PV, (o_started >> s) & 1u);
            o_started |= 1u << s;
          }
        }
        if (j == (s ? ns_a[1] : ns_a[0]) - 1) umma_commit_w(o_full + 8 * s);
        if (lane == 0) trace(7, s, j);
      };
      auto end_pv_step = [&]() {
        for (unsigned x = 0; x < nunits; ++x) umma_commit_w(v_empty + 8 * ((vbase + x) % VS));
        vbase += nunits;
        prev = 0;
        nunits = 0;
      };

      issue_qk(0, 0);
      if (ns_a[1] > 0) issue_qk(1, 0);
      for (int j = 0; j < nsteps; ++j) {
        mbar_wait(p_full, j & 1);
        pv_mma(0, j, pv_decide(0, j));
        if (j + 1 < ns_a[0]) issue_qk(0, j + 1);
        if (j < ns_a[1]) {
          mbar_wait(p_full + 8, j & 1);
          pv_mma(1, j, pv_decide(1, j));
          if (j + 1 < ns_a[1]) issue_qk(1, j + 1);
        }
        end_pv_step();
      }
      if (lane == 0 && p.counters) {
        atomicAdd(&p.counters[0], (unsigned long long)(ns_a[0] + ns_a[1]) * GT);
        atomicAdd(&p.counters[1], kept_m);
      }
    }
    __syncwarp();
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
    const uint32_t s_row = tmem + lane_off + C::S_COL + s * 128;   // this tile's scores
    const uint32_t p_row = s_row + C::P_OFF;                       // its P (bf16 pairs), aliasing S[64:128)
    const uint32_t o_row = tmem + lane_off + C::O_COL + s * D;
    const float sl2 = p.scale_log2;
    const float scale = p.scale;
    const float rescale_raw = p.rescale_raw;
    const int valid_len = p.valid_len;

    float T = 0.f;
    if constexpr (GM == 0) {
      const int pos = qi_s < p.thr_positions - 1 ? qi_s : p.thr_positions - 1;
      T = p.thr[(long long)hq * p.thr_positions + pos];  // thresholds.py:87
    }
    const float lam = p.gate_lambda;
    float m_true = -INFINITY;  // exact running row max (RunningMaxGate), raw units
    float m_ref = -INFINITY;   // raw reference max of this row over its kept tiles
    float l_sum = 0.f;         // row sum relative to m_ref
    bool o_valid = false;      // tile-uniform: O_s holds data
    unsigned dn = 0;
    int8_t* drow = p.decisions ? p.decisions + (((long long)b * p.heads_q + hq) * p.num_q_tiles + qi_s) * p.gate_cols
                               : nullptr;
    const uint32_t p_bar = p_full + 8 * s;

    for (int j = 0; j < nst; ++j) {
      // S_s(j) landed; so did every earlier MMA (PV_s(j-1) included): O_s is
      // quiescent and P_s may be rewritten
      mbar_wait(s_full + 8 * s, j & 1);
      if (r == 0) trace(0, s, j);
      tc_fence_after();
      uint32_t sv[128];
#pragma unroll
      for (int c = 0; c < 128; c += 32) tmem_ld32(s_row + c, &sv[c]);
      tmem_wait_ld();
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
      // row max per 64-key half (three-input FMNMX, four chains each)
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
      float mx[GT];
      if constexpr (GT == 2) {
        mx[0] = mh[0];
        mx[1] = mh[1];
      } else {
        mx[0] = fmaxf(mh[0], mh[1]);
      }
      if (BSFA_TRACE && r == 0) {
        asm volatile("" ::"f"(mx[0]));
        trace(8, s, j);
      }

      // ---- gate decision, OR over the tile's 128 rows
      uint32_t bits;
      if (GM == 1 || sb >= 0) {
        bits = uint32_t(sb);
      } else if constexpr (GM == 0) {
        // ThresholdGate: keep iff tile max (scaled) > T (gates.py:77-78)
        if constexpr (GT == 2 && BSFA_VOTE1) {
          // both gate tiles in ONE barrier: OR within the warp (REDUX), one word
          // per warp in shared memory (parity double-buffered: a warp reaches
          // step j+2's store only after every warp passed step j+1's barrier,
          // i.e. read step j's words), bar.sync, OR of the four words
          const uint32_t v = (mx[0] * scale > T ? 1u : 0u) | (mx[1] * scale > T ? 2u : 0u);
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
      if (r == 0) trace(2, s, j);
      if (bits == 0) {
        // S_s is free (our loads completed above): the next QK_s may overwrite it
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_bar);
        if (r == 0) {
          trace(3, s, j);
          trace(4, s, j);
        }
        continue;
      }
      const uint32_t hb = GT == 2 ? bits : 3u;

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
      // lazy rescale (reference max moved by more than 2^8); O_s is quiescent
      if (__any_sync(0xffffffffu, rescale)) {
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
      }

      // P = exp2(s * scale*log2e - m * scale*log2e) per 64-key half, bf16 pairs
      // into S_s[64:128) (TMEM lane r = row r, 32 columns per half)
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
              // part of the exponentials on the FMA pipe (relieves the MUFU queue)
              const uint64_t e1 = exp2_poly_x2(ffma2(f2_pack(p0, p1), 0ull, x1));
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
          tmem_st32(p_row + hh * 32, pk);
        }
        if (hh == 0 && r == 0) trace(3, s, j);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_bar);
      const uint64_t acc = fadd2(acc0, acc1);
      l_sum = l_sum * alpha + (f2_lo(acc) + f2_hi(acc));
      o_valid = true;
      if (r == 0) trace(4, s, j);
    }

    // ---- epilogue: O = O~ / l, lse = m * scale + ln l (engine.py:178-182)
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
