// BSFA forward (K1) for sm_100a, v4: one score buffer shared by the two query
// tiles, P in tensor memory, and each tile's softmax warps issue that tile's
// own PV MMAs.
//
// One CTA owns two query tiles (128 rows each) that read the same K/V: two q
// heads of one GQA group at query block i, or -- odd groups, MHA -- query
// blocks 2m+1 and 2m of one q head (`block_pair`).  Keys stream in steps of
// 128 (one QK^T MMA tile) holding GT = 128 / b_n gate tiles of the reference
// (tiling.py:19-69).
//
// TMEM (512 columns): O_0, O_1 (fp32, D columns each), ONE score buffer S
// (fp32, 128 columns) and P_0, P_1 (bf16 pairs, 64 columns each).  A tile's
// softmax warps copy S into registers and release it at once (`s_free`), so
// the tensor core computes the other tile's scores while this tile votes,
// exponentiates and writes P_s.  P never aliases S, so no QK waits for an
// exponential, and P stays in TMEM (tcgen05.st, TS-form PV).
//
// Issue: warp 9 issues only the QKs, strictly in the order QK_0(0) QK_1(0)
// QK_0(1) QK_1(1) ..., each as soon as the previous owner of S has read it.
// The PVs of tile s are issued by the tile's own warp 3 the moment its four
// warps have written P_s(j) (named-barrier hand-off, no mbarrier round trip):
// PV_s(j) therefore always enters the in-order tensor pipe before QK_{1-s}(j+1),
// which can only be issued after tile s read S(j+1), and no issuing warp ever
// serialises the two tiles' hand-offs (measured: the single issuer of v3 spent
// ~1000 cycles per step in mbarrier round trips on the S chain).
//
// V: each query tile has its own ring of VT units (64 keys x D), filled by its
// own TMA producer warp (10 + s) from that tile's decisions only, so a tile
// numbers its V units locally; a V gate tile is fetched iff the tile keeps it
// (engine.py:172-174: skipped tiles read no V).
//
// Warp roles (384 threads):
//   warps 4s..4s+3   softmax of query tile s, thread r owns row r (TMEM lane r);
//                    warp 4s+3 also issues PV_s and commits pv_done / v_empty / o_full
//   warp 8           TMA: Q once, K in 64-column chunks
//   warp 9           QK issuer (one elected lane) + TMEM owner
//   warps 10, 11     TMA: V units of query tile 0 / 1
// Per step and tile: QK = D/16 MMAs 128x128x16 (SS, K-major SW128); gate vote
// rowmax*scale > T OR-reduced over the 128 rows by BAR.RED.OR (gates.py:77-78);
// kept ones run the lazily rescaled online softmax (engine.py:57-68) and
// O_s += P_h V_h as 4 MMAs 128xDx16 (TS: P from TMEM, V MN-major SW128) per
// 64-key half.
#pragma once

#include "bsfa_kernel.cuh"

#ifndef BSFA_FWD4_KC
#define BSFA_FWD4_KC 0  // 0: default
#endif
#ifndef BSFA_FWD4_VT
#define BSFA_FWD4_VT 0
#endif

namespace bsfa {

template <int D, int GT>
struct FCfg4 {
  static constexpr int BN = 128 / GT;           // gate tile width (reference b_n)
  static constexpr int NCH = D / 64;            // 64-column swizzle atoms along head_dim
  static constexpr int Q_TILE = 128 * D * 2;
  static constexpr int Q_ATOM = 128 * 128;      // 128 rows x 128 bytes
  static constexpr int K_CHUNK = 128 * 128;     // 128 keys x 64 columns, bf16
  static constexpr int V_UNIT = 64 * D * 2;     // 64 keys of V
  static constexpr int V_ATOM = 64 * 128;       // 64 keys x 64 columns
  static constexpr int KC = BSFA_FWD4_KC ? BSFA_FWD4_KC : 4;
  static constexpr int VT = BSFA_FWD4_VT ? BSFA_FWD4_VT : (D == 128 ? 3 : 4);  // V units per query tile
  static constexpr int DQ = 8;                  // decision ring depth (V producers)
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * Q_TILE;
  static constexpr int OFF_V = OFF_K + KC * K_CHUNK;    // [2 tiles][VT units]
  static constexpr int OFF_BAR = OFF_V + 2 * VT * V_UNIT;
  // bar_q, k_full/empty[KC], v_full/empty[2][VT], s_full[2], s_free, pv_done[2], o_full[2]
  static constexpr int NUM_BARS = 1 + 2 * KC + 4 * VT + 2 + 1 + 2 + 2;
  static constexpr int OFF_DEC = (OFF_BAR + NUM_BARS * 8 + 15) / 16 * 16;  // u32 [2][DQ] tagged decisions
  static constexpr int OFF_DECC = OFF_DEC + 2 * DQ * 4;                    // u32 [2] decisions consumed
  static constexpr int OFF_TMEMPTR = OFF_DECC + 2 * 4;
  static constexpr int SMEM_BYTES = OFF_TMEMPTR + 16 + 1024;  // + alignment slack
  static constexpr int O_COL = 0;            // O_s at s * D
  static constexpr int S_COL = 2 * D;        // the shared score buffer
  static constexpr int P_COL = S_COL + 128;  // P_s (bf16 pairs) at P_COL + s * 64
  static constexpr int TMEM_COLS = 512;
  static constexpr int NUM_THREADS = 12 * 32;
  static constexpr int KPROD_WARP = 8, QK_WARP = 9, VPROD_WARP = 10;  // + tile
  static constexpr int REG_OTHER = 56;
  static constexpr int REG_LAUNCH = (65536 / NUM_THREADS) / 8 * 8;                            // 168
  static constexpr int REG_SOFT = (NUM_THREADS * REG_LAUNCH - 128 * REG_OTHER) / 256 / 8 * 8;  // 224
  static_assert(GT == 1 || GT == 2, "b_n in {64, 128}");
  static_assert(D == 64 || D == 128, "head_dim 64 or 128");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
  static_assert(P_COL + 128 <= TMEM_COLS, "TMEM budget");
  static_assert(KC >= 2, "K ring");
  static_assert(VT >= 2, "V ring must hold one step of a tile");
};

// GM: gate class -- 0 ThresholdGate (voted), 1 statically known steps (DenseGate,
// FrontierOnlyGate, SlidingWindowGate: no vote), 2 RunningMaxGate (voted).
template <int D, int GT, int GM, bool CAUSAL>
__global__ void __launch_bounds__(FCfg4<D, GT>::NUM_THREADS, 1)
    bsfa_fwd4_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const KernelParams p) {
  using C = FCfg4<D, GT>;
  constexpr int KC = C::KC, VT = C::VT, DQ = C::DQ, NCH = C::NCH;

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
  const uint32_t v_full = k_empty + 8 * KC;     // [2][VT]
  const uint32_t v_empty = v_full + 16 * VT;    // [2][VT]
  const uint32_t s_full = v_empty + 16 * VT;    // [2]  QK_s(j) landed in S
  const uint32_t s_free = s_full + 16;          // the tile that owned S copied it to registers (4 warps)
  const uint32_t pv_done = s_free + 8;          // [2]  the tile's last PV landed (one phase per PV step)
  const uint32_t o_full = pv_done + 16;         // [2]  every PV_s landed
  // decision hand-off to the V producers: tagged words ((n + 1) << 4 | bits) in a
  // DQ ring per tile, polled with volatile loads; dec_cons[s] = decisions consumed
  const uint32_t dec_sm = sbase + C::OFF_DEC;
  const uint32_t dec_cons = sbase + C::OFF_DECC;
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
#pragma unroll
  for (int t = 0; t < 2; ++t) ns_a[t] = qi_a[t] < 0 ? 0 : (CAUSAL ? qi_a[t] + 1 : p.num_steps);
  const int nsteps = ns_a[0];  // tile 0 is never the shorter one
  const int gate_mode = p.gate_mode;
  const int window = p.gate_window;
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
    for (int i = 0; i < 2 * VT; ++i) {
      mbar_init(v_full + 8 * i, 1);
      mbar_init(v_empty + 8 * i, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(s_full + 8 * s, 1);
      mbar_init(pv_done + 8 * s, 1);
      mbar_init(o_full + 8 * s, 1);
    }
    mbar_init(s_free, 4);
    fence_mbarrier_init();
  }
  if (warp == C::VPROD_WARP) {
    for (int i = lane; i < 2 * DQ + 2; i += 32) sts_u32(dec_sm + 4 * i, 0u);  // dec rings + dec_cons
  }
  if (warp == C::QK_WARP) {
    tmem_alloc(tmem_ptr, C::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;

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
  } else if (warp >= C::VPROD_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
    // ======================= TMA: V units this query tile kept ========================
    const int s = warp - C::VPROD_WARP;
    const int ns = s ? ns_a[1] : ns_a[0];
    const int qs = s ? qi_a[1] : qi_a[0];
    if (ns > 0) {
      if (lane == 0) tma_prefetch_desc(&tm_v);
      unsigned vcount = 0, dn = 0;
      const uint32_t vf = v_full + 8 * VT * s, ve = v_empty + 8 * VT * s;
      const uint32_t vbuf = sV + s * VT * C::V_UNIT;
      for (int j = 0; j < ns; ++j) {
        const int sb = sbits(j, qs);
        uint32_t w;
        if (sb >= 0) {
          w = uint32_t(sb);
        } else {
          const uint32_t slot_addr = dec_sm + (s * DQ + int(dn % DQ)) * 4;
          uint32_t word = ld_volatile_u32(slot_addr);
          while ((word >> 4) != dn + 1) word = ld_volatile_u32(slot_addr);
          w = word & 0xFu;
          ++dn;
          __syncwarp();
          if (lane == 0) st_volatile_u32(dec_cons + 4 * s, dn);
        }
        const uint32_t hb = GT == 2 ? w : (w ? 3u : 0u);  // 64-key halves kept
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if ((hb >> hh) & 1u) {
            const int slot = int(vcount % VT);
            mbar_wait(ve + 8 * slot, ((vcount / VT) & 1) ^ 1);
            mbar_arrive_expect_tx_w(vf + 8 * slot, C::V_UNIT);
#pragma unroll
            for (int c = 0; c < NCH; ++c)
              tma_load_4d_w(vbuf + slot * C::V_UNIT + c * C::V_ATOM, &tm_v, vf + 8 * slot, c * 64,
                            j * 128 + hh * 64, g, b, kEvictLast);
            ++vcount;
          }
        }
      }
      if (lane == 0 && p.counters) {
        // in gate tiles: a b_n = 128 gate tile is two 64-key units
        atomicAdd(&p.counters[2], (unsigned long long)(vcount / (3 - GT)));
        atomicAdd(&p.counters[3], (unsigned long long)ns * GT);
      }
    }
    __syncwarp();
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  } else if (warp == C::QK_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
    // ======================= QK issuer (warp-convergent, one elected lane) ============
    if (nsteps > 0) {
      constexpr uint32_t IDESC_QK = make_idesc_bf16(128, 128, 0, 0);
      const uint64_t dq0 = make_sdesc_sw128(sQ, 16, 1024);
      const uint64_t dk0 = make_sdesc_sw128(sK, 16, 1024);
      mbar_wait(bar_q, 0);
      // S is owned by one tile at a time: every QK after the first waits for
      // the previous owner's tcgen05.ld (one s_free phase per read, in order)
      uint32_t sfree_ph = 0;
      for (int j = 0; j < nsteps; ++j) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (j >= ns_a[s]) continue;
          const unsigned u0 = unsigned(j) * NCH;
          const bool wait_s = s != 0 || j != 0;
          if (s == 0) {  // the first reader of K(j): S free + every chunk landed, tested together
            if (NCH == 2 && wait_s)
              mbar_wait3(s_free, sfree_ph & 1u, k_full + 8 * int(u0 % KC), (u0 / KC) & 1,
                         k_full + 8 * int((u0 + 1) % KC), ((u0 + 1) / KC) & 1);
            else if (wait_s)
              mbar_wait2(s_free, sfree_ph & 1u, k_full + 8 * int(u0 % KC), (u0 / KC) & 1);
            else
              for (int c = 0; c < NCH; ++c) mbar_wait(k_full + 8 * int((u0 + c) % KC), ((u0 + c) / KC) & 1);
          } else {
            mbar_wait(s_free, sfree_ph & 1u);
          }
          if (wait_s) ++sfree_ph;
          if (lane == 0) trace(10, s, j);
          tc_fence_after();
          const int last = j < ns_a[1] ? 1 : 0;  // last reader of K(j)
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            const int slot = int((u0 + c) % KC);
            umma_qk_chunk_w(tmem + C::S_COL, dq0 + uint64_t((s * C::Q_TILE + c * C::Q_ATOM) >> 4),
                            dk0 + uint64_t((slot * C::K_CHUNK) >> 4), IDESC_QK, c > 0 ? 1u : 0u);
            if (s == last) umma_commit_w(k_empty + 8 * slot);
          }
          umma_commit_w(s_full + 8 * s);
          if (lane == 0) trace(5, s, j);
        }
      }
    }
    __syncwarp();
    named_bar_sync(15, C::NUM_THREADS);
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
    return;
  } else {
    setmaxnreg_inc<C::REG_SOFT>();
    // ======================= softmax of query tile s (+ its PVs) ===================
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
    const bool pv_warp = wq == 3;  // issues this tile's PV MMAs
    const uint32_t lane_off = uint32_t(wq * 32) << 16;
    const uint32_t s_row = tmem + lane_off + C::S_COL;            // the shared score buffer
    const uint32_t p_row = tmem + lane_off + C::P_COL + s * 64;   // this tile's P (bf16 pairs)
    const uint32_t o_row = tmem + lane_off + C::O_COL + s * D;
    const float sl2 = p.scale_log2;
    const float scale = p.scale;
    const float rescale_raw = p.rescale_raw;
    const int valid_len = p.valid_len;
    constexpr uint32_t IDESC_PV = make_idesc_bf16(128, D, 0, 1);
    const uint64_t dv0 = make_sdesc_sw128(sV + s * VT * C::V_UNIT, C::V_ATOM, 1024);
    const uint32_t vf = v_full + 8 * VT * s, ve = v_empty + 8 * VT * s;

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
    unsigned dn = 0;           // voted decisions posted
    unsigned vcount = 0;       // V units this tile consumed (its producer's order)
    unsigned npv = 0;          // steps that issued PVs (pv_done phases)
    bool pv_pending = false;   // the last PV step has not been waited on yet
    unsigned long long kept_tiles = 0;
    int8_t* drow = p.decisions ? p.decisions + (((long long)b * p.heads_q + hq) * p.num_q_tiles + qi_s) * p.gate_cols
                               : nullptr;

    for (int j = 0; j < nst; ++j) {
      mbar_wait(s_full + 8 * s, j & 1);
      if (r == 0) trace(0, s, j);
      tc_fence_after();
      uint32_t sv[128];
#pragma unroll
      for (int c = 0; c < 128; c += 32) tmem_ld32(s_row + c, &sv[c]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_free);  // the other tile's QK may overwrite S
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
        asm volatile("" ::"f"(mx[0]));  // keep the clock read after the maxima
        trace(8, s, j);
      }

      // ---- gate decision, OR over the tile's 128 rows in the barrier hardware
      uint32_t bits;
      if (GM == 1 || sb >= 0) {
        bits = uint32_t(sb);
      } else if constexpr (GM == 0) {
        // ThresholdGate: keep iff tile max (scaled) > T (gates.py:77-78)
        bits = 0;
#pragma unroll
        for (int x = 0; x < GT; ++x) bits |= named_bar_red_or(1 + s, 128, mx[x] * scale > T ? 1u : 0u) << x;
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
      // bookkeeping spread over the tile's warps (every thread holds `bits`)
      if (GM != 1 && r == 64 && sb < 0) {
        // ring slot reuse: the producer consumed decision dn - DQ (it lags by a
        // few steps at most -- it gates this tile's PVs -- so this never spins)
        if (dn >= DQ)
          while (ld_volatile_u32(dec_cons + 4 * s) < dn - DQ + 1) {
          }
        st_volatile_u32(dec_sm + (s * DQ + int(dn % DQ)) * 4, ((dn + 1) << 4) | bits);
      }
      if (r == 96) kept_tiles += __popc(bits);
      if (drow && r == 0) {
#pragma unroll
        for (int x = 0; x < GT; ++x)
          drow[j * GT + x] = j == qi_s ? int8_t(2) : (((bits >> x) & 1u) ? int8_t(3) : int8_t(1));
      }
      if (GM != 1 && sb < 0) ++dn;
      if (r == 0) trace(2, s, j);
      if (bits == 0) {
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
      // the tile's last PVs must have landed before O_s is rescaled or P_s rewritten
      auto pv_wait = [&]() {
        if (pv_pending) {
          mbar_wait(pv_done + 8 * s, (npv - 1) & 1);
          pv_pending = false;
        }
      };
      // lazy rescale (reference max moved by more than 2^8)
      if (__any_sync(0xffffffffu, rescale)) {
        pv_wait();
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
      }

      // P = exp2(s * scale*log2e - m * scale*log2e) per 64-key half, bf16 pairs
      // into P_s (TMEM lane r = row r, 32 columns per half)
      const float neg = (m_ref == -INFINITY) ? 0.f : -m_ref * sl2;
      const uint64_t sl2x2 = f2_pack(sl2, sl2);
      const uint64_t negx2 = f2_pack(neg, neg);
      uint64_t acc0 = 0, acc1 = 0;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        if ((hb >> hh) & 1u) {
          uint32_t pk[32];
#pragma unroll
          for (int c = 0; c < 64; c += 4) {
            const int e = hh * 64 + c;
            const uint64_t x0 = ffma2(f2_pack(__uint_as_float(sv[e]), __uint_as_float(sv[e + 1])), sl2x2, negx2);
            const uint64_t x1 = ffma2(f2_pack(__uint_as_float(sv[e + 2]), __uint_as_float(sv[e + 3])), sl2x2, negx2);
            const float p0 = ex2_approx(f2_lo(x0)), p1 = ex2_approx(f2_hi(x0));
            float p2, p3;
            if (BSFA_EXP_EMU == 2 || (BSFA_EXP_EMU == 1 && ((c >> 2) & 1))) {
              // part of the exponentials on the FMA pipe (relieves the MUFU)
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
          pv_wait();  // the previous PVs of this tile have read P_s
          tmem_st32(p_row + hh * 32, pk);
        }
        if (hh == 0 && r == 0) trace(3, s, j);
      }
      tmem_wait_st();
      tc_fence_before();
      // ---- hand P_s(j) to this tile's PV warp: warps 0-2 arrive, warp 3 waits
      if (!pv_warp) {
        named_bar_arrive(5 + s, 128);
      } else {
        named_bar_sync(5 + s, 128);
        tc_fence_after();
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if ((hb >> hh) & 1u) {
            const unsigned slot = vcount % VT;
            mbar_wait(vf + 8 * slot, (vcount / VT) & 1);
            tc_fence_after();
            umma_pv64_w(tmem + C::O_COL + s * D, tmem + C::P_COL + s * 64 + hh * 32,
                        dv0 + uint64_t((slot * C::V_UNIT) >> 4), IDESC_PV, o_valid || hh == 1 && (hb & 1u) ? 1u : 0u);
            umma_commit_w(ve + 8 * slot);  // the unit is free once this PV landed
            ++vcount;
          }
        }
        umma_commit_w(pv_done + 8 * s);
        if (lane == 0) trace(7, s, j);
      }
      ++npv;
      pv_pending = true;
      const uint64_t acc = fadd2(acc0, acc1);
      l_sum = l_sum * alpha + (f2_lo(acc) + f2_hi(acc));
      o_valid = true;
      if (r == 0) trace(4, s, j);
    }
    // every PV of this tile landed -> epilogue (one commit covers the warp's MMAs)
    if (pv_warp) umma_commit_w(o_full + 8 * s);

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
    if (bad && p.status) atomicOr(p.status, 1);
    if (r == 96 && p.counters) {
      atomicAdd(&p.counters[0], (unsigned long long)nst * GT);
      atomicAdd(&p.counters[1], kept_tiles);
    }
    tc_fence_before();
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  }
}

}  // namespace bsfa
