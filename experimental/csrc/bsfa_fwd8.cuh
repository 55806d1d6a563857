// BSFA forward (K1) for sm_100a, v8 (experimental): 64-key steps, one 64-column
// score buffer PER query tile and double-buffered P, ThresholdGate at
// 128x64 tiles only.
//
// TMEM (2D + 256 <= 512 columns): O_0, O_1 (fp32, D each), S_0, S_1 (fp32, 64
// columns: one gate tile of scores), P_s[2] (bf16 pairs, 32 columns each).
// A step is one 64-key gate tile (tiling.py:19-69).  A tile's next QK waits
// only for its OWN softmax to copy S_s into registers -- never for the other
// tile, its exponentials or a PV -- so each tile's chain is
//   QK_s(j) -> tcgen05.ld -> s_free_s -> QK_s(j+1)
// and the two tiles' chains run side by side.  The price: QK MMAs at N = 64,
// which read Q from shared memory twice as often (2/3 of the MMA rate in
// isolation, tools/microbench/mma_modes.cu).
//
// Issue order (one thread): iteration j: QK_0(j+1) QK_1(j+1) PV_0(j-1) PV_1(j-1)
// -- the PVs trail a step so their V units (requested after the vote) have
// landed.  P_s[j&1] is rewritten at step j+2 only after pv_done_s says PV_s(j)
// read it, an O rescale at step j waits for PV_s(j-1): pv_done per step
// parity, so a waited phase is never more than one behind or ahead.  Vote words and
// p_full are 4-deep rings: a tile's softmax can be up to two steps ahead of
// the issuer's PV reads.
#pragma once

#include "../../paper_2512_07011_b200/csrc/bsfa_common.cuh"

namespace bsfa {

template <int D>
struct FCfg8 {
  static constexpr int NCH = D / 64;
  static constexpr int Q_TILE = 128 * D * 2;
  static constexpr int Q_ATOM = 128 * 128;
  static constexpr int K_STEP = 64 * D * 2;  // 64 keys, NCH atoms of 64 rows x 128 B
  static constexpr int K_ATOM = 64 * 128;
  static constexpr int V_UNIT = 64 * D * 2;
  static constexpr int V_ATOM = 64 * 128;
  static constexpr int KS = D == 128 ? 4 : 8;
  static constexpr int VS = D == 128 ? 6 : 8;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * Q_TILE;
  static constexpr int OFF_V = OFF_K + KS * K_STEP;
  static constexpr int OFF_BAR = OFF_V + VS * V_UNIT;
  // bar_q, k_full/empty[KS], v_full/empty[VS], s_full[2], s_free[2], p_full[2][4], pv_done[2][2], o_full[2]
  static constexpr int NUM_BARS = 1 + 2 * KS + 2 * VS + 2 + 2 + 8 + 4 + 2;
  static constexpr int OFF_VOTE = (OFF_BAR + NUM_BARS * 8 + 15) / 16 * 16;  // u32 [2 tiles][4][4 warps]
  static constexpr int OFF_TMEMPTR = OFF_VOTE + 2 * 4 * 4 * 4;
  static constexpr int SMEM_BYTES = OFF_TMEMPTR + 16 + 1024;
  static constexpr int O_COL = 0, S_COL = 2 * D, P_COL = 2 * D + 128;
  static constexpr int TMEM_COLS = 512;
  static constexpr int NUM_THREADS = 12 * 32;
  static constexpr int KPROD_WARP = 8, MMA_WARP = 9, VPROD_WARP = 10;
  static constexpr int REG_OTHER = 56;
  static constexpr int REG_LAUNCH = (65536 / NUM_THREADS) / 8 * 8;
  static constexpr int REG_SOFT = (NUM_THREADS * REG_LAUNCH - 128 * REG_OTHER) / 256 / 8 * 8;
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
  static_assert(P_COL + 128 <= TMEM_COLS, "TMEM budget");
};

template <int D, bool CAUSAL>
__global__ void __launch_bounds__(FCfg8<D>::NUM_THREADS, 1)
    bsfa_fwd8_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const KernelParams p) {
  using C = FCfg8<D>;
  constexpr int KS = C::KS, VS = C::VS, NCH = C::NCH;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = opaque_u32((sraw + 1023u) & ~1023u);
  uint8_t* smem = smem_raw + (sbase - sraw);
  const uint32_t sQ = sbase + C::OFF_Q;
  const uint32_t sK = sbase + C::OFF_K;
  const uint32_t sV = sbase + C::OFF_V;
  const uint32_t bar_q = sbase + C::OFF_BAR;
  const uint32_t k_full = bar_q + 8;
  const uint32_t k_empty = k_full + 8 * KS;
  const uint32_t v_full = k_empty + 8 * KS;
  const uint32_t v_empty = v_full + 8 * VS;
  const uint32_t s_full = v_empty + 8 * VS;  // [2]
  const uint32_t s_free = s_full + 16;       // [2]  (4 warps of the tile)
  const uint32_t p_full = s_free + 16;       // [2][4]  (4 warps)
  const uint32_t pv_done = p_full + 64;      // [2][2 step parity]
  const uint32_t o_full = pv_done + 32;      // [2]
  const uint32_t vote_sm = sbase + C::OFF_VOTE;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEMPTR);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- work unit: the v3 order (head pairs, or query-block pairs for odd groups)
  int qi_a[2], hq_a[2], ns_a[2];
  int b_, g_;
  {
    const int unit = blockIdx.x;
    if (p.block_pair) {
      const int per_bg = ((p.num_q_tiles + 1) / 2) * p.group;
      const int bg = unit / per_bg;
      const int rem = unit - bg * per_bg;
      const int m = rem / p.group;
      b_ = bg / p.heads_kv;
      g_ = bg - b_ * p.heads_kv;
      const int qi = p.num_q_tiles - 1 - 2 * m;
      qi_a[0] = qi;
      qi_a[1] = qi - 1;
      hq_a[0] = hq_a[1] = g_ * p.group + (rem - m * p.group);
    } else {
      const int pairs = p.group / 2;
      const int per_bg = p.num_q_tiles * pairs;
      const int bg = unit / per_bg;
      const int rem = unit - bg * per_bg;
      const int qi = p.num_q_tiles - 1 - rem / pairs;
      const int pr = rem - (rem / pairs) * pairs;
      b_ = bg / p.heads_kv;
      g_ = bg - b_ * p.heads_kv;
      qi_a[0] = qi_a[1] = qi;
      hq_a[0] = g_ * p.group + 2 * pr;
      hq_a[1] = hq_a[0] + 1;
    }
  }
  const int b = b_, g = g_;
  // 64-key steps: causal query tile i reaches key blocks 0 .. 2i+1 (frontier 2i, 2i+1)
#pragma unroll
  for (int t = 0; t < 2; ++t) ns_a[t] = qi_a[t] < 0 ? 0 : (CAUSAL ? 2 * qi_a[t] + 2 : 2 * p.num_steps);
  const int nsteps = ns_a[0];
  auto frontier = [&](int j, int qi) { return (j >> 1) == qi; };  // tiling.py:50-60

  if (warp == C::KPROD_WARP && lane == 0) {
    mbar_init(bar_q, 1);
    for (int i = 0; i < KS; ++i) {
      mbar_init(k_full + 8 * i, 1);
      mbar_init(k_empty + 8 * i, 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(v_full + 8 * i, 1);
      mbar_init(v_empty + 8 * i, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(s_full + 8 * s, 1);
      mbar_init(s_free + 8 * s, 4);
      for (int x = 0; x < 4; ++x) mbar_init(p_full + 32 * s + 8 * x, 4);
      mbar_init(pv_done + 16 * s, 1);
      mbar_init(pv_done + 16 * s + 8, 1);
      mbar_init(o_full + 8 * s, 1);
    }
    fence_mbarrier_init();
  }
  if (warp == C::MMA_WARP) {
    tmem_alloc(tmem_ptr, C::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;

  if (warp == C::KPROD_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
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
      for (int j = 0; j < nsteps; ++j) {
        const int st = j % KS;
        mbar_wait(k_empty + 8 * st, ((j / KS) & 1) ^ 1);
        mbar_arrive_expect_tx_w(k_full + 8 * st, C::K_STEP);
#pragma unroll
        for (int c = 0; c < NCH; ++c)
          tma_load_4d_w(sK + st * C::K_STEP + c * C::K_ATOM, &tm_k, k_full + 8 * st, c * 64, j * 64, g, b,
                        kEvictLast);
      }
    }
    __syncwarp();
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  } else if (warp == C::VPROD_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
    if (nsteps > 0) {
      if (lane == 0) tma_prefetch_desc(&tm_v);
      unsigned vcount = 0;
      for (int j = 0; j < nsteps; ++j) {
        uint32_t any = 0;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (j >= ns_a[s]) continue;
          if (frontier(j, s ? qi_a[1] : qi_a[0])) {
            any = 1;
          } else {
            named_bar_sync(1 + s, 160);  // the tile's vote (128 softmax threads + this warp)
            const uint4 w = lds_u128(vote_sm + (s * 4 + (j & 3)) * 16);
            any |= w.x | w.y | w.z | w.w;
          }
        }
        if (any) {
          const int slot = int(vcount % VS);
          mbar_wait(v_empty + 8 * slot, ((vcount / VS) & 1) ^ 1);
          mbar_arrive_expect_tx_w(v_full + 8 * slot, C::V_UNIT);
#pragma unroll
          for (int c = 0; c < NCH; ++c)
            tma_load_4d_w(sV + slot * C::V_UNIT + c * C::V_ATOM, &tm_v, v_full + 8 * slot, c * 64, j * 64, g, b,
                          kEvictLast);
          ++vcount;
        }
      }
      if (lane == 0 && p.counters) {
        atomicAdd(&p.counters[2], (unsigned long long)vcount);
        atomicAdd(&p.counters[3], (unsigned long long)nsteps);
      }
    }
    __syncwarp();
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  } else if (warp == C::MMA_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
    if (nsteps > 0) {
      constexpr uint32_t IDESC_QK = make_idesc_bf16(128, 64, 0, 0);
      constexpr uint32_t IDESC_PV = make_idesc_bf16(128, D, 0, 1);
      const uint64_t dq0 = make_sdesc_sw128(sQ, 16, 1024);
      const uint64_t dk0 = make_sdesc_sw128(sK, 16, 1024);
      const uint64_t dv0 = make_sdesc_sw128(sV, C::V_ATOM, 1024);
      mbar_wait(bar_q, 0);
      auto issue_qk = [&](int s, int j) {
        const int st = j % KS;
        if (s == 0) mbar_wait(k_full + 8 * st, (j / KS) & 1);
        tc_fence_after();
        umma_qk_tile_w<D, 64>(tmem + C::S_COL + s * 64, dq0 + uint64_t((s * C::Q_TILE) >> 4),
                              dk0 + uint64_t((st * C::K_STEP) >> 4), IDESC_QK);
        if (s == (j < ns_a[1] ? 1 : 0)) umma_commit_w(k_empty + 8 * st);  // last reader of K(j)
        umma_commit_w(s_full + 8 * s);
      };
      unsigned vbase = 0;
      uint32_t o_started = 0;
      unsigned long long kept_m = 0;
      // the V unit of step j (numbered in the producer's fetch order) and whether
      // either tile kept it
      auto step_pvs = [&](int j) {
        uint32_t kept[2] = {0u, 0u};
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (j >= ns_a[s]) continue;
          mbar_wait(p_full + 32 * s + 8 * (j & 3), (j >> 2) & 1);
          tc_fence_after();
          if (frontier(j, s ? qi_a[1] : qi_a[0])) {
            kept[s] = 1;
          } else {
            const uint4 w = lds_u128(vote_sm + (s * 4 + (j & 3)) * 16);
            kept[s] = (w.x | w.y | w.z | w.w) ? 1u : 0u;
          }
          kept_m += kept[s];
        }
        if (kept[0] | kept[1]) {
          const unsigned uu = vbase;
          mbar_wait(v_full + 8 * (uu % VS), (uu / VS) & 1);
          tc_fence_after();
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            if (kept[s]) {
              umma_pv64_w(tmem + C::O_COL + s * D, tmem + C::P_COL + s * 64 + (j & 1) * 32,
                          dv0 + uint64_t(((uu % VS) * C::V_UNIT) >> 4), IDESC_PV, (o_started >> s) & 1u);
              o_started |= 1u << s;
            }
          }
          umma_commit_w(v_empty + 8 * (uu % VS));
          ++vbase;
        }
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (j >= ns_a[s]) continue;
          umma_commit_w(pv_done + 16 * s + 8 * (j & 1));  // one phase per step (per step parity)
          if (j == (s ? ns_a[1] : ns_a[0]) - 1) umma_commit_w(o_full + 8 * s);
        }
      };
      issue_qk(0, 0);
      if (ns_a[1] > 0) issue_qk(1, 0);
      for (int j = 0; j <= nsteps; ++j) {
        if (j + 1 < nsteps) {
          mbar_wait(s_free + 0, j & 1);
          issue_qk(0, j + 1);
        }
        if (j + 1 < ns_a[1]) {
          mbar_wait(s_free + 8, j & 1);
          issue_qk(1, j + 1);
        }
        if (j >= 1) step_pvs(j - 1);
      }
      if (lane == 0 && p.counters) {
        atomicAdd(&p.counters[0], (unsigned long long)(ns_a[0] + ns_a[1]));
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
    const int s = warp >> 2;
    const int wq = warp & 3;
    const int r = wq * 32 + lane;
    const int hq = s ? hq_a[1] : hq_a[0];
    const int qi_s = s ? qi_a[1] : qi_a[0];
    const int nst = s ? ns_a[1] : ns_a[0];
    if (qi_s < 0) {
      named_bar_arrive(15, C::NUM_THREADS);
      return;
    }
    const uint32_t lane_off = uint32_t(wq * 32) << 16;
    const uint32_t s_row = tmem + lane_off + C::S_COL + s * 64;
    const uint32_t o_row = tmem + lane_off + C::O_COL + s * D;
    const float sl2 = p.scale_log2;
    const float scale = p.scale;
    const float rescale_raw = p.rescale_raw;
    const int valid_len = p.valid_len;
    const int pos = qi_s < p.thr_positions - 1 ? qi_s : p.thr_positions - 1;
    const float T = p.thr[(long long)hq * p.thr_positions + pos];  // thresholds.py:87
    float m_ref = -INFINITY, l_sum = 0.f;
    bool o_valid = false;
    int8_t* drow = p.decisions ? p.decisions + (((long long)b * p.heads_q + hq) * p.num_q_tiles + qi_s) * p.gate_cols
                               : nullptr;
    for (int j = 0; j < nst; ++j) {
      mbar_wait(s_full + 8 * s, j & 1);
      tc_fence_after();
      uint32_t sv[64];
      tmem_ld32(s_row, &sv[0]);
      tmem_ld32(s_row + 32, &sv[32]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_free + 8 * s);  // QK_s(j+1) may overwrite S_s
      const bool fr = frontier(j, qi_s);
      if (CAUSAL && fr) {  // key j*64 + c vs row qi_s*128 + r
        const int off = (j & 1) * 64;
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (off + c > r) sv[c] = __float_as_uint(-INFINITY);
      }
      if (!CAUSAL && (j + 1) * 64 > valid_len) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (j * 64 + c >= valid_len) sv[c] = __float_as_uint(-INFINITY);
      }
      float mx;
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
        mx = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3));
      }
      uint32_t kept;
      if (fr) {
        kept = 1;
      } else {
        // ThresholdGate (gates.py:77-78): OR of the warps' votes; words in a
        // 4-deep ring (the issuer reads step j's words up to two steps later)
        const uint32_t wv = __reduce_or_sync(0xffffffffu, mx * scale > T ? 1u : 0u);
        const uint32_t slot = vote_sm + (s * 4 + (j & 3)) * 16;
        if (lane == 0) sts_u32(slot + wq * 4, wv);
        named_bar_sync(1 + s, 160);
        const uint4 all = lds_u128(slot);
        kept = (all.x | all.y | all.z | all.w) ? 1u : 0u;
      }
      if (drow && r == 0) drow[j] = fr ? int8_t(2) : (kept ? int8_t(3) : int8_t(1));
      const uint32_t p_bar = p_full + 32 * s + 8 * (j & 3);
      if (!kept) {
        __syncwarp();
        if (lane == 0) mbar_arrive(p_bar);
        continue;
      }
      const float m_new = fmaxf(m_ref, mx);
      float alpha = 1.f;
      bool rescale = false;
      if (!o_valid) {
        m_ref = m_new;
      } else if (m_new > m_ref + rescale_raw) {
        alpha = ex2_approx((m_ref - m_new) * sl2);
        m_ref = m_new;
        rescale = true;
      }
      if (__any_sync(0xffffffffu, rescale)) {
        if (j > 0) mbar_wait(pv_done + 16 * s + 8 * ((j - 1) & 1), ((j - 1) >> 1) & 1);  // PV_s(j-1): O quiescent
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
      const float neg = (m_ref == -INFINITY) ? 0.f : -m_ref * sl2;
      const uint64_t sl2x2 = f2_pack(sl2, sl2), negx2 = f2_pack(neg, neg);
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
      // P_s[j&1] was last read by PV_s(j-2)
      if (j >= 2) mbar_wait(pv_done + 16 * s + 8 * (j & 1), ((j - 2) >> 1) & 1);
      tc_fence_after();
      tmem_st32(tmem + lane_off + C::P_COL + s * 64 + (j & 1) * 32, pk);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_bar);
      const uint64_t acc = fadd2(acc0, acc1);
      l_sum = l_sum * alpha + (f2_lo(acc) + f2_hi(acc));
      o_valid = true;
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
        if (p.inject_fault && qi_s == 0 && r == 0 && hq == 0 && c == 0 && e == 0) a0 += 1.0f;
        bad |= !isfinite(a0) || !isfinite(a1);
        pk[e / 2] = pack_bf16x2(a0, a1);
      }
      store_o32(p, orow + c, pk);
    }
    p.lse[((long long)b * p.heads_q + hq) * p.seq_len + row] = m_ref * scale + logf(l_sum);
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
