// BSFA forward (K1) and calibration block-max (K2) for b_n = 64: the
// "gate-step" kernel.  One step = one 64-key gate tile (the reference's
// default 128x64 tiles, tiling.py:19-69).
//
// Same CTA decomposition as bsfa_kernel (NQ = 2 q heads of one GQA group per
// CTA sharing every K/V tile), but each query tile owns a ring of TWO 64-key
// S buffers in TMEM, so QK_s(j+1) is computed while the softmax works on
// S_s(j): the softmax no longer waits for PV + QK after releasing P.
//
// TMEM (512 columns at d = 128): O_0, O_1 (fp32, d cols) and S_{s,b}
// (fp32, 64 cols, b = j mod 2); P (bf16) overwrites the first 32 columns of
// its S buffer and is read by the PV MMA from TMEM.
//
// Per tile s and step j (b = j mod 2):
//   MMA   QK_s(j)  : S_{s,b} = Q_s K_j^T           8 x tcgen05.mma 128x64x16 (SS)
//   soft  wait S_{s,b}; 2 x tcgen05.ld; mask; row max; gate vote (BAR.RED.OR);
//         if kept: exponentials, P -> TMEM; release buffer b (p_full[s][b])
//   MMA   wait p_full[s][b]; if kept: O_s += P V_j   4 x tcgen05.mma 128xdx16 (TS)
//         then QK_s(j+2) into buffer b (it follows PV_s(j) in the tensor pipe)
// A lazy O rescale (running max grew by > 2^8, rare) waits on pv_done[s]
// (committed after every PV_s) for the last PV issued before this step.
#pragma once

#include "bsfa_kernel.cuh"

namespace bsfa {

template <int D, int NQ, bool CALIB>
struct GsCfg {
  static constexpr int NCH = D / 64;
  static constexpr int Q_TILE = 128 * D * 2;
  static constexpr int K_TILE = 64 * D * 2;  // one 64-key step
  static constexpr int V_UNIT = 64 * D * 2;
  static constexpr int KS = D == 128 ? 4 : 6;
  static constexpr int VS = CALIB ? 0 : (D == 128 ? 5 : 8);
  static constexpr int DQ = 8;             // decision ring depth (dynamic steps)
  static constexpr int MAXA = 4096;        // calibration: max off-frontier gate tiles per row
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + NQ * Q_TILE;
  static constexpr int OFF_V = OFF_K + KS * K_TILE;
  static constexpr int OFF_CAL = OFF_V + VS * V_UNIT;
  static constexpr int CAL_BYTES = CALIB ? NQ * MAXA * 4 : 0;
  static constexpr int OFF_BAR = OFF_CAL + CAL_BYTES;
  // bar_q, k ring, v ring, s_full[NQ][2], p_full[NQ][2], o_full[NQ], pv_done[NQ], dec ring
  static constexpr int NUM_BARS = 1 + 2 * KS + 2 * VS + 6 * NQ + 2 * NQ * DQ;
  static constexpr int OFF_DEC = (OFF_BAR + NUM_BARS * 8 + 15) / 16 * 16;  // u32 [NQ][DQ]
  static constexpr int OFF_DECM = OFF_DEC + NQ * DQ * 4;                    // u32 [NQ][2] (per S buffer)
  static constexpr int OFF_TMEMPTR = OFF_DECM + NQ * 2 * 4;
  static constexpr int SMEM_BYTES = OFF_TMEMPTR + 16 + 1024;
  static constexpr int O_COL = 0;
  static constexpr int S_COL = CALIB ? 0 : NQ * D;  // S_{s,b} at S_COL + (2s + b) * 64
  static constexpr int TMEM_NEED = S_COL + NQ * 2 * 64;
  static constexpr int TMEM_COLS = TMEM_NEED <= 128 ? 128 : (TMEM_NEED <= 256 ? 256 : 512);
  static constexpr int SOFTMAX_WARPS = 4 * NQ;
  static constexpr int KPROD_WARP = SOFTMAX_WARPS;
  static constexpr int MMA_WARP = SOFTMAX_WARPS + 1;
  static constexpr int VPROD_WARP = SOFTMAX_WARPS + 2;
  static constexpr int NUM_THREADS = (SOFTMAX_WARPS + 4) * 32;
  static constexpr int REG_LAUNCH = (65536 / NUM_THREADS) / 8 * 8 > 248 ? 248 : (65536 / NUM_THREADS) / 8 * 8;
  static constexpr int REG_OTHER = 56;
  static constexpr int REG_SOFT_MAX = (NUM_THREADS * REG_LAUNCH - 128 * REG_OTHER) / (SOFTMAX_WARPS * 32) / 8 * 8;
  static constexpr int REG_SOFT = REG_SOFT_MAX > 248 ? 248 : REG_SOFT_MAX;
  static_assert(NQ == 1 || NQ == 2, "one or two query tiles per CTA");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
  static_assert(TMEM_NEED <= 512, "TMEM budget");
};

// kind of 64-key step j for query block qi: frontier = the two gate tiles of
// block qi (tiling.py:50-60), always processed
__device__ __forceinline__ int gs_step_kind(int gate_mode, int j, int qi) {
  if ((j >> 1) == qi || gate_mode == kGateDense) return kStepAll;
  if (gate_mode == kGateFrontier) return kStepNone;
  return kStepDynamic;
}

template <int D, int NQ, bool CALIB>
__global__ void __launch_bounds__(GsCfg<D, NQ, CALIB>::NUM_THREADS, 1)
    bsfa_kernel_gs(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const KernelParams p) {
  using C = GsCfg<D, NQ, CALIB>;
  constexpr int KS = C::KS, VS = C::VS, DQ = C::DQ;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = opaque_u32((sraw + 1023u) & ~1023u);
  uint8_t* smem = smem_raw + (sbase - sraw);
  const uint32_t sQ = sbase + C::OFF_Q;
  const uint32_t sK = sbase + C::OFF_K;
  const uint32_t sV = sbase + C::OFF_V;
  int* cvals = reinterpret_cast<int*>(smem + C::OFF_CAL);
  const uint32_t bar_q = sbase + C::OFF_BAR;
  const uint32_t k_full = bar_q + 8;           // [KS]
  const uint32_t k_empty = k_full + 8 * KS;    // [KS]
  const uint32_t v_full = k_empty + 8 * KS;    // [VS]
  const uint32_t v_empty = v_full + 8 * VS;    // [VS]
  const uint32_t s_full = v_empty + 8 * VS;    // [NQ][2] QK into buffer landed
  const uint32_t p_full = s_full + 16 * NQ;    // [NQ][2] softmax done with buffer (P written)
  const uint32_t o_full = p_full + 16 * NQ;    // [NQ] last MMA of tile s landed
  const uint32_t pv_done = o_full + 8 * NQ;    // [NQ] one commit per PV_s
  const uint32_t dec_full = pv_done + 8 * NQ;  // [NQ][DQ]
  const uint32_t dec_empty = dec_full + 8 * NQ * DQ;
  const uint32_t dec_sm = sbase + C::OFF_DEC;
  const uint32_t decm_sm = sbase + C::OFF_DECM;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEMPTR);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  const int pairs = p.group / NQ;
  const int per_bg = p.num_q_tiles * pairs;
  const int unit = blockIdx.x;
  const int bg = unit / per_bg;
  const int rem = unit - bg * per_bg;
  const int qi = p.num_q_tiles - 1 - rem / pairs;
  const int pr = rem - (rem / pairs) * pairs;
  const int b = bg / p.heads_kv;
  const int g = bg - b * p.heads_kv;
  const int hq0 = g * p.group + pr * NQ;
  // 64-key steps: causal -> through the frontier (gate tiles 2i, 2i+1);
  // calibration -> the off-frontier prefix j < 2i (calibration.py:110-113)
  const int nsteps = CALIB ? 2 * qi : (p.causal ? 2 * qi + 2 : p.gate_cols);
  const int gate_mode = p.gate_mode;
  const bool causal = p.causal != 0;
  const int valid_len = p.valid_len;
  const bool tr_cta = BSFA_TRACE && p.trace && (int)blockIdx.x == p.trace_cta;

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
    for (int i = 0; i < 2 * NQ; ++i) {
      mbar_init(s_full + 8 * i, 1);
      mbar_init(p_full + 8 * i, 4);  // the 4 softmax warps of the tile
    }
    for (int s = 0; s < NQ; ++s) {
      mbar_init(o_full + 8 * s, 1);
      mbar_init(pv_done + 8 * s, 1);
    }
    for (int i = 0; i < NQ * DQ; ++i) {
      mbar_init(dec_full + 8 * i, 1);
      mbar_init(dec_empty + 8 * i, 1);
    }
    fence_mbarrier_init();
  }
  if constexpr (CALIB) {
    for (int i = threadIdx.x; i < NQ * C::MAXA; i += blockDim.x) cvals[i] = float_to_ordered(-INFINITY);
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
    // ======================= TMA producer: Q, K
    if (nsteps > 0) {
      if (lane == 0) {
        tma_prefetch_desc(&tm_q);
        tma_prefetch_desc(&tm_k);
      }
      mbar_arrive_expect_tx_w(bar_q, NQ * C::Q_TILE);
#pragma unroll
      for (int s = 0; s < NQ; ++s)
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_4d_w(sQ + s * C::Q_TILE + c * 128 * 128, &tm_q, bar_q, c * 64, qi * 128, hq0 + s, b, kEvictFirst);
      for (int j = 0; j < nsteps; ++j) {
        const int st = j % KS;
        mbar_wait(k_empty + 8 * st, ((j / KS) & 1) ^ 1);
        mbar_arrive_expect_tx_w(k_full + 8 * st, C::K_TILE);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_4d_w(sK + st * C::K_TILE + c * 64 * 128, &tm_k, k_full + 8 * st, c * 64, j * 64, g, b, kEvictLast);
      }
    }
    __syncwarp();
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  } else if (warp == C::VPROD_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
    // ======================= TMA producer: V of gate tiles kept by some query tile
    if constexpr (!CALIB) {
      if (nsteps > 0) {
        if (lane == 0) tma_prefetch_desc(&tm_v);
        unsigned vcount = 0, dn = 0;
        auto load_unit = [&](int j) {
          const int slot = int(vcount % VS);
          mbar_wait(v_empty + 8 * slot, ((vcount / VS) & 1) ^ 1);
          mbar_arrive_expect_tx_w(v_full + 8 * slot, C::V_UNIT);
#pragma unroll
          for (int c = 0; c < C::NCH; ++c)
            tma_load_4d_w(sV + slot * C::V_UNIT + c * 64 * 128, &tm_v, v_full + 8 * slot, c * 64, j * 64, g, b,
                          kEvictLast);
          ++vcount;
        };
        for (int j = 0; j < nsteps; ++j) {
          const int kind = gs_step_kind(gate_mode, j, qi);
          if (kind == kStepAll) {
            load_unit(j);
          } else if (kind == kStepDynamic) {
            // fetched on the first keep (tile 0's vote first); never if all skip
            uint32_t prev = 0;
            const int di = int(dn % DQ);
            const uint32_t ph = (dn / DQ) & 1;
#pragma unroll
            for (int s = 0; s < NQ; ++s) {
              mbar_wait(dec_full + 8 * (s * DQ + di), ph);
              const uint32_t w = lds_u32(dec_sm + (s * DQ + di) * 4);
              __syncwarp();
              mbar_arrive_w(dec_empty + 8 * (s * DQ + di));
              if (w && !prev) load_unit(j);
              prev |= w;
            }
            ++dn;
          }
        }
        if (lane == 0 && p.counters) {
          atomicAdd(&p.counters[2], (unsigned long long)vcount);
          atomicAdd(&p.counters[3], (unsigned long long)nsteps);
        }
      }
    }
    __syncwarp();
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  } else if (warp == C::MMA_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
    // ======================= MMA issuer (warp-convergent, one elected issuer)
    if (nsteps > 0) {
      constexpr uint32_t IDESC_QK = make_idesc_bf16(128, 64, 0, 0);
      constexpr uint32_t IDESC_PV = make_idesc_bf16(128, D, 0, 1);
      const uint64_t dq0 = make_sdesc_sw128(sQ, 16, 1024);
      const uint64_t dk0 = make_sdesc_sw128(sK, 16, 1024);
      const uint64_t dv0 = make_sdesc_sw128(sV, 64 * 128, 1024);
      mbar_wait(bar_q, 0);

      // QK_s(j) into S_{s, j mod 2}; the K stage is released after the last tile's QK
      auto issue_qk = [&](int s, int j) {
        const int st = j % KS;
        if (s == 0) mbar_wait(k_full + 8 * st, (j / KS) & 1);
        tc_fence_after();
        umma_qk_tile_w<D, 64>(tmem + C::S_COL + (2 * s + (j & 1)) * 64, dq0 + uint64_t((s * C::Q_TILE) >> 4),
                              dk0 + uint64_t((st * C::K_TILE) >> 4), IDESC_QK);
        if (s == NQ - 1) umma_commit_w(k_empty + 8 * st);
        umma_commit_w(s_full + 8 * (2 * s + (j & 1)));
      };

      // prologue: both buffers of both tiles
      for (int j = 0; j < 2 && j < nsteps; ++j)
#pragma unroll
        for (int s = 0; s < NQ; ++s) issue_qk(s, j);

      unsigned vcount = 0;
      uint32_t o_started = 0;
      for (int j = 0; j < nsteps; ++j) {
        const int kind = CALIB ? kStepDynamic : gs_step_kind(gate_mode, j, qi);
        const int bb = j & 1;
        bool unit_assigned = false;
#pragma unroll
        for (int s = 0; s < NQ; ++s) {
          mbar_wait(p_full + 8 * (2 * s + bb), (j >> 1) & 1);
          if (BSFA_TRACE && tr_cta && lane == 0 && j < kTraceSteps)
            p.trace[(kEvPSeen * 2 + s) * kTraceSteps + j] = clock64();
          tc_fence_after();
          if constexpr (!CALIB) {
            uint32_t keep;
            if (kind == kStepAll) keep = 1;
            else if (kind == kStepNone) keep = 0;
            else keep = lds_u32(decm_sm + (2 * s + bb) * 4);
            if (keep) {
              if (!unit_assigned) {
                const unsigned u = vcount;
                mbar_wait(v_full + 8 * (u % VS), (u / VS) & 1);
                unit_assigned = true;
                if (BSFA_TRACE && tr_cta && lane == 0 && j < kTraceSteps)
                  p.trace[(kEvVReady * 2 + s) * kTraceSteps + j] = clock64();
              }
              tc_fence_after();
              umma_pv64_w(tmem + C::O_COL + s * D, tmem + C::S_COL + (2 * s + bb) * 64,
                          dv0 + uint64_t(((vcount % VS) * C::V_UNIT) >> 4), IDESC_PV, (o_started >> s) & 1u);
              o_started |= 1u << s;
              umma_commit_w(pv_done + 8 * s);
            }
            if (s == NQ - 1 && unit_assigned) {
              umma_commit_w(v_empty + 8 * (vcount % VS));
              ++vcount;
            }
            if (j == nsteps - 1) umma_commit_w(o_full + 8 * s);
          }
          // QK_s(j+2) reuses buffer bb; it follows PV_s(j) in the tensor pipe
          if (j + 2 < nsteps) issue_qk(s, j + 2);
          if (BSFA_TRACE && tr_cta && lane == 0 && j < kTraceSteps)
            p.trace[(kEvIssued * 2 + s) * kTraceSteps + j] = clock64();
        }
      }
    }
    __syncwarp();
    named_bar_sync(15, C::NUM_THREADS);
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
    return;
  } else if (warp < C::SOFTMAX_WARPS) {
    setmaxnreg_inc<C::REG_SOFT>();
    // ======================= softmax of query tile s, one thread per row
    const int s = warp >> 2;
    const int wq = warp & 3;
    const int r = wq * 32 + lane;
    const int hq = hq0 + s;
    const uint32_t lane_off = uint32_t(wq * 32) << 16;
    const uint32_t o_row = tmem + lane_off + C::O_COL + s * D;
    const float sl2 = p.scale_log2;
    const float scale = p.scale;
    const float rescale_raw = p.rescale_raw;
    const bool tr0 = BSFA_TRACE && tr_cta && r == 0;

    float T = 0.f;
    if (!CALIB && gate_mode == kGateThreshold) {
      const int pos = qi < p.thr_positions - 1 ? qi : p.thr_positions - 1;
      T = p.thr[(long long)hq * p.thr_positions + pos];
    }

    float m_ref = -INFINITY;
    float l_sum = 0.f;
    bool o_valid = false;
    unsigned dn = 0;
    unsigned n_pv = 0;  // PVs of this tile issued so far (one per kept step)
    unsigned long long kept_tiles = 0;

    for (int j = 0; j < nsteps; ++j) {
      const int bb = j & 1;
      const uint32_t s_row = tmem + lane_off + C::S_COL + (2 * s + bb) * 64;
      mbar_wait(s_full + 8 * (2 * s + bb), (j >> 1) & 1);
      if (tr0 && j < kTraceSteps) p.trace[(kEvSReady * 2 + s) * kTraceSteps + j] = clock64();
      tc_fence_after();
      uint32_t sv[64];
      tmem_ld32(s_row, &sv[0]);
      tmem_ld32(s_row + 32, &sv[32]);
      tmem_wait_ld();

      const int kind = CALIB ? kStepDynamic : gs_step_kind(gate_mode, j, qi);
      if (!CALIB) {
        if ((j >> 1) == qi && causal) {  // frontier: key offset 64*(j-2i)+c vs row r
          const int off = (j & 1) * 64;
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (off + c > r) sv[c] = __float_as_uint(-INFINITY);
        }
        if (!causal && (j + 1) * 64 > valid_len) {
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (j * 64 + c >= valid_len) sv[c] = __float_as_uint(-INFINITY);
        }
      }
      float mh;
      {
        float a0 = fmax3(__uint_as_float(sv[0]), __uint_as_float(sv[1]), __uint_as_float(sv[2]));
        float a1 = fmax3(__uint_as_float(sv[3]), __uint_as_float(sv[4]), __uint_as_float(sv[5]));
        float a2 = fmax3(__uint_as_float(sv[6]), __uint_as_float(sv[7]), __uint_as_float(sv[8]));
        float a3 = fmax3(__uint_as_float(sv[9]), __uint_as_float(sv[10]), __uint_as_float(sv[11]));
        float a4 = fmax3(__uint_as_float(sv[12]), __uint_as_float(sv[13]), __uint_as_float(sv[14]));
        float a5 = fmax3(__uint_as_float(sv[15]), __uint_as_float(sv[16]), __uint_as_float(sv[17]));
        float a6 = fmax3(__uint_as_float(sv[18]), __uint_as_float(sv[19]), __uint_as_float(sv[20]));
        float a7 = fmax3(__uint_as_float(sv[21]), __uint_as_float(sv[22]), __uint_as_float(sv[23]));
#pragma unroll
        for (int c = 24; c < 56; c += 16) {
          a0 = fmax3(a0, __uint_as_float(sv[c]), __uint_as_float(sv[c + 1]));
          a1 = fmax3(a1, __uint_as_float(sv[c + 2]), __uint_as_float(sv[c + 3]));
          a2 = fmax3(a2, __uint_as_float(sv[c + 4]), __uint_as_float(sv[c + 5]));
          a3 = fmax3(a3, __uint_as_float(sv[c + 6]), __uint_as_float(sv[c + 7]));
          a4 = fmax3(a4, __uint_as_float(sv[c + 8]), __uint_as_float(sv[c + 9]));
          a5 = fmax3(a5, __uint_as_float(sv[c + 10]), __uint_as_float(sv[c + 11]));
          a6 = fmax3(a6, __uint_as_float(sv[c + 12]), __uint_as_float(sv[c + 13]));
          a7 = fmax3(a7, __uint_as_float(sv[c + 14]), __uint_as_float(sv[c + 15]));
        }
        a0 = fmax3(a0, __uint_as_float(sv[56]), __uint_as_float(sv[57]));
        a1 = fmax3(a1, __uint_as_float(sv[58]), __uint_as_float(sv[59]));
        a2 = fmax3(a2, __uint_as_float(sv[60]), __uint_as_float(sv[61]));
        a3 = fmax3(a3, __uint_as_float(sv[62]), __uint_as_float(sv[63]));
        mh = fmax3(fmax3(a0, a1, a2), fmax3(a3, a4, a5), fmaxf(a6, a7));
      }

      if constexpr (CALIB) {
        float m = mh;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
        if (lane == 0) atomicMax(&cvals[s * C::MAXA + j], float_to_ordered(m * scale));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full + 8 * (2 * s + bb));
        continue;
      } else {
        uint32_t keep;
        if (kind == kStepAll) {
          keep = 1;
        } else if (kind == kStepNone) {
          keep = 0;
        } else {
          keep = named_bar_red_or(1 + s, 128, mh * scale > T ? 1u : 0u);
        }
        if (tr0 && j < kTraceSteps) p.trace[(kEvVoted * 2 + s) * kTraceSteps + j] = clock64();
        if (r == 0) {
          if (kind == kStepDynamic) {
            const int di = int(dn % DQ);
            mbar_wait(dec_empty + 8 * (s * DQ + di), ((dn / DQ) & 1) ^ 1);
            sts_u32(dec_sm + (s * DQ + di) * 4, keep);
            mbar_arrive(dec_full + 8 * (s * DQ + di));
          }
          sts_u32(decm_sm + (2 * s + bb) * 4, keep);
        }
        if (kind == kStepDynamic) ++dn;
        if (!keep) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(p_full + 8 * (2 * s + bb));
          if (r == 0 && p.decisions) {
            int8_t* drow = p.decisions + (((long long)b * p.heads_q + hq) * p.num_q_tiles + qi) * p.gate_cols;
            drow[j] = int8_t(1);
          }
          if (tr0 && j < kTraceSteps) p.trace[(kEvPDone * 2 + s) * kTraceSteps + j] = clock64();
          continue;
        }

        const float m_new = fmaxf(m_ref, mh);
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
          // every PV_s issued so far (n_pv of them) must have landed
          mbar_wait(pv_done + 8 * s, (n_pv - 1) & 1);
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
        const uint64_t sl2x2 = f2_pack(sl2, sl2);
        const uint64_t negx2 = f2_pack(neg, neg);
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 64; c += 4) {
          const uint64_t x0 = ffma2(f2_pack(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])), sl2x2, negx2);
          const uint64_t x1 = ffma2(f2_pack(__uint_as_float(sv[c + 2]), __uint_as_float(sv[c + 3])), sl2x2, negx2);
          const float p0 = ex2_approx(f2_lo(x0)), p1 = ex2_approx(f2_hi(x0));
          float p2, p3;
          if (BSFA_EXP_EMU == 2 || (BSFA_EXP_EMU == 1 && ((c >> 2) & 1))) {
            const uint64_t x1d = BSFA_EXP_CHAIN ? ffma2(f2_pack(p0, p1), 0ull, x1) : x1;
            const uint64_t e1 = exp2_poly_x2(x1d);
            p2 = f2_lo(e1);
            p3 = f2_hi(e1);
          } else {
            p2 = ex2_approx(f2_lo(x1));
            p3 = ex2_approx(f2_hi(x1));
          }
          sv[c] = __float_as_uint(p0);
          sv[c + 1] = __float_as_uint(p1);
          sv[c + 2] = __float_as_uint(p2);
          sv[c + 3] = __float_as_uint(p3);
          pk[c / 2] = pack_bf16x2(p0, p1);
          pk[c / 2 + 1] = pack_bf16x2(p2, p3);
        }
        tmem_st32(s_row, pk);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full + 8 * (2 * s + bb));
        if (tr0 && j < kTraceSteps) p.trace[(kEvPDone * 2 + s) * kTraceSteps + j] = clock64();
        ++n_pv;

        uint64_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
#pragma unroll
        for (int c = 0; c < 64; c += 8) {
          acc0 = fadd2(acc0, f2_pack(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])));
          acc1 = fadd2(acc1, f2_pack(__uint_as_float(sv[c + 2]), __uint_as_float(sv[c + 3])));
          acc2 = fadd2(acc2, f2_pack(__uint_as_float(sv[c + 4]), __uint_as_float(sv[c + 5])));
          acc3 = fadd2(acc3, f2_pack(__uint_as_float(sv[c + 6]), __uint_as_float(sv[c + 7])));
        }
        const uint64_t acc = fadd2(fadd2(acc0, acc1), fadd2(acc2, acc3));
        l_sum = l_sum * alpha + (f2_lo(acc) + f2_hi(acc));
        if (r == 0) {
          ++kept_tiles;
          if (p.decisions) {
            int8_t* drow = p.decisions + (((long long)b * p.heads_q + hq) * p.num_q_tiles + qi) * p.gate_cols;
            drow[j] = (j >> 1) == qi ? int8_t(2) : int8_t(3);
          }
        }
        o_valid = true;
      }
    }

    if constexpr (CALIB) {
      const int A = nsteps;
      named_bar_sync(3 + s, 128);
      int* vals = cvals + s * C::MAXA;
      if (p.c_maxima) {
        float* out = p.c_maxima + ((long long)hq * p.num_q_tiles + qi) * p.gate_cols;
        for (int x = r; x < A; x += 128) out[x] = ordered_to_float(vals[x]);
      }
      int n2 = 1;
      while (n2 < A) n2 <<= 1;
      for (int kk = 2; kk <= n2; kk <<= 1) {
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
          for (int x = r; x < n2; x += 128) {
            const int y = x ^ jj;
            if (y > x) {
              const int a = vals[x], c = vals[y];
              const bool desc = (x & kk) == 0;
              if (desc ? (a < c) : (a > c)) {
                vals[x] = c;
                vals[y] = a;
              }
            }
          }
          named_bar_sync(3 + s, 128);
        }
      }
      if (r < p.c_num_levels) {
        const int k = p.c_levels[r];
        float cut;
        bool tie = false;
        if (k == 0) {
          cut = INFINITY;
        } else if (A <= k) {
          cut = -INFINITY;
        } else {
          cut = ordered_to_float(vals[k]);
          tie = vals[k - 1] == vals[k];
        }
        const long long idx = (((long long)r * p.c_num_layers + p.c_layer) * p.heads_q + hq) * p.c_positions + qi;
        if (isfinite(cut)) {
          p.c_sum[idx] += (double)cut;
          p.c_fin[idx] += 1;
        } else if (cut < 0.f) {
          p.c_neg[idx] += 1;
        } else {
          p.c_pos[idx] += 1;
        }
        if (tie) atomicAdd(&p.c_ties[r], 1ull);
      }
    } else {
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
          if (p.inject_fault && qi == 0 && r == 0 && s == 0 && c == 0 && e == 0) a0 += 1.0f;  // O[0][0] += 1
          bad |= !isfinite(a0) || !isfinite(a1);
          pk[e / 2] = pack_bf16x2(a0, a1);
        }
        store_o32(p, orow + c, pk);
      }
      p.lse[((long long)b * p.heads_q + hq) * p.seq_len + row] = m_ref * scale + logf(l_sum);
      if (bad && p.status) atomicOr(p.status, 1);
      if (r == 0 && p.counters) {
        atomicAdd(&p.counters[0], (unsigned long long)nsteps);
        atomicAdd(&p.counters[1], kept_tiles);
      }
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
