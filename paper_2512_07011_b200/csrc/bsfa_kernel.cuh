// BSFA forward (K1) and calibration block-max (K2) kernels for sm_100a.
//
// One CTA owns NQ query tiles of 128 rows that share one kv head (two q heads
// of a GQA group when NQ == 2) and streams the causally reachable 128-key
// tiles of that kv head.  Warp roles:
//   warps [0, 8*NQ)   softmax: 8 warps (256 threads) per query tile, two
//                     threads per row (TMEM lane), each owning one 64-key
//                     half of the 128-key tile (= one gate tile at b_n=64)
//   warp 8*NQ         TMA producer (Q once, K every tile, V only when kept)
//   warp 8*NQ+1       MMA issuer (tcgen05, single thread) + TMEM owner
//
// Per 128-key tile j and query tile s:
//   QK:  S_s = Q_s K_j^T           tcgen05.mma SS, fp32 accumulator in TMEM
//   gate: rowmax per gate tile (b_n columns) -> CTA-wide OR of
//         (rowmax * scale > T) over the 128 rows (bar.red.or) == the
//         reference's  tile.s_max > T  (gates.py:77-78, engine.py:30-38)
//   skip: no V TMA, no exp, no PV MMA, no statistics update (engine.py:172-174)
//   keep: online softmax (engine.py:57-68) with lazily rescaled O in TMEM;
//         P (bf16) written back into the S columns, O += P V_j (tcgen05.mma TS)
// Calibration (CALIB=true) runs the same QK front end over the off-frontier
// prefix j < A_p only (calibration.py:108-115) and reduces tile maxima.
#pragma once

#include "ptx.cuh"

namespace bsfa {

enum : int { kGateThreshold = 0, kGateDense = 1, kGateFrontier = 2 };

struct KernelParams {
  int batch, heads_q, heads_kv, group;
  int seq_len;       // padded sequence length (multiple of 128)
  int valid_len;     // unpadded length (non-causal key masking)
  int num_q_tiles;   // seq_len / 128
  int num_kv_tiles;  // seq_len / 128
  int gate_cols;     // seq_len / b_n
  int causal;
  int gate_mode;
  int thr_positions;
  float scale;
  float scale_log2;
  float rescale_raw;  // lazy-rescale threshold in raw score units
  int inject_fault;
  const float* thr;
  __nv_bfloat16* o;
  long long o_sb, o_sh, o_sn;
  float* lse;
  int8_t* decisions;
  unsigned long long* counters;
  int* status;
  // calibration
  int c_layer, c_num_layers, c_positions, c_num_levels;
  int c_levels[16];
  double* c_sum;
  int* c_fin;
  int* c_neg;
  int* c_pos;
  unsigned long long* c_ties;
  float* c_maxima;
};

template <int D, int NH, int NQ, bool CALIB>
struct KCfg {
  static constexpr int KT = 128;             // keys per MMA tile
  static constexpr int BN = KT / NH;         // gate tile width (reference b_n)
  static constexpr int NCH = D / 64;         // 128-byte swizzle atoms along head_dim
  static constexpr int Q_TILE = 128 * D * 2;
  static constexpr int K_TILE = KT * D * 2;
  static constexpr int V_TILE = BN * D * 2;  // one gate tile of V
  static constexpr int KS = CALIB ? 3 : (D == 128 ? 2 : 3);
  static constexpr int VS = CALIB ? 0 : 65536 / V_TILE;  // slots of one V gate tile (64 KB ring)
  static constexpr int DQ = KS;              // decision ring depth (see producer)
  static constexpr int MAXA = 4096;          // calibration: max off-frontier gate tiles per row
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + NQ * Q_TILE;
  static constexpr int OFF_V = OFF_K + KS * K_TILE;
  static constexpr int OFF_CAL = OFF_V + VS * V_TILE;
  static constexpr int CAL_BYTES = CALIB ? NQ * MAXA * 4 : 0;
  static constexpr int OFF_BAR = OFF_CAL + CAL_BYTES;
  static constexpr int NUM_BARS = 1 + 2 * KS + 2 * VS + NQ * (3 + DQ);
  static constexpr int OFF_XCH = OFF_BAR + NUM_BARS * 8;                  // row max / vote exchange
  static constexpr int XCH_BYTES = NQ * (2 * 2 * 128 * 4 + 16 * 4);
  static constexpr int OFF_DEC = OFF_XCH + XCH_BYTES;
  static constexpr int OFF_TMEMPTR = OFF_DEC + NQ * DQ * 4;
  static constexpr int SMEM_BYTES = OFF_TMEMPTR + 16 + 1024;  // + alignment slack
  // TMEM columns
  static constexpr int O_COL = 0;
  static constexpr int S_COL = CALIB ? 0 : NQ * D;
  static constexpr int TMEM_NEED = S_COL + NQ * KT;
  static constexpr int TMEM_COLS = TMEM_NEED <= 128 ? 128 : (TMEM_NEED <= 256 ? 256 : 512);
  static constexpr int SOFTMAX_WARPS = NQ * 8;  // two threads per row: 64-key column halves
  static constexpr int NUM_THREADS = SOFTMAX_WARPS * 32 + 64;
  static constexpr int PRODUCER_WARP = SOFTMAX_WARPS;
  static constexpr int MMA_WARP = SOFTMAX_WARPS + 1;
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
  static_assert(TMEM_NEED <= 512, "TMEM budget");
  static_assert(CALIB || VS >= 2 * NH, "V ring must hold two tiles");
};

template <int D, int NH, int NQ, bool CALIB>
__global__ void __launch_bounds__(NQ * 256 + 64, 1)
    bsfa_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v, const KernelParams p) {
  using C = KCfg<D, NH, NQ, CALIB>;
  constexpr int KT = C::KT, BN = C::BN, KS = C::KS, VS = C::VS, DQ = C::DQ;
  constexpr uint32_t HMASK = (1u << NH) - 1u;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + C::OFF_Q;
  uint8_t* sK = smem + C::OFF_K;
  uint8_t* sV = smem + C::OFF_V;
  int* cvals = reinterpret_cast<int*>(smem + C::OFF_CAL);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* bar_q = bars;
  uint64_t* k_full = bar_q + 1;
  uint64_t* k_empty = k_full + KS;
  uint64_t* v_full = k_empty + KS;
  uint64_t* v_empty = v_full + VS;
  uint64_t* s_full = v_empty + VS;
  uint64_t* p_full = s_full + NQ;
  uint64_t* o_full = p_full + NQ;
  uint64_t* dec_full = o_full + NQ;  // [NQ][DQ]
  volatile uint32_t* dec_words = reinterpret_cast<volatile uint32_t*>(smem + C::OFF_DEC);  // [NQ][DQ]
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEMPTR);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- work unit: (batch, kv head) major, heaviest query tile first, q-head pair minor
  const int pairs = p.group / NQ;
  const int per_bg = p.num_q_tiles * pairs;
  const int unit = blockIdx.x;
  const int bg = unit / per_bg;
  const int rem = unit - bg * per_bg;
  const int qi = p.num_q_tiles - 1 - rem / pairs;
  const int pair = rem - (rem / pairs) * pairs;
  const int b = bg / p.heads_kv;
  const int g = bg - b * p.heads_kv;
  const int hq0 = g * p.group + pair * NQ;
  const int ntiles = CALIB ? qi : (p.causal ? qi + 1 : p.num_kv_tiles);

  // ---- setup
  if (warp == C::PRODUCER_WARP && lane == 0) {
    mbar_init(bar_q, 1);
    for (int i = 0; i < KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int s = 0; s < NQ; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 8);
      mbar_init(&o_full[s], 1);
      for (int i = 0; i < DQ; ++i) mbar_init(&dec_full[s * DQ + i], 1);
    }
    fence_mbarrier_init();
  }
  if constexpr (CALIB) {
    // tile-maxima scratch starts at -inf (ordered-int encoding)
    const int ninit = NQ * C::MAXA;
    for (int i = threadIdx.x; i < ninit; i += blockDim.x) cvals[i] = float_to_ordered(-INFINITY);
  }
  if (warp == C::MMA_WARP) {
    tmem_alloc(tmem_ptr, C::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;

  if (warp == C::PRODUCER_WARP) {
    // ======================= TMA producer =======================
    if (lane == 0 && ntiles > 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      if constexpr (!CALIB) tma_prefetch_desc(&tm_v);
      mbar_arrive_expect_tx(bar_q, NQ * C::Q_TILE);
#pragma unroll
      for (int s = 0; s < NQ; ++s)
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_4d(sQ + s * C::Q_TILE + c * 128 * 128, &tm_q, bar_q, c * 64, qi * 128, hq0 + s, b,
                      kEvictFirst);

      auto load_k = [&](int j) {
        const int st = j % KS;
        mbar_wait(&k_empty[st], ((j / KS) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[st], C::K_TILE);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_4d(sK + st * C::K_TILE + c * KT * 128, &tm_k, &k_full[st], c * 64, j * KT, g, b, kEvictLast);
      };
      const int pre = ntiles < KS ? ntiles : KS;
      for (int j = 0; j < pre; ++j) load_k(j);

      unsigned long long vcount = 0;
      for (int j = 0; j < ntiles; ++j) {
        if constexpr (!CALIB) {
          // V gate tiles in decision order: tiles kept by query tile 0 first,
          // then any extra tiles kept only by query tile 1.  The MMA warp
          // derives the identical slot sequence from the same decision words.
          uint32_t have = 0;
#pragma unroll
          for (int s = 0; s < NQ; ++s) {
            const int di = s * DQ + (j % DQ);
            mbar_wait(&dec_full[di], (j / DQ) & 1);
            const uint32_t bits = dec_words[di] & HMASK;
            const uint32_t extra = bits & ~have;
            have |= bits;
#pragma unroll
            for (int h = 0; h < NH; ++h) {
              if ((extra >> h) & 1u) {
                const int slot = int(vcount % VS);
                mbar_wait(&v_empty[slot], uint32_t((vcount / VS) & 1) ^ 1u);
                mbar_arrive_expect_tx(&v_full[slot], C::V_TILE);
#pragma unroll
                for (int c = 0; c < C::NCH; ++c)
                  tma_load_4d(sV + slot * C::V_TILE + c * BN * 128, &tm_v, &v_full[slot], c * 64,
                              j * KT + h * BN, g, b, kEvictLast);
                ++vcount;
              }
            }
          }
        }
        // K_{j+KS} reuses K_j's stage; issuing it only after tile j's
        // decisions were consumed bounds how far the softmax warps can run
        // ahead of this loop (by KS tiles), which is what makes the DQ = KS
        // decision ring safe.
        if (j + KS < ntiles) load_k(j + KS);
      }
      if (p.counters && !CALIB) atomicAdd(&p.counters[2], vcount);
    }
    __syncwarp();
  } else if (warp == C::MMA_WARP) {
    // ======================= MMA issuer =======================
    if (lane == 0 && ntiles > 0) {
      constexpr uint32_t IDESC_QK = make_idesc_bf16(128, KT, 0, 0);
      constexpr uint32_t IDESC_PV = make_idesc_bf16(128, D, 0, 1);
      const uint32_t sQa = smem_u32(sQ);
      const uint32_t sKa = smem_u32(sK);
      const uint32_t sVa = smem_u32(sV);
      mbar_wait(bar_q, 0);
      tc_fence_after();

      auto issue_qk = [&](int s, int j) {
        const int st = j % KS;
        if (s == 0) {
          mbar_wait(&k_full[st], (j / KS) & 1);
          tc_fence_after();
        }
        const uint32_t d_tmem = tmem + C::S_COL + s * KT;
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = make_sdesc_sw128(sQa + s * C::Q_TILE + c * 128 * 128 + kk * 32, 16, 1024);
            const uint64_t bd = make_sdesc_sw128(sKa + st * C::K_TILE + c * KT * 128 + kk * 32, 16, 1024);
            umma_ss(d_tmem, ad, bd, IDESC_QK, (c | kk) != 0 ? 1u : 0u);
          }
        umma_commit(&s_full[s]);
        if (s == NQ - 1) umma_commit(&k_empty[st]);
      };

#pragma unroll
      for (int s = 0; s < NQ; ++s) issue_qk(s, 0);

      unsigned long long vcount = 0;
      uint32_t o_started = 0;
      for (int j = 0; j < ntiles; ++j) {
        if constexpr (CALIB) {
#pragma unroll
          for (int s = 0; s < NQ; ++s) {
            mbar_wait(&p_full[s], j & 1);
            tc_fence_after();
            if (j + 1 < ntiles) issue_qk(s, j + 1);
          }
        } else {
          uint32_t have = 0;
          int slot_of[NH];
#pragma unroll
          for (int h = 0; h < NH; ++h) slot_of[h] = 0;
          const unsigned long long first = vcount;
#pragma unroll
          for (int s = 0; s < NQ; ++s) {
            mbar_wait(&p_full[s], j & 1);
            const uint32_t bits = dec_words[s * DQ + (j % DQ)] & HMASK;
            const uint32_t extra = bits & ~have;
            have |= bits;
#pragma unroll
            for (int h = 0; h < NH; ++h) {
              if ((extra >> h) & 1u) {
                slot_of[h] = int(vcount % VS);
                mbar_wait(&v_full[slot_of[h]], uint32_t((vcount / VS) & 1));
                ++vcount;
              }
            }
            tc_fence_after();
            const uint32_t o_tmem = tmem + C::O_COL + s * D;
            const uint32_t p_tmem = tmem + C::S_COL + s * KT;
#pragma unroll
            for (int h = 0; h < NH; ++h) {
              if ((bits >> h) & 1u) {
                const uint32_t vb = sVa + slot_of[h] * C::V_TILE;
#pragma unroll
                for (int kk = 0; kk < BN / 16; ++kk) {
                  const uint64_t bd = make_sdesc_sw128(vb + kk * 16 * 128, BN * 128, 1024);
                  umma_ts(o_tmem, p_tmem + (h * BN + kk * 16) / 2, bd, IDESC_PV, (o_started >> s) & 1u);
                  o_started |= 1u << s;
                }
              }
            }
            if (j + 1 < ntiles)
              issue_qk(s, j + 1);
            else
              umma_commit(&o_full[s]);
          }
          for (unsigned long long x = first; x < vcount; ++x) umma_commit(&v_empty[int(x % VS)]);
        }
      }
    }
    __syncwarp();
  } else if (warp < C::SOFTMAX_WARPS) {
    // ======================= softmax warpgroups =======================
    // Query tile s has 8 warps: warp quarter wq owns TMEM lanes [32wq, 32wq+32)
    // (= rows), column half ch owns keys [64ch, 64ch+64) of each 128-key tile.
    // With b_n = 64 a thread's half is exactly one gate tile.
    const int s = warp >> 3;
    const int wq = warp & 3;
    const int ch = (warp >> 2) & 1;
    const int r = wq * 32 + lane;  // row inside the query tile == TMEM lane
    const int hq = hq0 + s;
    const uint32_t lane_off = uint32_t(wq * 32) << 16;
    const uint32_t s_tm = tmem + lane_off + C::S_COL + s * KT;
    constexpr int DH = D / 2;  // O columns owned by this thread
    const uint32_t o_tm = tmem + lane_off + C::O_COL + s * D + ch * DH;
    const uint32_t bar_id = 1 + s;
    const float sl2 = p.scale_log2;
    float* xrow = reinterpret_cast<float*>(smem + C::OFF_XCH) + s * (2 * 2 * 128);  // [2 parity][2 half][128]
    uint32_t* xwarp = reinterpret_cast<uint32_t*>(smem + C::OFF_XCH + NQ * 2 * 2 * 128 * 4) + s * 16;  // [2][8]

    float T = 0.f;
    if (!CALIB && p.gate_mode == kGateThreshold) {
      const int pos = qi < p.thr_positions - 1 ? qi : p.thr_positions - 1;
      T = p.thr[(long long)hq * p.thr_positions + pos];
    }

    // Ping-pong between the two query tiles (NQ == 2): the softmax sections
    // alternate (named barriers TURN0/TURN1, 512 threads each) so one tile's
    // exponentials overlap the other tile's PV + QK on the tensor cores
    // instead of both competing for the MUFUs and then both idling.
    const uint32_t turn_mine = 3 + s, turn_other = 3 + (s ^ 1);
    if (NQ == 2 && !CALIB && s == 1) named_bar_arrive(turn_other, 512);

    float m_ref = -INFINITY;  // raw (unscaled) reference max of this row
    float l_part = 0.f;       // row-sum of this thread's columns, relative to m_ref
    bool o_valid = false;
    unsigned long long kept_tiles = 0;

    for (int j = 0; j < ntiles; ++j) {
      mbar_wait(&s_full[s], j & 1);
      if (NQ == 2 && !CALIB) named_bar_sync(turn_mine, 512);
      tc_fence_after();
      uint32_t sv[64];
      tmem_ld32(s_tm + ch * 64, &sv[0]);
      tmem_ld32(s_tm + ch * 64 + 32, &sv[32]);
      tmem_wait_ld();

      const bool frontier = (j == qi);
      if (!CALIB) {
        if (frontier && p.causal) {
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (ch * 64 + c > r) sv[c] = __float_as_uint(-INFINITY);
        }
        if (!p.causal && (j + 1) * KT > p.valid_len) {
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (j * KT + ch * 64 + c >= p.valid_len) sv[c] = __float_as_uint(-INFINITY);
        }
      }
      float pm;
      {
        float m0 = fmaxf(__uint_as_float(sv[0]), __uint_as_float(sv[1]));
        float m1 = fmaxf(__uint_as_float(sv[2]), __uint_as_float(sv[3]));
#pragma unroll
        for (int c = 4; c < 64; c += 4) {
          m0 = fmaxf(m0, fmaxf(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])));
          m1 = fmaxf(m1, fmaxf(__uint_as_float(sv[c + 2]), __uint_as_float(sv[c + 3])));
        }
        pm = fmaxf(m0, m1);
      }

      if constexpr (CALIB) {
        float m = pm;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
        if (lane == 0) atomicMax(&cvals[s * C::MAXA + j * NH + (NH == 2 ? ch : 0)], float_to_ordered(m * p.scale));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[s]);
        continue;
      } else {
        // ---- exchange row maxima and gate votes between the two column halves
        const int par = j & 1;
        const bool vote = (p.gate_mode == kGateThreshold) && (pm * p.scale > T);
        const uint32_t wv = __ballot_sync(0xffffffffu, vote);
        xrow[(par * 2 + ch) * 128 + r] = pm;
        if (lane == 0) xwarp[par * 8 + ch * 4 + wq] = wv != 0u ? 1u : 0u;
        named_bar_sync(bar_id, 256);
        const float pm_other = xrow[(par * 2 + (ch ^ 1)) * 128 + r];
        const uint32_t v0 = xwarp[par * 8 + 0] | xwarp[par * 8 + 1] | xwarp[par * 8 + 2] | xwarp[par * 8 + 3];
        const uint32_t v1 = xwarp[par * 8 + 4] | xwarp[par * 8 + 5] | xwarp[par * 8 + 6] | xwarp[par * 8 + 7];
        uint32_t bits;
        if (frontier || p.gate_mode == kGateDense) {
          bits = HMASK;
        } else if (p.gate_mode == kGateFrontier) {
          bits = 0;
        } else {
          bits = (NH == 2) ? (v0 | (v1 << 1)) : (v0 | v1);
        }
        if (r == 0 && ch == 0) {
          const int di = s * DQ + (j % DQ);
          dec_words[di] = bits;
          mbar_arrive(&dec_full[di]);
          kept_tiles += __popc(bits);
          if (p.decisions) {
            int8_t* drow = p.decisions + (((long long)b * p.heads_q + hq) * p.num_q_tiles + qi) * p.gate_cols;
#pragma unroll
            for (int h = 0; h < NH; ++h)
              drow[j * NH + h] = frontier ? int8_t(2) : (((bits >> h) & 1u) ? int8_t(3) : int8_t(1));
          }
        }
        if (bits == 0) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[s]);
          if (NQ == 2 && !(s == 1 && j == ntiles - 1)) named_bar_arrive(turn_other, 512);
          continue;
        }

        const bool mine = (NH == 2) ? ((bits >> ch) & 1u) : true;
        const bool theirs = (NH == 2) ? ((bits >> (ch ^ 1)) & 1u) : true;
        float mx = mine ? pm : -INFINITY;
        if (theirs) mx = fmaxf(mx, pm_other);
        const float m_new = fmaxf(m_ref, mx);
        const bool need = m_new > m_ref + p.rescale_raw;
        float alpha = 1.f;
        if (!o_valid) {
          m_ref = m_new;
        } else if (need) {
          alpha = ex2_approx((m_ref - m_new) * sl2);
          m_ref = m_new;
        }
        if (mine) {
          // P = exp2(s * scale*log2e - m * scale*log2e), bf16-packed over S
          const float neg = (m_ref == -INFINITY) ? 0.f : -m_ref * sl2;
          const uint64_t sl2x2 = f2_pack(sl2, sl2);
          const uint64_t negx2 = f2_pack(neg, neg);
          uint64_t acc0 = 0, acc1 = 0;
          uint32_t pk[32];
#pragma unroll
          for (int c = 0; c < 64; c += 4) {
            const uint64_t x0 = ffma2(f2_pack(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])), sl2x2, negx2);
            const uint64_t x1 =
                ffma2(f2_pack(__uint_as_float(sv[c + 2]), __uint_as_float(sv[c + 3])), sl2x2, negx2);
            const float p0 = ex2_approx(f2_lo(x0)), p1 = ex2_approx(f2_hi(x0));
            const float p2 = ex2_approx(f2_lo(x1)), p3 = ex2_approx(f2_hi(x1));
            acc0 = fadd2(acc0, f2_pack(p0, p1));
            acc1 = fadd2(acc1, f2_pack(p2, p3));
            pk[c / 2] = pack_bf16x2(p0, p1);
            pk[c / 2 + 1] = pack_bf16x2(p2, p3);
          }
          tmem_st32(s_tm + ch * 32, pk);
          const uint64_t acc = fadd2(acc0, acc1);
          l_part = l_part * alpha + (f2_lo(acc) + f2_hi(acc));
        } else {
          l_part = l_part * alpha;
        }

        if (o_valid && __any_sync(0xffffffffu, need)) {
          const uint64_t ax2 = f2_pack(alpha, alpha);
#pragma unroll
          for (int c = 0; c < DH; c += 32) {
            uint32_t ov[32];
            tmem_ld32(o_tm + c, ov);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              const uint64_t t = fmul2(f2_pack(__uint_as_float(ov[e]), __uint_as_float(ov[e + 1])), ax2);
              ov[e] = __float_as_uint(f2_lo(t));
              ov[e + 1] = __float_as_uint(f2_hi(t));
            }
            tmem_st32(o_tm + c, ov);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[s]);
        if (NQ == 2 && !(s == 1 && j == ntiles - 1)) named_bar_arrive(turn_other, 512);
        o_valid = true;
      }
    }

    if constexpr (CALIB) {
      // ---- order statistics of this row of tile maxima (calibration.py:116-153)
      const int A = ntiles * NH;
      const int t = ch * 128 + r;  // 0..255
      named_bar_sync(bar_id, 256);
      int* vals = cvals + s * C::MAXA;
      if (p.c_maxima) {
        float* out = p.c_maxima + ((long long)hq * p.num_q_tiles + qi) * p.gate_cols;
        for (int x = t; x < A; x += 256) out[x] = ordered_to_float(vals[x]);
      }
      int n2 = 1;
      while (n2 < A) n2 <<= 1;
      for (int kk = 2; kk <= n2; kk <<= 1) {
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
          for (int x = t; x < n2; x += 256) {
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
          named_bar_sync(bar_id, 256);
        }
      }
      if (t < p.c_num_levels) {
        const int k = p.c_levels[t];
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
        const long long idx =
            (((long long)t * p.c_num_layers + p.c_layer) * p.heads_q + hq) * p.c_positions + qi;
        if (isfinite(cut)) {
          p.c_sum[idx] += (double)cut;
          p.c_fin[idx] += 1;
        } else if (cut < 0.f) {
          p.c_neg[idx] += 1;
        } else {
          p.c_pos[idx] += 1;
        }
        if (tie) atomicAdd(&p.c_ties[t], 1ull);
      }
    } else {
      // ---- epilogue: O / l -> bf16, lse = m*scale + ln(l)   (engine.py:178-182)
      xrow[(2 * 2 - 1 - ch) * 128 + r] = l_part;  // slots [1][*] of the exchange buffer are free now
      mbar_wait(&o_full[s], 0);
      tc_fence_after();
      named_bar_sync(bar_id, 256);
      const float l_sum = l_part + xrow[(2 + ch) * 128 + r];
      const float inv_l = 1.f / l_sum;
      bool bad = !(l_sum > 0.f);
      const int row = qi * 128 + r;
      __nv_bfloat16* orow =
          p.o + (long long)b * p.o_sb + (long long)hq * p.o_sh + (long long)row * p.o_sn + ch * DH;
#pragma unroll
      for (int c = 0; c < DH; c += 32) {
        uint32_t ov[32];
        tmem_ld32(o_tm + c, ov);
        tmem_wait_ld();
        if (p.inject_fault && qi == 0 && r == 0 && ch == 0 && c == 0)
          ov[0] = __float_as_uint(__uint_as_float(ov[0]) + l_sum);  // +1.0 on O[0][0]
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float a0 = __uint_as_float(ov[e]), a1 = __uint_as_float(ov[e + 1]);
          bad |= !isfinite(a0) || !isfinite(a1);
          pk[e / 2] = pack_bf16x2(a0 * inv_l, a1 * inv_l);
        }
        uint4* dst = reinterpret_cast<uint4*>(orow + c);
#pragma unroll
        for (int e = 0; e < 4; ++e) dst[e] = make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
      }
      if (ch == 0) p.lse[((long long)b * p.heads_q + hq) * p.seq_len + row] = m_ref * p.scale + logf(l_sum);
      if (bad && p.status) atomicOr(p.status, 1);
      if (r == 0 && ch == 0 && p.counters) {
        atomicAdd(&p.counters[0], (unsigned long long)ntiles * NH);
        atomicAdd(&p.counters[1], kept_tiles);
      }
    }
    tc_fence_before();
  }

  __syncthreads();
  if (warp == C::MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

}  // namespace bsfa
