// BSFA forward (K1) and calibration block-max (K2) kernels for sm_100a.
//
// One CTA owns one query tile (128 rows of one q head, query block i) and
// streams the reachable 128-key tiles of that head's kv head.  Warp roles:
//   warps 0..4TPR-1  softmax: TPR threads per row (TMEM lane = row), each
//                    owning 128/TPR consecutive keys of every 128-key tile
//   warp 4TPR        TMA producer for Q and K (K ring, unconditional)
//   warp 4TPR+1      tcgen05 issuer (single thread) + TMEM owner
//   warp 4TPR+2      TMA producer for V: fetches a V gate tile only when the
//                    gate kept it (decision ring from the softmax warps)
// TMEM holds O (fp32, d columns) and an NS-deep ring of S tiles (fp32, 128
// columns); P (bf16) is written over its S slot and read by the PV MMA (A
// operand from TMEM).  QK^T for tile j+NS is issued right after PV of tile j,
// so the score tiles are computed ahead of the softmax.
//
// Per 128-key tile j:
//   QK:   S = Q K_j^T                     8 x tcgen05.mma 128x128x16 (SS)
//   gate: per gate tile, OR over rows of (rowmax * scale > T) == the
//         reference's tile.s_max > T (gates.py:77-78, engine.py:30-38)
//   skip: no V TMA, no exp, no PV MMA, no statistics update (engine.py:172-174)
//   keep: online softmax (engine.py:57-68), lazily rescaled O, O += P V_j
// Calibration (CALIB) runs the same QK front end over the off-frontier prefix
// j < A_p only (calibration.py:108-115) and reduces tile maxima in smem.
#pragma once

#include "ptx.cuh"

namespace bsfa {

enum : int { kGateThreshold = 0, kGateDense = 1, kGateFrontier = 2 };
constexpr uint32_t kRescaleFlag = 0x80000000u;  // decision-word bit: O rescale before this tile's PV

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

template <int D, int NH, bool CALIB, int TPR>
struct KCfg {
  static constexpr int KT = 128;             // keys per MMA tile
  static constexpr int BN = KT / NH;         // gate tile width (reference b_n)
  static constexpr int NCH = D / 64;         // 128-byte swizzle atoms along head_dim
  static constexpr int Q_TILE = 128 * D * 2;
  static constexpr int K_TILE = KT * D * 2;
  static constexpr int V_TILE = BN * D * 2;  // one gate tile of V
  static constexpr int NS = CALIB ? 4 : 3;   // S ring depth in TMEM
  static constexpr int KS = CALIB ? 4 : 2;   // K ring depth in smem (QK issue is paced by the S ring)
  static constexpr int VS = CALIB ? 0 : (D == 128 ? 6 : 12) / (3 - NH);  // V gate-tile slots
  static constexpr int DQ = 8;               // decision ring depth (>= NS)
  static constexpr int MAXA = 4096;          // calibration: max off-frontier gate tiles per row
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_TILE;
  static constexpr int OFF_V = OFF_K + KS * K_TILE;
  static constexpr int OFF_CAL = OFF_V + VS * V_TILE;
  static constexpr int CAL_BYTES = CALIB ? MAXA * 4 : 0;
  static constexpr int OFF_BAR = OFF_CAL + CAL_BYTES;
  static constexpr int NUM_BARS = 1 + 2 * KS + 2 * VS + 2 * NS + 2 * DQ + 3;
  static constexpr int OFF_XCH = OFF_BAR + NUM_BARS * 8;  // [2 parity][TPR][128] f32 + [2][16] u32 + [TPR][128] f32
  static constexpr int XCH_BYTES = 2 * TPR * 128 * 4 + 2 * 16 * 4 + TPR * 128 * 4;
  static constexpr int OFF_DEC = OFF_XCH + XCH_BYTES;
  static constexpr int OFF_TMEMPTR = OFF_DEC + DQ * 4;
  static constexpr int SMEM_BYTES = OFF_TMEMPTR + 16 + 1024;  // + alignment slack
  // TMEM columns
  static constexpr int O_COL = 0;
  static constexpr int S_COL = CALIB ? 0 : D;
  static constexpr int TMEM_NEED = S_COL + NS * KT;
  static constexpr int TMEM_COLS = TMEM_NEED <= 128 ? 128 : (TMEM_NEED <= 256 ? 256 : 512);
  static constexpr int CW = 128 / TPR;       // key columns per softmax thread
  static constexpr int SOFTMAX_WARPS = 4 * TPR;
  static constexpr int KPROD_WARP = SOFTMAX_WARPS;
  static constexpr int MMA_WARP = SOFTMAX_WARPS + 1;
  static constexpr int VPROD_WARP = SOFTMAX_WARPS + 2;
  static constexpr int NUM_THREADS = (SOFTMAX_WARPS + 3) * 32;
  static_assert(TPR == 2 || TPR == 4, "2 or 4 threads per row");
  static_assert(D / TPR >= 32, "O columns per thread must be a multiple of 32");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
  static_assert(TMEM_NEED <= 512, "TMEM budget");
  static_assert(CALIB || VS >= NH * NS, "V ring must cover the S ring");
  static_assert(DQ >= NS && DQ >= KS, "decision ring depth");
};

template <int D, int NH, bool CALIB, int TPR>
__global__ void __launch_bounds__((4 * TPR + 3) * 32, 1)
    bsfa_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v, const KernelParams p) {
  using C = KCfg<D, NH, CALIB, TPR>;
  constexpr int KT = C::KT, BN = C::BN, KS = C::KS, VS = C::VS, NS = C::NS, DQ = C::DQ;
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
  uint64_t* p_full = s_full + NS;
  uint64_t* dec_full = p_full + NS;
  uint64_t* dec_empty = dec_full + DQ;
  uint64_t* o_full = dec_empty + DQ;
  uint64_t* o_quiet = o_full + 1;     // MMA commit: every issued MMA has landed (rescale may touch O)
  uint64_t* o_rescaled = o_full + 2;  // softmax warps: O rescaled, PV may resume
  volatile uint32_t* dec_words = reinterpret_cast<volatile uint32_t*>(smem + C::OFF_DEC);
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEMPTR);
  const uint32_t xch_row = smem_u32(smem + C::OFF_XCH);         // f32 [2][TPR][128]  partial row maxima
  const uint32_t xch_vote = xch_row + 2 * TPR * 128 * 4;        // u32 [2][16]        per-warp votes
  const uint32_t xch_l = xch_vote + 2 * 16 * 4;                 // f32 [TPR][128]     partial row sums

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- work unit: (batch, kv head) major, heaviest query block first, the
  //      q heads of the GQA group minor (they share every K/V tile in L2)
  const int per_bg = p.num_q_tiles * p.group;
  const int unit = blockIdx.x;
  const int bg = unit / per_bg;
  const int rem = unit - bg * per_bg;
  const int qi = p.num_q_tiles - 1 - rem / p.group;
  const int b = bg / p.heads_kv;
  const int g = bg - b * p.heads_kv;
  const int hq = g * p.group + (rem - (rem / p.group) * p.group);
  const int ntiles = CALIB ? qi : (p.causal ? qi + 1 : p.num_kv_tiles);

  // ---- setup
  if (warp == C::KPROD_WARP && lane == 0) {
    mbar_init(bar_q, 1);
    for (int i = 0; i < KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], C::SOFTMAX_WARPS);
    }
    for (int i = 0; i < DQ; ++i) {
      mbar_init(&dec_full[i], 1);
      mbar_init(&dec_empty[i], 1);
    }
    mbar_init(o_full, 1);
    mbar_init(o_quiet, 1);
    mbar_init(o_rescaled, C::SOFTMAX_WARPS);
    fence_mbarrier_init();
  }
  if constexpr (CALIB) {
    for (int i = threadIdx.x; i < C::MAXA; i += blockDim.x) cvals[i] = float_to_ordered(-INFINITY);
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
    // ======================= TMA producer: Q, K (warp-convergent, one elected issuer)
    if (ntiles > 0) {
      if (lane == 0) {
        tma_prefetch_desc(&tm_q);
        tma_prefetch_desc(&tm_k);
      }
      mbar_arrive_expect_tx_w(bar_q, C::Q_TILE);
#pragma unroll
      for (int c = 0; c < C::NCH; ++c)
        tma_load_4d_w(sQ + c * 128 * 128, &tm_q, bar_q, c * 64, qi * 128, hq, b, kEvictFirst);
      for (int j = 0; j < ntiles; ++j) {
        const int st = j % KS;
        mbar_wait(&k_empty[st], ((j / KS) & 1) ^ 1);
        mbar_arrive_expect_tx_w(&k_full[st], C::K_TILE);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_4d_w(sK + st * C::K_TILE + c * KT * 128, &tm_k, &k_full[st], c * 64, j * KT, g, b, kEvictLast);
      }
    }
    __syncwarp();
  } else if (warp == C::VPROD_WARP) {
    // ======================= TMA producer: V of kept gate tiles =======================
    if constexpr (!CALIB) {
      if (ntiles > 0) {
        if (lane == 0) tma_prefetch_desc(&tm_v);
        unsigned long long vcount = 0;
        for (int j = 0; j < ntiles; ++j) {
          const int di = j % DQ;
          mbar_wait(&dec_full[di], (j / DQ) & 1);
          const uint32_t bits = __shfl_sync(0xffffffffu, dec_words[di], 0) & HMASK;
          __syncwarp();
          mbar_arrive_w(&dec_empty[di]);
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            if ((bits >> h) & 1u) {
              const int slot = int(vcount % VS);
              mbar_wait(&v_empty[slot], uint32_t((vcount / VS) & 1) ^ 1u);
              mbar_arrive_expect_tx_w(&v_full[slot], C::V_TILE);
#pragma unroll
              for (int c = 0; c < C::NCH; ++c)
                tma_load_4d_w(sV + slot * C::V_TILE + c * BN * 128, &tm_v, &v_full[slot], c * 64, j * KT + h * BN,
                              g, b, kEvictLast);
              ++vcount;
            }
          }
        }
        if (lane == 0 && p.counters) atomicAdd(&p.counters[2], vcount);
      }
    }
    __syncwarp();
  } else if (warp == C::MMA_WARP) {
    // ======================= MMA issuer (warp-convergent, one elected issuer) ==========
    if (ntiles > 0) {
      constexpr uint32_t IDESC_QK = make_idesc_bf16(128, KT, 0, 0);
      constexpr uint32_t IDESC_PV = make_idesc_bf16(128, D, 0, 1);
      // descriptor templates; per-MMA offsets only touch the 14-bit start-address field
      const uint64_t dq0 = make_sdesc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t dk0 = make_sdesc_sw128(smem_u32(sK), 16, 1024);
      const uint64_t dv0 = make_sdesc_sw128(smem_u32(sV), BN * 128, 1024);
      mbar_wait(bar_q, 0);

      auto issue_qk = [&](int t) {
        const int st = t % KS;
        mbar_wait(&k_full[st], (t / KS) & 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + C::S_COL + (t % NS) * KT;
        const uint64_t dk = dk0 + uint64_t((st * C::K_TILE) >> 4);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_ss_w(d_tmem, dq0 + uint64_t((c * 128 * 128 + kk * 32) >> 4),
                      dk + uint64_t((c * KT * 128 + kk * 32) >> 4), IDESC_QK, (c | kk) != 0 ? 1u : 0u);
        umma_commit_w(&s_full[t % NS]);
        umma_commit_w(&k_empty[st]);
      };

      const int pre = ntiles < NS ? ntiles : NS;
      for (int t = 0; t < pre; ++t) issue_qk(t);

      unsigned long long vcount = 0;
      uint32_t o_started = 0;
      uint32_t n_rescale = 0;
      for (int j = 0; j < ntiles; ++j) {
        const int sb = j % NS;
        mbar_wait(&p_full[sb], (j / NS) & 1);
        if constexpr (!CALIB) {
          const uint32_t word = __shfl_sync(0xffffffffu, dec_words[j % DQ], 0);
          const uint32_t bits = word & HMASK;
          if (word & kRescaleFlag) {
            // the softmax warps rescale O in TMEM: let every in-flight MMA land,
            // then hold PV_j until they are done
            umma_commit_w(o_quiet);
            mbar_wait(o_rescaled, n_rescale & 1);
            ++n_rescale;
          }
          const uint32_t p_tmem = tmem + C::S_COL + sb * KT;
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            if ((bits >> h) & 1u) {
              const int slot = int(vcount % VS);
              mbar_wait(&v_full[slot], uint32_t((vcount / VS) & 1));
              ++vcount;
              tc_fence_after();
              const uint64_t dv = dv0 + uint64_t((slot * C::V_TILE) >> 4);
#pragma unroll
              for (int kk = 0; kk < BN / 16; ++kk) {
                umma_ts_w(tmem + C::O_COL, p_tmem + (h * BN + kk * 16) / 2, dv + uint64_t((kk * 16 * 128) >> 4),
                          IDESC_PV, o_started);
                o_started = 1;
              }
              umma_commit_w(&v_empty[slot]);
            }
          }
          if (j == ntiles - 1) umma_commit_w(o_full);
        } else {
          tc_fence_after();
        }
        if (j + NS < ntiles) issue_qk(j + NS);  // reuses S slot sb, ordered after PV_j
      }
    }
    __syncwarp();
  } else if (warp < C::SOFTMAX_WARPS) {
    // ======================= softmax =======================
    // TPR threads per row: warp quarter wq owns TMEM lanes [32wq, 32wq+32),
    // column chunk cq owns keys [CW*cq, CW*cq + CW) of every 128-key tile.
    constexpr int CW = C::CW;
    constexpr int NTHR = 128 * TPR;
    const int wq = warp & 3;
    const int cq = warp >> 2;
    const int gh = (NH == 2) ? (cq * CW) / 64 : 0;  // gate tile holding this chunk
    const int r = wq * 32 + lane;                   // row inside the query tile == TMEM lane
    const uint32_t lane_off = uint32_t(wq * 32) << 16;
    constexpr int DH = D / TPR;  // O columns owned by this thread
    const uint32_t o_tm = tmem + lane_off + C::O_COL + cq * DH;
    const float sl2 = p.scale_log2;

    float T = 0.f;
    if (!CALIB && p.gate_mode == kGateThreshold) {
      const int pos = qi < p.thr_positions - 1 ? qi : p.thr_positions - 1;
      T = p.thr[(long long)hq * p.thr_positions + pos];
    }

    float m_ref = -INFINITY;  // raw (unscaled) reference max of this row
    float l_part = 0.f;       // row sum over this thread's columns, relative to m_ref
    bool o_valid = false;
    uint32_t n_rescale = 0;
    unsigned long long kept_tiles = 0;

    for (int j = 0; j < ntiles; ++j) {
      const int sb = j % NS;
      const uint32_t s_row = tmem + lane_off + C::S_COL + sb * KT;
      mbar_wait(&s_full[sb], (j / NS) & 1);
      tc_fence_after();
      uint32_t sv[CW];
#pragma unroll
      for (int c = 0; c < CW; c += 32) tmem_ld32(s_row + cq * CW + c, &sv[c]);
      tmem_wait_ld();

      const bool frontier = (j == qi);
      if (!CALIB) {
        if (frontier && p.causal) {
#pragma unroll
          for (int c = 0; c < CW; ++c)
            if (cq * CW + c > r) sv[c] = __float_as_uint(-INFINITY);
        }
        if (!p.causal && (j + 1) * KT > p.valid_len) {
#pragma unroll
          for (int c = 0; c < CW; ++c)
            if (j * KT + cq * CW + c >= p.valid_len) sv[c] = __float_as_uint(-INFINITY);
        }
      }
      float pm;
      {
        float m0 = fmaxf(__uint_as_float(sv[0]), __uint_as_float(sv[1]));
        float m1 = fmaxf(__uint_as_float(sv[2]), __uint_as_float(sv[3]));
        float m2 = fmaxf(__uint_as_float(sv[4]), __uint_as_float(sv[5]));
        float m3 = fmaxf(__uint_as_float(sv[6]), __uint_as_float(sv[7]));
#pragma unroll
        for (int c = 8; c < CW; c += 8) {
          m0 = fmaxf(m0, fmaxf(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])));
          m1 = fmaxf(m1, fmaxf(__uint_as_float(sv[c + 2]), __uint_as_float(sv[c + 3])));
          m2 = fmaxf(m2, fmaxf(__uint_as_float(sv[c + 4]), __uint_as_float(sv[c + 5])));
          m3 = fmaxf(m3, fmaxf(__uint_as_float(sv[c + 6]), __uint_as_float(sv[c + 7])));
        }
        pm = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
      }

      if constexpr (CALIB) {
        float m = pm;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
        if (lane == 0) atomicMax(&cvals[j * NH + gh], float_to_ordered(m * p.scale));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sb]);
        continue;
      } else {
        // ---- exchange partial row maxima and gate votes between the chunks
        const int par = j & 1;
        const bool vote = (p.gate_mode == kGateThreshold) && (pm * p.scale > T);
        const uint32_t wv = __ballot_sync(0xffffffffu, vote);
        // conservative rescale request: this chunk's max outgrows the reference
        const uint32_t wr = __ballot_sync(0xffffffffu, o_valid && pm > m_ref + p.rescale_raw);
        sts_f32(xch_row + ((par * TPR + cq) * 128 + r) * 4, pm);
        if (lane == 0) sts_u32(xch_vote + (par * 16 + warp) * 4, (wv != 0u ? 1u : 0u) | (wr != 0u ? 2u : 0u));
        named_bar_sync(1, NTHR);
        float pq[TPR];
#pragma unroll
        for (int q = 0; q < TPR; ++q) pq[q] = (q == cq) ? pm : lds_f32(xch_row + ((par * TPR + q) * 128 + r) * 4);
        uint32_t vw[TPR];  // OR of the 4 warp votes of chunk q
#pragma unroll
        for (int q = 0; q < TPR; ++q) {
          const uint4 v4 = lds_u128(xch_vote + (par * 16 + 4 * q) * 4);
          vw[q] = v4.x | v4.y | v4.z | v4.w;
        }
        uint32_t vote_h0 = 0, vote_h1 = 0, rq = 0;
#pragma unroll
        for (int q = 0; q < TPR; ++q) {
          if ((q * CW) / 64 == 0) vote_h0 |= vw[q] & 1u; else vote_h1 |= vw[q] & 1u;
          rq |= vw[q] & 2u;
        }
        uint32_t bits;
        if (frontier || p.gate_mode == kGateDense) {
          bits = HMASK;
        } else if (p.gate_mode == kGateFrontier) {
          bits = 0;
        } else {
          bits = (NH == 2) ? (vote_h0 | (vote_h1 << 1)) : (vote_h0 | vote_h1);
        }
        const bool do_rescale = rq != 0u && bits != 0u;
        if (warp == 0 && lane == 0) {
          const int di = j % DQ;
          mbar_wait(&dec_empty[di], ((j / DQ) & 1) ^ 1);
          dec_words[di] = bits | (do_rescale ? kRescaleFlag : 0u);
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
          if (lane == 0) mbar_arrive(&p_full[sb]);
          continue;
        }

        const bool mine = (bits >> gh) & 1u;
        float mx = -INFINITY;
#pragma unroll
        for (int q = 0; q < TPR; ++q) {
          const int hq_gate = (NH == 2) ? (q * CW) / 64 : 0;
          if ((bits >> hq_gate) & 1u) mx = fmaxf(mx, pq[q]);
        }
        const float m_new = fmaxf(m_ref, mx);
        float alpha = 1.f;
        if (!o_valid) {
          m_ref = m_new;
        } else if (do_rescale && m_new > m_ref + p.rescale_raw) {
          alpha = ex2_approx((m_ref - m_new) * sl2);
          m_ref = m_new;
        }
        if (mine) {
          // P = exp2(s * scale*log2e - m * scale*log2e), bf16-packed over S
          const float neg = (m_ref == -INFINITY) ? 0.f : -m_ref * sl2;
          const uint64_t sl2x2 = f2_pack(sl2, sl2);
          const uint64_t negx2 = f2_pack(neg, neg);
          uint64_t acc0 = 0, acc1 = 0;
          uint32_t pk[CW / 2];
#pragma unroll
          for (int c = 0; c < CW; c += 4) {
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
          // P columns [cq*CW/2, (cq+1)*CW/2) of the slot
          if constexpr (CW == 64) {
            tmem_st32(s_row + cq * (CW / 2), pk);
          } else {
            tmem_st16(s_row + cq * (CW / 2), pk);
          }
          const uint64_t acc = fadd2(acc0, acc1);
          l_part = l_part * alpha + (f2_lo(acc) + f2_hi(acc));
        } else {
          l_part = l_part * alpha;
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sb]);
        if (do_rescale) {
          // rare: the running max grew by > 2^8; rescale this thread's O columns
          // once every issued MMA (incl. PV_{j-1}) has landed
          mbar_wait(o_quiet, n_rescale & 1);
          ++n_rescale;
          tc_fence_after();
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
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(o_rescaled);
        }
        o_valid = true;
      }
    }

    if constexpr (CALIB) {
      // ---- order statistics of this row of tile maxima (calibration.py:116-153)
      const int A = ntiles * NH;
      const int t = cq * 128 + r;  // 0..NTHR-1
      named_bar_sync(1, NTHR);
      int* vals = cvals;
      if (p.c_maxima) {
        float* out = p.c_maxima + ((long long)hq * p.num_q_tiles + qi) * p.gate_cols;
        for (int x = t; x < A; x += NTHR) out[x] = ordered_to_float(vals[x]);
      }
      int n2 = 1;
      while (n2 < A) n2 <<= 1;
      for (int kk = 2; kk <= n2; kk <<= 1) {
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
          for (int x = t; x < n2; x += NTHR) {
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
          named_bar_sync(1, NTHR);
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
      sts_f32(xch_l + (cq * 128 + r) * 4, l_part);
      mbar_wait(o_full, 0);
      tc_fence_after();
      named_bar_sync(1, NTHR);
      float l_sum = 0.f;
#pragma unroll
      for (int q = 0; q < TPR; ++q) l_sum += (q == cq) ? l_part : lds_f32(xch_l + (q * 128 + r) * 4);
      const float inv_l = 1.f / l_sum;
      bool bad = !(l_sum > 0.f);
      const int row = qi * 128 + r;
      __nv_bfloat16* orow =
          p.o + (long long)b * p.o_sb + (long long)hq * p.o_sh + (long long)row * p.o_sn + cq * DH;
#pragma unroll
      for (int c = 0; c < DH; c += 32) {
        uint32_t ov[32];
        tmem_ld32(o_tm + c, ov);
        tmem_wait_ld();
        if (p.inject_fault && qi == 0 && r == 0 && cq == 0 && c == 0)
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
      if (cq == 0) p.lse[((long long)b * p.heads_q + hq) * p.seq_len + row] = m_ref * p.scale + logf(l_sum);
      if (bad && p.status) atomicOr(p.status, 1);
      if (warp == 0 && lane == 0 && p.counters) {
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
