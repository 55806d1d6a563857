// BSFA forward (K1) and calibration block-max (K2) kernels for sm_100a.
//
// One CTA owns one query tile (128 rows of one q head, query block i) and
// streams the reachable key tiles (one gate tile of b_n keys each) of that
// head's kv head.  Warp roles:
//   warps 0..7   softmax, two groups of 4 warps.  Group g owns the key tiles
//                j = g (mod 2) of this query tile: thread r of a group owns
//                row r (TMEM lane r) over all 128 keys of the tile, keeps its
//                own running max / sum and accumulates into its own O slot.
//                The two partial states are merged in the epilogue (the same
//                rescale-and-add the online softmax does between tiles).
//   warp 8       TMA producer for Q and K (K ring, unconditional)
//   warp 9       tcgen05 issuer (warp-convergent, one elected lane) + TMEM owner
//   warp 10      TMA producer for V: fetches a V gate tile only when the
//                gate kept it (decision ring from the softmax groups)
// TMEM: O_0, O_1 (fp32, d columns each) and a ring of S slots (fp32, b_n
// columns; 4 slots at b_n = 64, i.e. two per group); P (bf16) is written
// over its slot and read by the PV MMA (A operand from TMEM).  QK^T of a
// group's next tile is already in flight while the group works on the
// current one, and the other group's PV runs under its exponentials.
//
// Per key tile j of b_n = 64 or 128 keys (group g = j mod 2):
//   QK:   S = Q K_j^T                     tcgen05.mma 128 x b_n x 16 (SS)
//   gate: per gate tile, OR over rows of (rowmax * scale > T) == the
//         reference's tile.s_max > T (gates.py:77-78, engine.py:30-38)
//   skip: no V TMA, no exp, no PV MMA, no statistics update (engine.py:172-174)
//   keep: online softmax (engine.py:57-68), lazily rescaled O_g, O_g += P V_j
// Calibration (CALIB) runs the same QK front end over the off-frontier prefix
// j < A_p only (calibration.py:108-115) and reduces tile maxima in smem.
#pragma once

#include "ptx.cuh"

// Fraction of exponentials computed by polynomial on the FMA pipe instead of
// the MUFU: 0 = none, 1 = 1/4, 2 = 1/2.
#ifndef BSFA_EXP_EMU
#define BSFA_EXP_EMU 1
#endif
// Softmax groups take turns (named-barrier hand-off) so each group's
// exponentials run while the other group's PV/QK are on the tensor cores,
// instead of both groups sharing the MUFUs and then both waiting.
#ifndef BSFA_TURNS
#define BSFA_TURNS 0
#endif

namespace bsfa {

enum : int { kGateThreshold = 0, kGateDense = 1, kGateFrontier = 2 };
constexpr uint32_t kRescaleFlag = 0x80000000u;  // decision-word bit: rescale O_g before this tile's PV

struct KernelParams {
  int batch, heads_q, heads_kv, group;
  int seq_len;       // padded sequence length (multiple of 128)
  int valid_len;     // unpadded length (non-causal key masking)
  int num_q_tiles;   // seq_len / 128
  int num_kv_tiles;  // seq_len / b_n
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
  // debug: per-tile clock64 timestamps of one CTA (bsfa_debug_trace)
  long long* trace;
  int trace_cta;
};

// trace slots: trace[ev * kTraceTiles + j]
constexpr int kTraceTiles = 4096;
enum : int { kEvSReady = 0, kEvVoted = 1, kEvPDone = 2, kEvPSeen = 3, kEvIssued = 4, kEvVReady = 5, kEvKReady = 6 };

template <int D, int KT_, bool CALIB>
struct KCfg {
  static constexpr int KT = KT_;             // keys per MMA tile == gate tile width (reference b_n)
  static constexpr int NCH = D / 64;         // 128-byte swizzle atoms along head_dim
  static constexpr int Q_TILE = 128 * D * 2;
  static constexpr int K_TILE = KT * D * 2;
  static constexpr int V_TILE = KT * D * 2;
  static constexpr int NG = 2;               // softmax groups (alternate key tiles)
  // S slots in TMEM (slot = tile mod NS).  With 64-key tiles each group owns
  // two slots, so QK^T of its next tile runs while it works on the current one.
  static constexpr int NS_FIT = (512 - NG * D) / KT;
  static constexpr int NS = CALIB ? 512 / KT / 2 : (NS_FIT < 4 ? NS_FIT : 4);
  // K ring 96 KB (TMA latency from L2/HBM is 2-4k cycles under load: K must be
  // requested several tiles ahead); V ring 80 KB.
  static constexpr int KS = (D == 128 ? 98304 : 65536) / K_TILE;
  static constexpr int VS = CALIB ? 0 : (D == 128 ? 81920 : 65536) / V_TILE;
  static constexpr int DQ = 16;              // decision ring depth
  static constexpr int MAXA = 4096;          // calibration: max off-frontier gate tiles per row
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_TILE;
  static constexpr int OFF_V = OFF_K + KS * K_TILE;
  static constexpr int OFF_CAL = OFF_V + VS * V_TILE;
  static constexpr int CAL_BYTES = CALIB ? MAXA * 4 : 0;
  static constexpr int OFF_BAR = OFF_CAL + CAL_BYTES;
  static constexpr int NUM_BARS = 1 + 2 * KS + 2 * VS + 2 * NS + 2 * DQ + 1 + 2 * NG;
  static constexpr int OFF_XCH = OFF_BAR + NUM_BARS * 8;  // votes u32 [NG][2][4], final (m,l) f32 [NG][128][2]
  static constexpr int XCH_BYTES = NG * 2 * 4 * 4 + NG * 128 * 8;
  static constexpr int OFF_DEC = OFF_XCH + XCH_BYTES;
  static constexpr int OFF_TMEMPTR = OFF_DEC + DQ * 4;
  static constexpr int SMEM_BYTES = OFF_TMEMPTR + 16 + 1024;  // + alignment slack
  // TMEM columns
  static constexpr int S_COL = CALIB ? 0 : NG * D;  // O_g at g*D
  static constexpr int TMEM_NEED = S_COL + NS * KT;
  static constexpr int TMEM_COLS = TMEM_NEED <= 128 ? 128 : (TMEM_NEED <= 256 ? 256 : 512);
  static constexpr int SOFTMAX_WARPS = 4 * NG;
  static constexpr int KPROD_WARP = SOFTMAX_WARPS;
  static constexpr int MMA_WARP = SOFTMAX_WARPS + 1;
  static constexpr int VPROD_WARP = SOFTMAX_WARPS + 2;
  static constexpr int NUM_THREADS = (SOFTMAX_WARPS + 3) * 32;
  static_assert(KT == 64 || KT == 128, "64- or 128-key tiles");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
  static_assert(TMEM_NEED <= 512, "TMEM budget");
  static_assert(NS >= 2, "at least one S slot per softmax group");
  static_assert(CALIB || VS >= 2, "V ring must hold two tiles");
  static_assert(DQ >= NS && DQ >= KS, "decision ring depth");
};

template <int D, int KT_, bool CALIB>
__global__ void __launch_bounds__(11 * 32, 1)
    bsfa_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v, const KernelParams p) {
  using C = KCfg<D, KT_, CALIB>;
  constexpr int KT = C::KT, KS = C::KS, VS = C::VS, NS = C::NS, DQ = C::DQ, NG = C::NG;
  constexpr int TPQ = 128 / KT;  // key tiles per query-block width

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
  uint64_t* o_quiet = o_full + 1;        // [NG] MMA commit: all issued MMAs landed (O_g may be rescaled)
  uint64_t* o_rescaled = o_quiet + NG;   // [NG] group g finished rescaling O_g
  volatile uint32_t* dec_words = reinterpret_cast<volatile uint32_t*>(smem + C::OFF_DEC);
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEMPTR);
  const uint32_t xch_vote = smem_u32(smem + C::OFF_XCH);  // u32 [NG][2][4] per-warp gate votes
  const uint32_t xch_fin = xch_vote + NG * 2 * 4 * 4;      // f32 [NG][128][2] final (m, l) per row

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
  // reachable key tiles: causal -> through the frontier (key tiles overlapping
  // the query rows, tiling.py:50-60); calibration -> the off-frontier prefix only
  const int ntiles = CALIB ? qi * TPQ : (p.causal ? (qi + 1) * TPQ : p.num_kv_tiles);
  const int fr_lo = qi * TPQ;  // first frontier tile

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
      mbar_init(&p_full[i], 4);  // the 4 warps of the owning group
    }
    for (int i = 0; i < DQ; ++i) {
      mbar_init(&dec_full[i], 1);
      mbar_init(&dec_empty[i], 1);
    }
    mbar_init(o_full, 1);
    for (int i = 0; i < NG; ++i) {
      mbar_init(&o_quiet[i], 1);
      mbar_init(&o_rescaled[i], 4);
    }
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
          const uint32_t keep = __shfl_sync(0xffffffffu, dec_words[di], 0);
          __syncwarp();
          mbar_arrive_w(&dec_empty[di]);
          if (keep) {
            const int slot = int(vcount % VS);
            mbar_wait(&v_empty[slot], uint32_t((vcount / VS) & 1) ^ 1u);
            mbar_arrive_expect_tx_w(&v_full[slot], C::V_TILE);
#pragma unroll
            for (int c = 0; c < C::NCH; ++c)
              tma_load_4d_w(sV + slot * C::V_TILE + c * KT * 128, &tm_v, &v_full[slot], c * 64, j * KT, g, b,
                            kEvictLast);
            ++vcount;
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
      const uint64_t dv0 = make_sdesc_sw128(smem_u32(sV), KT * 128, 1024);
      mbar_wait(bar_q, 0);

      auto issue_qk = [&](int t) {
        const int st = t % KS;
        mbar_wait(&k_full[st], (t / KS) & 1);
        if (p.trace && (int)blockIdx.x == p.trace_cta && lane == 0 && t < kTraceTiles)
          p.trace[kEvKReady * kTraceTiles + t] = clock64();
        tc_fence_after();
        const uint32_t d_tmem = tmem + C::S_COL + (t % NS) * KT;
        umma_qk_tile_w<D, KT>(d_tmem, dq0, dk0 + uint64_t((st * C::K_TILE) >> 4), IDESC_QK);
        umma_commit_w(&s_full[t % NS]);
        umma_commit_w(&k_empty[st]);
      };

      const int pre = ntiles < NS ? ntiles : NS;
      for (int t = 0; t < pre; ++t) issue_qk(t);

      unsigned long long vcount = 0;
      uint32_t o_started = 0;  // bit g: O_g holds a partial sum
      uint32_t n_rescale = 0;  // bit g: parity of group g's rescale hand-offs
      for (int j = 0; j < ntiles; ++j) {
        const int sb = j % NS;
        mbar_wait(&p_full[sb], (j / NS) & 1);
        const bool tr = p.trace && (int)blockIdx.x == p.trace_cta && lane == 0 && j < kTraceTiles;
        if (tr) p.trace[kEvPSeen * kTraceTiles + j] = clock64();
        if constexpr (!CALIB) {
          const int og = j % NG;
          const uint32_t word = __shfl_sync(0xffffffffu, dec_words[j % DQ], 0);
          const uint32_t keep = word & 1u;
          const uint32_t p_tmem = tmem + C::S_COL + sb * KT;
          if (word & kRescaleFlag) {
            // group og rescales O_og in TMEM: let every issued MMA land first,
            // and hold PV_j until the rescale is done (rare: max grew by > 2^8)
            umma_commit_w(&o_quiet[og]);
            mbar_wait(&o_rescaled[og], (n_rescale >> og) & 1);
            n_rescale ^= 1u << og;
            tc_fence_after();
          }
          if (keep) {
            const int slot = int(vcount % VS);
            mbar_wait(&v_full[slot], uint32_t((vcount / VS) & 1));
            if (tr) p.trace[kEvVReady * kTraceTiles + j] = clock64();
            ++vcount;
            tc_fence_after();
            const uint64_t dv = dv0 + uint64_t((slot * C::V_TILE) >> 4);
#pragma unroll
            for (int q = 0; q < KT / 64; ++q) {  // 64 keys per batch
              umma_pv64_w(tmem + og * D, p_tmem + q * 32, dv + uint64_t(q * 512), IDESC_PV, (o_started >> og) & 1u);
              o_started |= 1u << og;
            }
            umma_commit_w(&v_empty[slot]);
          }
          if (j == ntiles - 1) umma_commit_w(o_full);
        } else {
          tc_fence_after();
        }
        // QK_{j+NS} reuses slot sb; issued after PV_j, so its commit also
        // certifies that every earlier PV into O_{j mod NG} has landed.
        if (j + NS < ntiles) issue_qk(j + NS);
        if (tr) p.trace[kEvIssued * kTraceTiles + j] = clock64();
      }
    }
    __syncwarp();
  } else if (warp < C::SOFTMAX_WARPS) {
    // ======================= softmax groups =======================
    const int grp = warp >> 2;     // key tiles j = grp (mod NG)
    const int wq = warp & 3;
    const int r = wq * 32 + lane;  // row inside the query tile == TMEM lane
    const uint32_t lane_off = uint32_t(wq * 32) << 16;
    const uint32_t o_tm = tmem + lane_off + grp * D;  // this group's O slot
    const float sl2 = p.scale_log2;
    const uint32_t vote_base = xch_vote + grp * 2 * 4 * 4;

    float T = 0.f;
    if (!CALIB && p.gate_mode == kGateThreshold) {
      const int pos = qi < p.thr_positions - 1 ? qi : p.thr_positions - 1;
      T = p.thr[(long long)hq * p.thr_positions + pos];
    }

    constexpr bool kTurns = !CALIB && BSFA_TURNS;
    const uint32_t turn_mine = 5 + grp, turn_other = 5 + (grp ^ 1);
    if (kTurns && grp == 1) named_bar_arrive(turn_other, 256);  // group 0 goes first

    float m_ref = -INFINITY;  // raw (unscaled) reference max of this row over this group's kept tiles
    float l_sum = 0.f;        // row sum relative to m_ref
    bool o_valid = false;     // group-uniform: O_g holds data
    uint32_t n_rescale = 0;
    unsigned long long kept_tiles = 0;

    for (int j = grp; j < ntiles; j += NG) {
      const int sb = j % NS;
      const int use = j / NS;
      const uint32_t s_row = tmem + lane_off + C::S_COL + sb * KT;
      mbar_wait(&s_full[sb], use & 1);
      const bool tr = p.trace && (int)blockIdx.x == p.trace_cta && r == 0 && j < kTraceTiles;
      if (tr) p.trace[kEvSReady * kTraceTiles + j] = clock64();
      if (kTurns) named_bar_sync(turn_mine, 256);
      tc_fence_after();
      uint32_t sv[KT];
#pragma unroll
      for (int c = 0; c < KT; c += 32) tmem_ld32(s_row + c, &sv[c]);
      tmem_wait_ld();

      const bool frontier = (j >= fr_lo) && (j < fr_lo + TPQ);
      if (!CALIB) {
        if (frontier && p.causal) {
          const int off = (j - fr_lo) * KT;  // key - row offset inside the query block
#pragma unroll
          for (int c = 0; c < KT; ++c)
            if (off + c > r) sv[c] = __float_as_uint(-INFINITY);
        }
        if (!p.causal && (j + 1) * KT > p.valid_len) {
#pragma unroll
          for (int c = 0; c < KT; ++c)
            if (j * KT + c >= p.valid_len) sv[c] = __float_as_uint(-INFINITY);
        }
      }
      float rm;  // row max of the tile (one gate tile)
      {
        float m0 = fmaxf(__uint_as_float(sv[0]), __uint_as_float(sv[1]));
        float m1 = fmaxf(__uint_as_float(sv[2]), __uint_as_float(sv[3]));
        float m2 = fmaxf(__uint_as_float(sv[4]), __uint_as_float(sv[5]));
        float m3 = fmaxf(__uint_as_float(sv[6]), __uint_as_float(sv[7]));
#pragma unroll
        for (int c = 8; c < KT; c += 8) {
          m0 = fmaxf(m0, fmaxf(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])));
          m1 = fmaxf(m1, fmaxf(__uint_as_float(sv[c + 2]), __uint_as_float(sv[c + 3])));
          m2 = fmaxf(m2, fmaxf(__uint_as_float(sv[c + 4]), __uint_as_float(sv[c + 5])));
          m3 = fmaxf(m3, fmaxf(__uint_as_float(sv[c + 6]), __uint_as_float(sv[c + 7])));
        }
        rm = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
      }

      if constexpr (CALIB) {
        {
          float m = rm;
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
          if (lane == 0) atomicMax(&cvals[j], float_to_ordered(m * p.scale));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sb]);
        continue;
      } else {
        // ---- gate: OR over the group's 128 rows of (rowmax * scale > T)
        // one group-wide exchange per tile: gate vote (bit 0) and a rescale
        // request (bit 1: this row's max outgrows the running reference)
        const bool gvote = p.gate_mode == kGateThreshold && rm * p.scale > T;
        const bool rreq = o_valid && rm > m_ref + p.rescale_raw;
        const uint32_t wv = (__ballot_sync(0xffffffffu, gvote) != 0u ? 1u : 0u) |
                            (__ballot_sync(0xffffffffu, rreq) != 0u ? 2u : 0u);
        const uint32_t par = use & 1;
        if (lane == 0) sts_u32(vote_base + (par * 4 + wq) * 4, wv);
        named_bar_sync(1 + grp, 128);
        const uint4 v4 = lds_u128(vote_base + par * 4 * 4);
        const uint32_t vw = v4.x | v4.y | v4.z | v4.w;
        uint32_t bits;
        if (frontier || p.gate_mode == kGateDense) {
          bits = 1u;
        } else if (p.gate_mode == kGateFrontier) {
          bits = 0;
        } else {
          bits = vw & 1u;
        }
        const bool do_rescale = bits && (vw & 2u);
        if (tr) p.trace[kEvVoted * kTraceTiles + j] = clock64();
        if (r == 0) {
          const int di = j % DQ;
          mbar_wait(&dec_empty[di], ((j / DQ) & 1) ^ 1);
          dec_words[di] = bits | (do_rescale ? kRescaleFlag : 0u);
          mbar_arrive(&dec_full[di]);
          kept_tiles += bits;
          if (p.decisions) {
            int8_t* drow = p.decisions + (((long long)b * p.heads_q + hq) * p.num_q_tiles + qi) * p.gate_cols;
            drow[j] = frontier ? int8_t(2) : (bits ? int8_t(3) : int8_t(1));
          }
        }
        if (bits == 0) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[sb]);
          if (tr) p.trace[kEvPDone * kTraceTiles + j] = clock64();
          if (kTurns && j + 1 < ntiles) named_bar_arrive(turn_other, 256);
          continue;
        }

        const float m_new = fmaxf(m_ref, rm);
        float alpha = 1.f;
        if (!o_valid) {
          m_ref = m_new;
        } else if (do_rescale && m_new > m_ref + p.rescale_raw) {
          alpha = ex2_approx((m_ref - m_new) * sl2);
          m_ref = m_new;
        }

        // P = exp2(s * scale*log2e - m * scale*log2e), bf16-packed over the S slot
        const float neg = (m_ref == -INFINITY) ? 0.f : -m_ref * sl2;
        const uint64_t sl2x2 = f2_pack(sl2, sl2);
        const uint64_t negx2 = f2_pack(neg, neg);
        uint64_t acc0 = 0, acc1 = 0;
#pragma unroll
        for (int cb = 0; cb < KT; cb += 32) {
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 32; c += 4) {
            const int e = cb + c;
            const uint64_t x0 = ffma2(f2_pack(__uint_as_float(sv[e]), __uint_as_float(sv[e + 1])), sl2x2, negx2);
            const uint64_t x1 =
                ffma2(f2_pack(__uint_as_float(sv[e + 2]), __uint_as_float(sv[e + 3])), sl2x2, negx2);
            const float p0 = ex2_approx(f2_lo(x0)), p1 = ex2_approx(f2_hi(x0));
            float p2, p3;
            // offload part of the exponentials from the MUFU to the FMA pipe
            if (BSFA_EXP_EMU == 2 || (BSFA_EXP_EMU == 1 && ((c >> 2) & 1))) {
              const uint64_t e1 = exp2_poly_x2(x1);
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
          tmem_st16(s_row + cb / 2, pk);
        }
        const uint64_t acc = fadd2(acc0, acc1);
        l_sum = l_sum * alpha + (f2_lo(acc) + f2_hi(acc));

        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sb]);
        if (tr) p.trace[kEvPDone * kTraceTiles + j] = clock64();
        if (kTurns && j + 1 < ntiles) named_bar_arrive(turn_other, 256);
        if (do_rescale) {
          // hand-off with the MMA warp: wait until every issued MMA (incl. the
          // group's previous PV) has landed, rescale O_grp, release PV_j
          mbar_wait(&o_quiet[grp], n_rescale & 1);
          ++n_rescale;
          tc_fence_after();
          const uint64_t ax2 = f2_pack(alpha, alpha);
#pragma unroll
          for (int c = 0; c < D; c += 32) {
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
          if (lane == 0) mbar_arrive(&o_rescaled[grp]);
        }
        o_valid = true;
      }
    }

    if constexpr (CALIB) {
      // ---- order statistics of this row of tile maxima (calibration.py:116-153)
      constexpr int NTHR = 128 * NG;
      const int A = ntiles;
      const int t = grp * 128 + r;
      named_bar_sync(3, NTHR);
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
          named_bar_sync(3, NTHR);
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
      // ---- epilogue: merge the two groups' (m, l, O) and normalise
      //      (engine.py:178-182: O = O~/l, lse = m*scale + ln l)
      sts_f32(xch_fin + (grp * 128 + r) * 8, m_ref);
      sts_f32(xch_fin + (grp * 128 + r) * 8 + 4, l_sum);
      mbar_wait(o_full, 0);
      tc_fence_after();
      named_bar_sync(3, 128 * NG);
      float mg[NG], lg[NG];
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        mg[q] = lds_f32(xch_fin + (q * 128 + r) * 8);
        lg[q] = lds_f32(xch_fin + (q * 128 + r) * 8 + 4);
      }
      float m_all = -INFINITY;
#pragma unroll
      for (int q = 0; q < NG; ++q)
        if (lg[q] > 0.f) m_all = fmaxf(m_all, mg[q]);
      float wgt[NG];
      float l_all = 0.f;
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        wgt[q] = lg[q] > 0.f ? ex2_approx((mg[q] - m_all) * sl2) : 0.f;
        l_all += lg[q] * wgt[q];
      }
      const float inv_l = 1.f / l_all;
      bool bad = !(l_all > 0.f);
      constexpr int DH = D / NG;  // output columns written by this thread
      const int row = qi * 128 + r;
      __nv_bfloat16* orow =
          p.o + (long long)b * p.o_sb + (long long)hq * p.o_sh + (long long)row * p.o_sn + grp * DH;
#pragma unroll
      for (int c = 0; c < DH; c += 32) {
        float acc[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) acc[e] = 0.f;
#pragma unroll
        for (int q = 0; q < NG; ++q) {
          if (lg[q] > 0.f) {  // an O slot nobody accumulated into holds garbage
            uint32_t ov[32];
            tmem_ld32(tmem + lane_off + q * D + grp * DH + c, ov);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) acc[e] = fmaf(__uint_as_float(ov[e]), wgt[q], acc[e]);
          }
        }
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float a0 = acc[e] * inv_l, a1 = acc[e + 1] * inv_l;
          if (p.inject_fault && qi == 0 && r == 0 && grp == 0 && c == 0 && e == 0) a0 += 1.0f;  // O[0][0] += 1
          bad |= !isfinite(a0) || !isfinite(a1);
          pk[e / 2] = pack_bf16x2(a0, a1);
        }
        uint4* dst = reinterpret_cast<uint4*>(orow + c);
#pragma unroll
        for (int e = 0; e < 4; ++e) dst[e] = make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
      }
      if (grp == 0) p.lse[((long long)b * p.heads_q + hq) * p.seq_len + row] = m_all * p.scale + logf(l_all);
      if (bad && p.status) atomicOr(p.status, 1);
      if (r == 0 && p.counters) {
        if (grp == 0) atomicAdd(&p.counters[0], (unsigned long long)ntiles);
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
