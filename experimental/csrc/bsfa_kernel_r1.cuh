// BSFA forward (K1) and calibration block-max (K2) kernels for sm_100a.
//
// One CTA owns NQ query tiles (128 rows each) of the same query block i:
// NQ = 2 q heads of one GQA group (they share every K/V tile, and their
// causal extents are identical), NQ = 1 when the group size is odd.  The CTA
// streams the reachable keys of the kv head in steps of 128 keys; one step is
// one 128-key QK^T MMA tile holding GT = 128 / b_n gate tiles (the
// reference's b_n-wide blocks, tiling.py:19-69).
//
// Warp roles:
//   warps 4s..4s+3   softmax group s (query tile s): thread r owns row r
//                    (TMEM lane r) over all 128 keys of a step
//   warp 4*NQ        TMA producer: Q once, K every step (unconditional)
//   warp 4*NQ+1      tcgen05 issuer (warp-convergent, one elected lane) + TMEM owner
//   warp 4*NQ+2      TMA producer for V: a V gate tile is fetched only once some
//                    query tile of the CTA kept it (first keep loads it, the
//                    other tile reuses it); skipped by every tile => never loaded
// TMEM (512 columns): O_s (fp32, d columns) and S_s (fp32, 128 columns) per
// query tile; P_s (bf16) is written over the first 64 columns of S_s and read
// by the PV MMA from TMEM.
//
// MMA issue order (ping-pong, tensor pipe executes in order):
//   QK_0(0) QK_1(0) | PV_0(0) QK_0(1) | PV_1(0) QK_1(1) | PV_0(1) QK_0(2) | ...
// so the tensor core works on one tile's PV/QK while the other tile's softmax
// runs.  S_s(j) being committed certifies that PV_s(j-1) has landed, so the
// softmax may rescale O_s in place before releasing P_s(j).
//
// Per step j and query tile s:
//   QK:   S = Q_s K_j^T                tcgen05.mma 128 x 128 x 16 (SS), K = d
//   gate: per gate tile h, OR over the 128 rows of (rowmax * scale > T) == the
//         reference's tile.s_max > T (gates.py:77-78, engine.py:30-38)
//   skip: no V TMA (unless the other tile kept it), no exp, no PV MMA, no
//         statistics update (engine.py:172-174)
//   keep: online softmax (engine.py:57-68) with lazily rescaled O_s,
//         O_s += P_h V_(j,h)              tcgen05.mma 128 x d x 16 (TS)
// Calibration (CALIB) runs the same QK front end over the off-frontier prefix
// (steps j < i, calibration.py:108-115) and reduces gate-tile maxima in smem.
#pragma once

#include "ptx.cuh"

// Fraction of exponentials computed by polynomial on the FMA pipe instead of
// the MUFU: 0 = none, 1 = 1/4, 2 = 1/2.  With P's second half in shared memory
// the softmax is issue-bound, not MUFU-bound: 0 measured fastest (l32k 6.23 ms
// vs 6.34 at 1/4 and 7.16 at 1/2).
#ifndef BSFA_EXP_EMU
#define BSFA_EXP_EMU 0
#endif
// Order the polynomial exponentials after the same group's MUFU exponentials.
#ifndef BSFA_EXP_CHAIN
#define BSFA_EXP_CHAIN 1
#endif
// Turn-taking between the two query tiles' softmax groups (NQ = 2): 0 = free
// running, 1 = the exponential phases alternate, 2 = whole steps alternate.
#ifndef BSFA_TURN
#define BSFA_TURN 0
#endif
// P of the second 64-key half in shared memory (PV from SMEM) instead of TMEM:
// the next QK of a tile is issued right after the PV of the first half, so it
// overlaps the second half's exponentials (S/P no longer alias across a step).
#ifndef BSFA_P_SMEM
#define BSFA_P_SMEM 1
#endif
// One tcgen05 issuer warp per query tile (the otherwise idle warp issues for
// tile 1), V in fixed slots per (step, gate tile): a tile's MMAs never wait
// behind the other tile's barriers.
#ifndef BSFA_SPLIT_ISSUE
#define BSFA_SPLIT_ISSUE 0
#endif
// Debug timeline (bsfa_debug_trace); compiled out of the production library.
#ifndef BSFA_TRACE
#define BSFA_TRACE 0
#endif

namespace bsfa {

enum : int { kGateThreshold = 0, kGateDense = 1, kGateFrontier = 2, kGateWindow = 3, kGateRunMax = 4 };
// static decision of a step (known to every role without the softmax)
enum : int { kStepDynamic = 0, kStepAll = 1, kStepNone = 2 };

struct KernelParams {
  int batch, heads_q, heads_kv, group;
  int seq_len;       // padded sequence length (multiple of 128)
  int valid_len;     // unpadded length (non-causal key masking)
  int num_q_tiles;   // seq_len / 128
  int num_steps;     // seq_len / 128 (128-key MMA steps)
  int gate_cols;     // seq_len / b_n
  int causal;
  int gate_mode;
  int thr_positions;
  float scale;
  float scale_log2;
  float rescale_raw;  // lazy-rescale threshold in raw score units
  int inject_fault;
  int gate_window;     // kGateWindow: trailing window in tokens (gates.py:81-98)
  float gate_lambda;   // kGateRunMax: lambda (gates.py:101-118)
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
  // debug: per-step clock64 timestamps of one CTA (bsfa_debug_trace)
  long long* trace;
  int trace_cta;
  // NQ = 2 forward with an odd GQA group (or MHA): the two query tiles are query
  // blocks 2m+1 and 2m of ONE q head instead of two q heads of one block
  int block_pair;
  // extra O destinations (peer GPUs' gathered-O buffers), same element offsets
  int num_o_peers;
  __nv_bfloat16* o_peer[7];
};

// 16 packed bf16x2 words (32 O elements of one row) -> O and every peer copy
__device__ __forceinline__ void store_o32(const KernelParams& p, long long off, const uint32_t* pk) {
  const uint4 w0 = make_uint4(pk[0], pk[1], pk[2], pk[3]), w1 = make_uint4(pk[4], pk[5], pk[6], pk[7]);
  const uint4 w2 = make_uint4(pk[8], pk[9], pk[10], pk[11]), w3 = make_uint4(pk[12], pk[13], pk[14], pk[15]);
  uint4* dst = reinterpret_cast<uint4*>(p.o + off);
  dst[0] = w0, dst[1] = w1, dst[2] = w2, dst[3] = w3;
  for (int i = 0; i < p.num_o_peers; ++i) {
    uint4* pd = reinterpret_cast<uint4*>(p.o_peer[i] + off);
    pd[0] = w0, pd[1] = w1, pd[2] = w2, pd[3] = w3;
  }
}

// trace slots: trace[(ev * 2 + s) * kTraceSteps + j]
constexpr int kTraceSteps = 2048;
enum : int { kEvSReady = 0, kEvVoted = 1, kEvPDone = 2, kEvPSeen = 3, kEvVReady = 4, kEvIssued = 5, kEvLdDone = 6, kEvExpDone = 7 };

template <int D, int GT, int NQ, bool CALIB, int TPR = 1>
struct KCfg {
  static constexpr int BN = 128 / GT;        // gate tile width (reference b_n)
  static constexpr int NCH = D / 64;         // 128-byte swizzle atoms along head_dim
  static constexpr int Q_TILE = 128 * D * 2;
  static constexpr int K_TILE = 128 * D * 2;  // one 128-key step
  static constexpr int V_UNIT = BN * D * 2;   // one gate tile of V
#ifndef BSFA_K_STAGES
#define BSFA_K_STAGES 3
#endif
#ifndef BSFA_V_BYTES
#define BSFA_V_BYTES 65536
#endif
  // second-half P in shared memory (forward, one thread per row)
  static constexpr bool PSM = !CALIB && TPR == 1 && BSFA_P_SMEM != 0;
  static constexpr int P_TILE = PSM ? 128 * 128 : 0;  // 128 rows x 64 keys bf16 per query tile
  static constexpr int KS = D == 128 ? (PSM ? 2 : BSFA_K_STAGES) : 3;
  static constexpr bool SPLIT = PSM && BSFA_SPLIT_ISSUE != 0;  // one issuer warp per query tile
  static constexpr int VS = CALIB ? 0 : (D == 128 ? BSFA_V_BYTES : 65536) / V_UNIT;
#ifndef BSFA_DQ
#define BSFA_DQ 4
#endif
  static constexpr int DQ = BSFA_DQ;          // decision ring depth (dynamic steps)
  static constexpr int MAXA = 4096;           // calibration: max off-frontier gate tiles per row
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + NQ * Q_TILE;
  static constexpr int OFF_V = OFF_K + KS * K_TILE;
  static constexpr int OFF_P = OFF_V + VS * V_UNIT;
  static constexpr int OFF_CAL = OFF_P + NQ * P_TILE;
  static constexpr int CAL_BYTES = CALIB ? NQ * MAXA * 4 : 0;
  static constexpr int OFF_BAR = OFF_CAL + CAL_BYTES;
  static constexpr int NUM_BARS = 1 + 2 * KS + 2 * VS + 4 * NQ + 2 * NQ * DQ + NQ;
  // per query tile: per-warp gate votes u32 [2 parity][4 warps]
  // per query tile (TPR = 2): half-row maxima f32 [2 parity][2 halves][128],
  // then the epilogue row sums f32 [2 halves][128]
  static constexpr int XCH_TILE = TPR == 2 ? (2 * 2 * 128 + 2 * 128) * 4 : 2 * 4 * 4;
  static constexpr int OFF_XCH = (OFF_BAR + NUM_BARS * 8 + 15) / 16 * 16;  // 16-B aligned: votes read as v4
  static constexpr int OFF_DEC = OFF_XCH + NQ * XCH_TILE;   // u32 [NQ][DQ] decision ring (V producer)
  static constexpr int OFF_DECM = OFF_DEC + NQ * DQ * 4;    // u32 [NQ] decision of the current step (MMA)
  static constexpr int OFF_TMEMPTR = OFF_DECM + NQ * 4;
  static constexpr int SMEM_BYTES = OFF_TMEMPTR + 16 + 1024;  // + alignment slack
  // TMEM columns
  static constexpr int O_COL = 0;                          // O_s at s * D
  static constexpr int S_COL = CALIB ? 0 : NQ * D;         // S_s at S_COL + s * 128
  // calibration has no O: S is double-buffered per query tile, S_{s,b} at (2s + b) * 128
  static constexpr int TMEM_NEED = CALIB ? NQ * 256 : S_COL + NQ * 128;
  static constexpr int TMEM_COLS = TMEM_NEED <= 128 ? 128 : (TMEM_NEED <= 256 ? 256 : 512);
  // one thread per row: warpgroup s is query tile s; the last warpgroup holds
  // the K producer, the MMA issuer, the V producer and one idle warp
  // TPR threads per row: warpgroup s*TPR + h owns key half h of query tile s
  static constexpr int SOFTMAX_WARPS = 4 * NQ * TPR;
  static constexpr int KPROD_WARP = SOFTMAX_WARPS;
  static constexpr int MMA_WARP = SOFTMAX_WARPS + 1;
  static constexpr int VPROD_WARP = SOFTMAX_WARPS + 2;
  static constexpr int NUM_THREADS = (SOFTMAX_WARPS + 4) * 32;
  // register split (setmaxnreg): softmax warps hold a 128-column score row,
  // its exponentials and the packed P row
  // The setmaxnreg pool is what the CTA was launched with: NUM_THREADS x the
  // launch-bound register count (65536 / NUM_THREADS, multiple of 8, <= 255).
  // Growing the softmax warps beyond pool - 128 x REG_OTHER would block forever.
  static constexpr int REG_LAUNCH = (65536 / NUM_THREADS) / 8 * 8 > 248 ? 248 : (65536 / NUM_THREADS) / 8 * 8;
  static constexpr int REG_OTHER = TPR == 2 ? 32 : 56;
  static constexpr int REG_SOFT_MAX = (NUM_THREADS * REG_LAUNCH - 128 * REG_OTHER) / (SOFTMAX_WARPS * 32) / 8 * 8;
  static constexpr int REG_SOFT = REG_SOFT_MAX > 248 ? 248 : REG_SOFT_MAX;
  static_assert(REG_SOFT >= REG_LAUNCH && REG_OTHER <= REG_LAUNCH, "register split");
  static constexpr bool SPLIT_REGS = true;
  static_assert(GT == 1 || GT == 2, "b_n in {64, 128}");
  static_assert(NQ == 1 || NQ == 2, "one or two query tiles per CTA");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
  static_assert(TMEM_NEED <= 512, "TMEM budget");
  static_assert(CALIB || VS >= 2 * GT, "V ring must hold two steps");
};

// Statically known decision bits (bit x = gate tile x of the step) of step j,
// or -1 when the step is decided by a vote over its scores.  Identical in
// every role, so the V producer can prefetch static keeps without a vote.
template <int GT>
__device__ __forceinline__ int step_static_bits(int gate_mode, int window, int j, int qi) {
  constexpr int kAll = (1 << GT) - 1;
  if (j == qi || gate_mode == kGateDense) return kAll;  // frontier (tiling.py:50-60) / DenseGate
  if (gate_mode == kGateFrontier) return 0;             // FrontierOnlyGate
  if (gate_mode == kGateWindow) {
    // SlidingWindowGate (gates.py:96-98): keep gate tile g iff its key range
    // intersects [i*b_m - w, (i+1)*b_m)
    constexpr int BN = 128 / GT;
    int bits = 0;
#pragma unroll
    for (int x = 0; x < GT; ++x) {
      const int gc = j * GT + x;
      if ((gc + 1) * BN > qi * 128 - window && gc * BN < (qi + 1) * 128) bits |= 1 << x;
    }
    return bits;
  }
  return -1;  // ThresholdGate / RunningMaxGate: voted
}

template <int D, int GT, int NQ, bool CALIB, int TPR = 1>
__global__ void __launch_bounds__(KCfg<D, GT, NQ, CALIB, TPR>::NUM_THREADS, 1)
    bsfa_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v, const KernelParams p) {
  using C = KCfg<D, GT, NQ, CALIB, TPR>;
  static_assert(TPR == 1 || (TPR == 2 && !CALIB), "two threads per row: forward only");
  constexpr int BN = C::BN, KS = C::KS, VS = C::VS, DQ = C::DQ;

  extern __shared__ uint8_t smem_raw[];
  // all shared-memory addresses are 32-bit shared-window offsets computed once
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = opaque_u32((sraw + 1023u) & ~1023u);
  uint8_t* smem = smem_raw + (sbase - sraw);
  const uint32_t sQ = sbase + C::OFF_Q;
  const uint32_t sK = sbase + C::OFF_K;
  const uint32_t sV = sbase + C::OFF_V;
  const uint32_t sP = sbase + C::OFF_P;
  int* cvals = reinterpret_cast<int*>(smem + C::OFF_CAL);
  // mbarriers (8 bytes each)
  const uint32_t bar_q = sbase + C::OFF_BAR;
  const uint32_t k_full = bar_q + 8;              // [KS]
  const uint32_t k_empty = k_full + 8 * KS;       // [KS]
  const uint32_t v_full = k_empty + 8 * KS;       // [VS]
  const uint32_t v_empty = v_full + 8 * VS;       // [VS]
  const uint32_t s_full = v_empty + 8 * VS;       // [NQ] QK_s(j) landed (and every earlier MMA)
  const uint32_t p_full = s_full + 8 * NQ;        // [NQ][2] P half written (half 0 also: O_s rescaled)
  const uint32_t o_full = p_full + 16 * NQ;       // [NQ] last PV_s landed
  const uint32_t dec_full = o_full + 8 * NQ;      // [NQ][DQ]
  const uint32_t dec_empty = dec_full + 8 * NQ * DQ;
  const uint32_t pv_done = dec_empty + 8 * NQ * DQ;  // [NQ] PSM: second-half PV_s(j) landed (P buffer free)
  const uint32_t xch_sm = sbase + C::OFF_XCH;
  const uint32_t dec_sm = sbase + C::OFF_DEC;
  const uint32_t decm_sm = sbase + C::OFF_DECM;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEMPTR);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- work unit: (batch, kv head) major, heaviest query block first, the
  //      head pairs of the GQA group minor (every pair reads the same K/V)
  // per query tile s: query block qi_a[s], q head hq_a[s], steps ns_a[s]
  const bool bpair = NQ == 2 && p.block_pair != 0;
  int qi_a[NQ], hq_a[NQ], ns_a[NQ];
  int b_, g_, qi_, hq0_;
  {
    const int unit = blockIdx.x;
    if (bpair) {
      // query blocks 2m+1 and 2m of one q head (heaviest first); they share K/V
      // up to the shorter tile's frontier, tile 1 simply stops one step earlier
      const int per_bg = ((p.num_q_tiles + 1) / 2) * p.group;
      const int bg = unit / per_bg;
      const int rem = unit - bg * per_bg;
      const int m = rem / p.group;
      b_ = bg / p.heads_kv;
      g_ = bg - b_ * p.heads_kv;
      qi_ = p.num_q_tiles - 1 - 2 * m;
      hq0_ = g_ * p.group + (rem - m * p.group);
      qi_a[0] = qi_;
      qi_a[NQ - 1] = qi_ - 1;  // -1: no second block (odd block count)
      hq_a[0] = hq_a[NQ - 1] = hq0_;
    } else {
      const int pairs = p.group / NQ;
      const int per_bg = p.num_q_tiles * pairs;
      const int bg = unit / per_bg;
      const int rem = unit - bg * per_bg;
      qi_ = p.num_q_tiles - 1 - rem / pairs;
      const int pr = rem - (rem / pairs) * pairs;
      b_ = bg / p.heads_kv;
      g_ = bg - b_ * p.heads_kv;
      hq0_ = g_ * p.group + pr * NQ;  // q head of query tile s = hq0 + s
#pragma unroll
      for (int t = 0; t < NQ; ++t) {
        qi_a[t] = qi_;
        hq_a[t] = hq0_ + t;
      }
    }
  }
  const int b = b_, g = g_, qi = qi_, hq0 = hq0_;
  // 128-key steps: causal -> through the frontier step i; calibration -> the
  // off-frontier prefix only (calibration.py:110-113)
  const int nsteps = CALIB ? qi : (p.causal ? qi + 1 : p.num_steps);
#pragma unroll
  for (int t = 0; t < NQ; ++t)
    ns_a[t] = qi_a[t] < 0 ? 0 : (CALIB ? qi_a[t] : (p.causal ? qi_a[t] + 1 : p.num_steps));
  const int gate_mode = p.gate_mode;
  const int window = p.gate_window;
  const bool causal = p.causal != 0;
  const int valid_len = p.valid_len;
  const bool tr_cta = BSFA_TRACE && p.trace && (int)blockIdx.x == p.trace_cta;

  // ---- setup
  if (warp == C::KPROD_WARP && lane == 0) {
    mbar_init(bar_q, 1);
    for (int i = 0; i < KS; ++i) {
      mbar_init((k_full + 8 * (i)), 1);
      mbar_init((k_empty + 8 * (i)), C::SPLIT ? NQ : 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init((v_full + 8 * (i)), 1);
      mbar_init((v_empty + 8 * (i)), C::SPLIT ? NQ : 1);
    }
    for (int s = 0; s < NQ; ++s) {
      mbar_init((s_full + 8 * (s)), 1);
      mbar_init((p_full + 8 * (2 * s)), 4);  // the 4 softmax warps of query tile s (of half h, TPR = 2)
      mbar_init((p_full + 8 * (2 * s + 1)), 4);
      mbar_init((o_full + 8 * (s)), 1);
    }
    for (int i = 0; i < NQ * DQ; ++i) {
      mbar_init((dec_full + 8 * (i)), 1);
      mbar_init((dec_empty + 8 * (i)), 1);
    }
    for (int s = 0; s < NQ; ++s) mbar_init((pv_done + 8 * (s)), 1);
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
  // ---- split issue (C::SPLIT): the tcgen05 work of query tile s, issued by its own warp
  auto split_issue = [&](int s) {
    constexpr uint32_t IDESC_QK = make_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t IDESC_PV = make_idesc_bf16(128, D, 0, 1);
    const uint64_t dq0 = make_sdesc_sw128(sQ, 16, 1024);
    const uint64_t dk0 = make_sdesc_sw128(sK, 16, 1024);
    const uint64_t dv0 = make_sdesc_sw128(sV, BN * 128, 1024);
    const uint64_t dp0 = make_sdesc_sw128(sP, 16, 1024);
    mbar_wait(bar_q, 0);
    auto issue_qk = [&](int j) {
      const int st = j % KS;
      mbar_wait((k_full + 8 * (st)), (j / KS) & 1);
      tc_fence_after();
      umma_qk_tile_w<D, 128>(tmem + C::S_COL + s * 128, dq0 + uint64_t((s * C::Q_TILE) >> 4),
                             dk0 + uint64_t((st * C::K_TILE) >> 4), IDESC_QK);
      umma_commit_w((k_empty + 8 * (st)));  // one of NQ releases of the stage
      umma_commit_w((s_full + 8 * (s)));
    };
    issue_qk(0);
    uint32_t use_par = 0;  // bit slot: v_full phase (one phase per use of the slot)
    uint32_t p1_par = 0;
    bool o_started = false;
    for (int j = 0; j < nsteps; ++j) {
      const int sb = step_static_bits<GT>(gate_mode, window, j, qi);
      mbar_wait((p_full + 8 * (2 * s)), j & 1);
      tc_fence_after();
      const uint32_t bits = sb >= 0 ? uint32_t(sb) : lds_u32(decm_sm + s * 4);
      uint32_t rd = 0;  // gate tiles whose V this tile reads this step
      if (bits & 1u) {
        const int slot = (GT * j) % VS;
        mbar_wait((v_full + 8 * (slot)), (use_par >> slot) & 1u);
        tc_fence_after();
        umma_pv64_w(tmem + C::O_COL + s * D, tmem + C::S_COL + s * 128, dv0 + uint64_t((slot * C::V_UNIT) >> 4),
                    IDESC_PV, o_started ? 1u : 0u);
        o_started = true;
        rd |= 1u;
      }
      if (j + 1 < nsteps) issue_qk(j + 1);  // S_s is free once P half 0 is consumed
      constexpr int x1 = GT == 2 ? 1 : 0;
      if ((bits >> x1) & 1u) {
        mbar_wait((p_full + 8 * (2 * s + 1)), p1_par & 1u);  // released for kept second halves only
        p1_par ^= 1u;
        const int slot = (GT * j + x1) % VS;
        if (GT == 2) mbar_wait((v_full + 8 * (slot)), (use_par >> slot) & 1u);
        tc_fence_after();
        umma_pv64_ss_w(tmem + C::O_COL + s * D, dp0 + uint64_t((s * C::P_TILE) >> 4),
                       dv0 + uint64_t((slot * C::V_UNIT) >> 4) + uint64_t(GT == 1 ? 512 : 0), IDESC_PV,
                       o_started ? 1u : 0u);
        o_started = true;
        rd |= 1u << x1;
      }
      umma_commit_w((pv_done + 8 * (s)));
      if (j == nsteps - 1) umma_commit_w((o_full + 8 * (s)));
      // hand this step's V slots back (after the producer announced them)
#pragma unroll
      for (int h = 0; h < GT; ++h) {
        const int slot = (GT * j + h) % VS;
        if ((rd >> h) & 1u) {
          umma_commit_w((v_empty + 8 * (slot)));
        } else {
          mbar_wait((v_full + 8 * (slot)), (use_par >> slot) & 1u);
          mbar_arrive_w((v_empty + 8 * (slot)));
        }
        use_par ^= 1u << slot;
      }
    }
  };
  // Register split: setmaxnreg inside each role (the regions must not merge,
  // or ptxas allocates the merged code at the smaller budget).  Every role
  // leaves through bsfa_role_exit: arrive on the teardown barrier; the MMA
  // warp waits for everyone there and frees TMEM.
  if (warp == C::KPROD_WARP) {
    if constexpr (C::SPLIT_REGS) setmaxnreg_dec<C::REG_OTHER>();
    // ======================= TMA producer: Q, K (warp-convergent, one elected issuer)
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
          tma_load_4d_w(sQ + s * C::Q_TILE + c * 128 * 128, &tm_q, bar_q, c * 64, (qi_a[s] < 0 ? 0 : qi_a[s]) * 128,
                        hq_a[s], b, kEvictFirst);
      for (int j = 0; j < nsteps; ++j) {
        const int st = j % KS;
        mbar_wait((k_empty + 8 * (st)), ((j / KS) & 1) ^ 1);
        mbar_arrive_expect_tx_w((k_full + 8 * (st)), C::K_TILE);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_4d_w(sK + st * C::K_TILE + c * 128 * 128, &tm_k, (k_full + 8 * (st)), c * 64, j * 128, g, b, kEvictLast);
      }
    }
    __syncwarp();
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  } else if (warp == C::VPROD_WARP) {
    if constexpr (C::SPLIT_REGS) setmaxnreg_dec<C::REG_OTHER>();
    // ======================= TMA producer: V gate tiles kept by some query tile =========
    if constexpr (!CALIB) {
      if (nsteps > 0) {
        if (lane == 0) tma_prefetch_desc(&tm_v);
        unsigned vcount = 0, dn = 0;
        if constexpr (C::SPLIT) {
          // fixed slot per (step, gate tile); every use of a slot is announced on
          // v_full (with the data, or empty), so both issuers track its phase alone
          uint32_t use_par = 0;
          auto use_slot = [&](int j, int h, bool load) {
            const int slot = (GT * j + h) % VS;
            mbar_wait((v_empty + 8 * (slot)), ((use_par >> slot) & 1u) ^ 1u);
            use_par ^= 1u << slot;
            if (load) {
              mbar_arrive_expect_tx_w((v_full + 8 * (slot)), C::V_UNIT);
#pragma unroll
              for (int c = 0; c < C::NCH; ++c)
                tma_load_4d_w(sV + slot * C::V_UNIT + c * BN * 128, &tm_v, (v_full + 8 * (slot)), c * 64,
                              j * 128 + h * BN, g, b, kEvictLast);
              ++vcount;
            } else {
              mbar_arrive_w((v_full + 8 * (slot)));
            }
          };
          for (int j = 0; j < nsteps; ++j) {
            const int sb = step_static_bits<GT>(gate_mode, window, j, qi);
            uint32_t done = 0;
            if (sb >= 0) {
#pragma unroll
              for (int h = 0; h < GT; ++h) use_slot(j, h, (sb >> h) & 1);
              continue;
            }
            const int di = int(dn % DQ);
            const uint32_t ph = (dn / DQ) & 1;
#pragma unroll
            for (int s = 0; s < NQ; ++s) {
              mbar_wait((dec_full + 8 * (s * DQ + di)), ph);
              const uint32_t w = lds_u32(dec_sm + (s * DQ + di) * 4);
              __syncwarp();
              mbar_arrive_w((dec_empty + 8 * (s * DQ + di)));
#pragma unroll
              for (int h = 0; h < GT; ++h)
                if (((w & ~done) >> h) & 1u) use_slot(j, h, true);
              done |= w;
            }
#pragma unroll
            for (int h = 0; h < GT; ++h)
              if (!((done >> h) & 1u)) use_slot(j, h, false);
            ++dn;
          }
        } else {
        auto load_unit = [&](int j, int h) {
          const int slot = int(vcount % VS);
          mbar_wait((v_empty + 8 * (slot)), ((vcount / VS) & 1) ^ 1);
          mbar_arrive_expect_tx_w((v_full + 8 * (slot)), C::V_UNIT);
#pragma unroll
          for (int c = 0; c < C::NCH; ++c)
            tma_load_4d_w(sV + slot * C::V_UNIT + c * BN * 128, &tm_v, (v_full + 8 * (slot)), c * 64, j * 128 + h * BN, g, b,
                          kEvictLast);
          ++vcount;
        };
        unsigned dn_a[NQ] = {};  // dynamic steps consumed per query tile
        for (int j = 0; j < nsteps; ++j) {
          // query tile 0's keeps are fetched as soon as its decision is known
          // (statically or by its vote); the tiles only tile 1 keeps follow its
          // decision (same order in the MMA warp)
          uint32_t prev = 0;
#pragma unroll
          for (int s = 0; s < NQ; ++s) {
            if (j >= ns_a[s]) continue;
            const int sbs = step_static_bits<GT>(gate_mode, window, j, qi_a[s]);
            uint32_t w;
            if (sbs >= 0) {
              w = uint32_t(sbs);
            } else {
              const int di = int(dn_a[s] % DQ);
              mbar_wait((dec_full + 8 * (s * DQ + di)), (dn_a[s] / DQ) & 1);
              w = lds_u32(dec_sm + (s * DQ + di) * 4);
              __syncwarp();
              mbar_arrive_w((dec_empty + 8 * (s * DQ + di)));
              ++dn_a[s];
            }
#pragma unroll
            for (int h = 0; h < GT; ++h)
              if (((w & ~prev) >> h) & 1u) load_unit(j, h);
            prev |= w;
          }
        }
        }
        if (lane == 0 && p.counters) {
          atomicAdd(&p.counters[2], (unsigned long long)vcount);
          atomicAdd(&p.counters[3], (unsigned long long)nsteps * GT);
        }
      }
    }
    __syncwarp();
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  } else if (warp == C::MMA_WARP) {
    if constexpr (C::SPLIT_REGS) setmaxnreg_dec<C::REG_OTHER>();
    // ======================= MMA issuer (warp-convergent, one elected issuer) ==========
    if (C::SPLIT && nsteps > 0) {
      split_issue(0);
    } else if (nsteps > 0) {
      constexpr uint32_t IDESC_QK = make_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t IDESC_PV = make_idesc_bf16(128, D, 0, 1);
      // descriptor templates; per-MMA offsets only touch the 14-bit start-address field
      const uint64_t dq0 = make_sdesc_sw128(sQ, 16, 1024);
      const uint64_t dk0 = make_sdesc_sw128(sK, 16, 1024);
      const uint64_t dv0 = make_sdesc_sw128(sV, BN * 128, 1024);
      const uint64_t dp0 = make_sdesc_sw128(sP, 16, 1024);
      mbar_wait(bar_q, 0);

      auto issue_qk = [&](int s, int j) {
        const int st = j % KS;
        if (s == 0) mbar_wait((k_full + 8 * (st)), (j / KS) & 1);
        tc_fence_after();
        // calibration: buffer j & 1, completion on s_full (b = 0) or the unused o_full slot (b = 1)
        const uint32_t d_tmem = CALIB ? tmem + (2 * s + (j & 1)) * 128 : tmem + C::S_COL + s * 128;
        umma_qk_tile_w<D, 128>(d_tmem, dq0 + uint64_t((s * C::Q_TILE) >> 4),
                               dk0 + uint64_t((st * C::K_TILE) >> 4), IDESC_QK);
        // the K stage is released by the last query tile that reads it (tile 1 of a
        // block pair has no QK at tile 0's frontier step)
        if (s == ((NQ == 2 && j < ns_a[NQ - 1]) ? NQ - 1 : 0)) umma_commit_w((k_empty + 8 * (st)));
        umma_commit_w(CALIB && (j & 1) ? (o_full + 8 * (s)) : (s_full + 8 * (s)));
      };

#pragma unroll
      for (int s = 0; s < NQ; ++s)
        if (ns_a[s] > 0) issue_qk(s, 0);
      if constexpr (CALIB) {
        // QK_s(j+2) goes into the buffer the softmax released for step j
#pragma unroll
        for (int s = 0; s < NQ; ++s)
          if (ns_a[s] > 1) issue_qk(s, 1);
        for (int j = 0; j + 2 < nsteps; ++j) {
#pragma unroll
          for (int s = 0; s < NQ; ++s) {
            if (j + 2 >= ns_a[s]) continue;
            mbar_wait((p_full + 8 * (2 * s + (j & 1))), (j >> 1) & 1);
            issue_qk(s, j + 2);
          }
        }
      }

      unsigned vbase = 0;      // V units consumed before this step
      uint32_t o_started = 0;  // bit s: O_s holds a partial sum
      if constexpr (C::PSM) {
        // Per step and tile: the first half (PV from TMEM, then the tile's next
        // QK into S_s, which overlaps the second half's exponentials), then the
        // second half (PV from shared memory).  V units are numbered at each
        // tile's first half, in the producer's order (tile 0's keeps, then tile
        // 1's additional ones).  (Serving both tiles' first halves before either
        // second half was measured slower.)
        uint32_t p1_par = 0;  // bit s: phase parity of p_full[s][1]
        for (int j = 0; j < nsteps; ++j) {
          uint32_t prev = 0;
          unsigned nunits = 0;
          unsigned uidx[GT];
#pragma unroll
          for (int s = 0; s < NQ; ++s) {
            if (j >= ns_a[s]) continue;
            const int sb = step_static_bits<GT>(gate_mode, window, j, qi_a[s]);
            mbar_wait((p_full + 8 * (2 * s)), j & 1);
            tc_fence_after();
            const uint32_t bits = sb >= 0 ? uint32_t(sb) : lds_u32(decm_sm + s * 4);
#pragma unroll
            for (int x = 0; x < GT; ++x)
              if (((bits & ~prev) >> x) & 1u) uidx[x] = vbase + nunits++;
            prev |= bits;
            if (bits & 1u) {
              const unsigned u = uidx[0];
              mbar_wait((v_full + 8 * (u % VS)), (u / VS) & 1);
              umma_pv64_w(tmem + C::O_COL + s * D, tmem + C::S_COL + s * 128,
                          dv0 + uint64_t(((u % VS) * C::V_UNIT) >> 4), IDESC_PV, (o_started >> s) & 1u);
              o_started |= 1u << s;
            }
            if (j + 1 < ns_a[s]) issue_qk(s, j + 1);  // S_s is free once P half 0 is consumed
            constexpr int x1 = GT == 2 ? 1 : 0;
            if ((bits >> x1) & 1u) {
              // released for kept second halves only: phase = this tile's count of them
              mbar_wait((p_full + 8 * (2 * s + 1)), (p1_par >> s) & 1u);
              p1_par ^= 1u << s;
              tc_fence_after();
              const unsigned u = uidx[x1];
              if (GT == 2) mbar_wait((v_full + 8 * (u % VS)), (u / VS) & 1);
              umma_pv64_ss_w(tmem + C::O_COL + s * D, dp0 + uint64_t((s * C::P_TILE) >> 4),
                             dv0 + uint64_t(((u % VS) * C::V_UNIT) >> 4) + uint64_t(GT == 1 ? 512 : 0), IDESC_PV,
                             (o_started >> s) & 1u);
              o_started |= 1u << s;
            }
            umma_commit_w((pv_done + 8 * (s)));
            if (j == ns_a[s] - 1) umma_commit_w((o_full + 8 * (s)));
          }
          for (unsigned x = 0; x < nunits; ++x) umma_commit_w((v_empty + 8 * ((vbase + x) % VS)));
          vbase += nunits;
        }
      } else if constexpr (!CALIB) {
      for (int j = 0; j < nsteps; ++j) {
        const int sb = step_static_bits<GT>(gate_mode, window, j, qi);
        uint32_t prev = 0;     // gate tiles already assigned a V slot this step
        unsigned nunits = 0;   // V units of this step
        unsigned uidx[GT];
#pragma unroll
        for (int s = 0; s < NQ; ++s) {
          // P of tile s arrives per 64-key half; the PV of half 0 runs while
          // the softmax computes half 1
          uint32_t bits = 0;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            mbar_wait((p_full + 8 * (2 * s + hh)), j & 1);
            if (BSFA_TRACE && tr_cta && lane == 0 && j < kTraceSteps && hh == 0)
              p.trace[(kEvPSeen * 2 + s) * kTraceSteps + j] = clock64();
            tc_fence_after();
            if constexpr (!CALIB) {
              if (hh == 0) bits = sb >= 0 ? uint32_t(sb) : lds_u32(decm_sm + s * 4);
              const int x = GT == 2 ? hh : 0;  // gate tile of this half
              if ((bits >> x) & 1u) {
                if (hh == 0 || GT == 2) {
                  if (!((prev >> x) & 1u)) uidx[x] = vbase + nunits++;
                  const unsigned u = uidx[x];
                  mbar_wait((v_full + 8 * (u % VS)), (u / VS) & 1);
                  if (BSFA_TRACE && tr_cta && lane == 0 && j < kTraceSteps)
                    p.trace[(kEvVReady * 2 + s) * kTraceSteps + j] = clock64();
                }
                const uint64_t dv = dv0 + uint64_t(((uidx[x] % VS) * C::V_UNIT) >> 4) +
                                    uint64_t(GT == 1 ? hh * 512 : 0);  // 64 key rows = 8 KB
                umma_pv64_w(tmem + C::O_COL + s * D, tmem + C::S_COL + s * 128 + hh * 32, dv, IDESC_PV,
                            (o_started >> s) & 1u);
                o_started |= 1u << s;
              }
            }
          }
          if constexpr (!CALIB) {
            prev |= bits;
            if (s == NQ - 1) {
              // every PV reading this step's V units has been issued
              for (unsigned x = 0; x < nunits; ++x) umma_commit_w((v_empty + 8 * ((vbase + x) % VS)));
              vbase += nunits;
            }
            if (j == nsteps - 1) umma_commit_w((o_full + 8 * (s)));
          }
          // QK_s(j+1) reuses S_s; issued after PV_s(j), so its commit also
          // certifies that PV_s(j) has landed (softmax may rescale O_s)
          if (j + 1 < nsteps) issue_qk(s, j + 1);
          if (BSFA_TRACE && tr_cta && lane == 0 && j < kTraceSteps)
            p.trace[(kEvIssued * 2 + s) * kTraceSteps + j] = clock64();
        }
      }
      }
    }
    __syncwarp();
    named_bar_sync(15, C::NUM_THREADS);
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
    return;
  } else if (TPR == 2 && warp < C::SOFTMAX_WARPS) {
    if constexpr (TPR == 2) {
      setmaxnreg_inc<C::REG_SOFT>();
      // ======================= softmax, two threads per row (TPR = 2) ============
      // Thread (s, h, r) owns row r of query tile s over the 64 keys [64h, 64h+64)
      // of every step (gate tile h at b_n = 64, half of the gate tile at 128).
      // The two threads of a row exchange half-row maxima at the vote barrier,
      // so both keep the same running max; each keeps its half's row sum.
      const int s = warp >> 3;
      const int h = (warp >> 2) & 1;
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
      const uint32_t xmax = xch_sm + s * C::XCH_TILE;  // f32 [2 par][2 h][128]
      const uint32_t xfin = xmax + 2 * 2 * 128 * 4;    // f32 [2 h][128]
      const bool lead = h == 0 && r == 0;
      const bool tr0 = BSFA_TRACE && tr_cta && lead;
      const uint32_t my_bit = GT == 2 ? (1u << h) : 1u;
      const uint32_t other_bit = GT == 2 ? (1u << (h ^ 1)) : 1u;
      const uint32_t p_mine = p_full + 16 * s + 8 * h;

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
        mbar_wait((s_full + 8 * (s)), j & 1);
        if (tr0 && j < kTraceSteps) p.trace[(kEvSReady * 2 + s) * kTraceSteps + j] = clock64();
        tc_fence_after();
        uint32_t sv[64];
        tmem_ld32(s_row + h * 64, &sv[0]);
        tmem_ld32(s_row + h * 64 + 32, &sv[32]);
        tmem_wait_ld();
        const int sb = step_static_bits<GT>(gate_mode, window, j, qi);
        if (j == qi && causal) {
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (h * 64 + c > r) sv[c] = __float_as_uint(-INFINITY);
        }
        if (!causal && (j + 1) * 128 > valid_len) {
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
          float a4 = fmax3(__uint_as_float(sv[12]), __uint_as_float(sv[13]), __uint_as_float(sv[14]));
          float a5 = fmax3(__uint_as_float(sv[15]), __uint_as_float(sv[16]), __uint_as_float(sv[17]));
#pragma unroll
          for (int c = 18; c < 60; c += 12) {
            a0 = fmax3(a0, __uint_as_float(sv[c]), __uint_as_float(sv[c + 1]));
            a1 = fmax3(a1, __uint_as_float(sv[c + 2]), __uint_as_float(sv[c + 3]));
            a2 = fmax3(a2, __uint_as_float(sv[c + 4]), __uint_as_float(sv[c + 5]));
            a3 = fmax3(a3, __uint_as_float(sv[c + 6]), __uint_as_float(sv[c + 7]));
            a4 = fmax3(a4, __uint_as_float(sv[c + 8]), __uint_as_float(sv[c + 9]));
            a5 = fmax3(a5, __uint_as_float(sv[c + 10]), __uint_as_float(sv[c + 11]));
          }
          a0 = fmax3(a0, __uint_as_float(sv[54]), __uint_as_float(sv[55]));
          a1 = fmax3(a1, __uint_as_float(sv[56]), __uint_as_float(sv[57]));
          a2 = fmax3(a2, __uint_as_float(sv[58]), __uint_as_float(sv[59]));
          a3 = fmax3(a3, __uint_as_float(sv[60]), __uint_as_float(sv[61]));
          a4 = fmax3(a4, __uint_as_float(sv[62]), __uint_as_float(sv[63]));
          mh = fmax3(fmax3(a0, a1, a2), fmax3(a3, a4, a5), -INFINITY);
        }
        // ---- exchange half-row maxima and vote, one barrier round (256 threads)
        const uint32_t par = j & 1;
        float mo = -INFINITY;
        uint32_t bits;
        if (sb == 0) {
          bits = 0;  // FrontierOnlyGate / window-excluded step: nobody needs maxima
        } else {
          sts_f32(xmax + ((par * 2 + h) * 128 + r) * 4, mh);
          if (sb > 0) {
            named_bar_sync(1 + s, 256);
            bits = uint32_t(sb);
          } else if (gate_mode == kGateThreshold) {
            if constexpr (GT == 2) {
              bits = named_bar_red_or(1 + s, 256, (h == 0 && mh * scale > T) ? 1u : 0u);
              bits |= named_bar_red_or(1 + s, 256, (h == 1 && mh * scale > T) ? 1u : 0u) << 1;
            } else {
              bits = named_bar_red_or(1 + s, 256, mh * scale > T ? 1u : 0u);
            }
          } else {
            // RunningMaxGate, gate tiles in key order (gates.py:101-118)
            if constexpr (GT == 2) {
              const uint32_t k0 = named_bar_red_or(1 + s, 256, (h == 0 && (mh - m_true) * scale >= lam) ? 1u : 0u);
              const float m_half0 = lds_f32(xmax + ((par * 2 + 0) * 128 + r) * 4);
              const float mrun = k0 ? fmaxf(m_true, m_half0) : m_true;
              const uint32_t k1 = named_bar_red_or(1 + s, 256, (h == 1 && (mh - mrun) * scale >= lam) ? 1u : 0u);
              bits = k0 | (k1 << 1);
            } else {
              const float mfull = fmaxf(mh, lds_f32(xmax + ((par * 2 + (h ^ 1)) * 128 + r) * 4));
              bits = named_bar_red_or(1 + s, 256, (mfull - m_true) * scale >= lam ? 1u : 0u);
            }
          }
          mo = lds_f32(xmax + ((par * 2 + (h ^ 1)) * 128 + r) * 4);
        }
        if (tr0 && j < kTraceSteps) p.trace[(kEvVoted * 2 + s) * kTraceSteps + j] = clock64();
        const bool mine = (bits & my_bit) != 0;
        const bool other = (bits & other_bit) != 0;
        if (gate_mode == kGateRunMax) {
          if (mine) m_true = fmaxf(m_true, mh);
          if (other) m_true = fmaxf(m_true, mo);
        }
        if (lead) {
          if (sb < 0) {
            const int di = int(dn % DQ);
            mbar_wait((dec_empty + 8 * (s * DQ + di)), ((dn / DQ) & 1) ^ 1);
            sts_u32(dec_sm + (s * DQ + di) * 4, bits);
            mbar_arrive((dec_full + 8 * (s * DQ + di)));
          }
          sts_u32(decm_sm + s * 4, bits);
        }
        if (sb < 0) ++dn;
        if (bits == 0) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(p_mine);
          if (lead && p.decisions) {
            int8_t* drow = p.decisions + (((long long)b * p.heads_q + hq) * p.num_q_tiles + qi) * p.gate_cols;
#pragma unroll
            for (int x = 0; x < GT; ++x) drow[j * GT + x] = int8_t(1);
          }
          continue;
        }
        // running max over the kept halves (identical in both threads of the row)
        const float m_step = fmaxf(mine ? mh : -INFINITY, other ? mo : -INFINITY);
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
        const bool kept_h = ((bits >> (GT == 2 ? h : 0)) & 1u) != 0;
        float psum = 0.f;
        if (kept_h) {
          const float neg = (m_ref == -INFINITY) ? 0.f : -m_ref * sl2;
          const uint64_t sl2x2 = f2_pack(sl2, sl2);
          const uint64_t negx2 = f2_pack(neg, neg);
          uint64_t acc0 = 0, acc1 = 0;
#pragma unroll
          for (int cb = 0; cb < 64; cb += 32) {  // two 32-key chunks: 16 packed registers live at a time
            uint32_t pk[16];
#pragma unroll
            for (int c = cb; c < cb + 32; c += 4) {
              const uint64_t x0 = ffma2(f2_pack(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])), sl2x2, negx2);
              const uint64_t x1 =
                  ffma2(f2_pack(__uint_as_float(sv[c + 2]), __uint_as_float(sv[c + 3])), sl2x2, negx2);
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
              acc0 = fadd2(acc0, f2_pack(p0, p1));
              acc1 = fadd2(acc1, f2_pack(p2, p3));
              pk[(c - cb) / 2] = pack_bf16x2(p0, p1);
              pk[(c - cb) / 2 + 1] = pack_bf16x2(p2, p3);
            }
            tmem_st16(s_row + h * 32 + cb / 2, pk);
          }
          const uint64_t acc = fadd2(acc0, acc1);
          psum = f2_lo(acc) + f2_hi(acc);
        }
        // the half-0 threads rescale the whole O row before releasing half 0 (after
        // their exponentials, when the score registers are free)
        // (PV of half 1 is issued after PV of half 0, so it follows the rescale)
        if (h == 0 && __any_sync(0xffffffffu, rescale)) {
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
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_mine);
        if (tr0 && j < kTraceSteps) p.trace[(kEvPDone * 2 + s) * kTraceSteps + j] = clock64();
        l_sum = l_sum * alpha + psum;
        if (lead) {
          kept_tiles += __popc(bits);
          if (p.decisions) {
            int8_t* drow = p.decisions + (((long long)b * p.heads_q + hq) * p.num_q_tiles + qi) * p.gate_cols;
#pragma unroll
            for (int x = 0; x < GT; ++x)
              drow[j * GT + x] = j == qi ? int8_t(2) : (((bits >> x) & 1u) ? int8_t(3) : int8_t(1));
          }
        }
        o_valid = true;
      }

      // ---- epilogue: O = O~ / (l_0 + l_1), lse = m * scale + ln l
      sts_f32(xfin + (h * 128 + r) * 4, l_sum);
      mbar_wait((o_full + 8 * (s)), 0);
      tc_fence_after();
      named_bar_sync(3 + s, 256);
      const float l_row = l_sum + lds_f32(xfin + ((h ^ 1) * 128 + r) * 4);
      const float inv_l = 1.f / l_row;
      bool bad = !(l_row > 0.f);
      const int row = qi * 128 + r;
      const long long orow = (long long)b * p.o_sb + (long long)hq * p.o_sh + (long long)row * p.o_sn + h * (D / 2);
#pragma unroll
      for (int c = 0; c < D / 2; c += 32) {
        uint32_t ov[32];
        tmem_ld32(o_row + h * (D / 2) + c, ov);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float a0 = __uint_as_float(ov[e]) * inv_l, a1 = __uint_as_float(ov[e + 1]) * inv_l;
          if (p.inject_fault && qi == 0 && r == 0 && s == 0 && h == 0 && c == 0 && e == 0) a0 += 1.0f;
          bad |= !isfinite(a0) || !isfinite(a1);
          pk[e / 2] = pack_bf16x2(a0, a1);
        }
        store_o32(p, orow + c, pk);
      }
      if (h == 0) p.lse[((long long)b * p.heads_q + hq) * p.seq_len + row] = m_ref * scale + logf(l_row);
      if (bad && p.status) atomicOr(p.status, 1);
      if (lead && p.counters) {
        atomicAdd(&p.counters[0], (unsigned long long)nsteps * GT);
        atomicAdd(&p.counters[1], kept_tiles);
      }
      tc_fence_before();
      named_bar_arrive(15, C::NUM_THREADS);
      return;
    }
  } else if (warp < C::SOFTMAX_WARPS) {
    if constexpr (C::SPLIT_REGS) setmaxnreg_inc<C::REG_SOFT>();
    // ======================= softmax group s (query tile s) =======================
    // Thread r owns row r (TMEM lane r) over all 128 keys of a step.  Critical
    // path per step: S -> registers, gate-tile maxima, gate vote, then per
    // 64-key half: exponentials -> packed P in TMEM -> signal the MMA warp
    // (the PV of half 0 overlaps the exponentials of half 1).  The row sum is
    // accumulated after P is released.
    const int s = warp >> 2;
    const int wq = warp & 3;
    const int r = wq * 32 + lane;  // row inside the query tile == TMEM lane
    const int hq = hq_a[s];
    const int qi_s = qi_a[s];      // this tile's query block
    const int nst = ns_a[s];       // this tile's steps (a block pair's tile 1 has one fewer)
    if (qi_s < 0) {                // a block pair's missing second block (odd block count)
      named_bar_arrive(15, C::NUM_THREADS);
      return;
    }
    const uint32_t lane_off = uint32_t(wq * 32) << 16;
    const uint32_t s_row = tmem + lane_off + C::S_COL + s * 128;
    const uint32_t o_row = tmem + lane_off + C::O_COL + s * D;
    const float sl2 = p.scale_log2;
    const float scale = p.scale;
    const float rescale_raw = p.rescale_raw;
    const bool tr0 = BSFA_TRACE && tr_cta && r == 0;
    const uint32_t p_half = p_full + 16 * s;

    float T = 0.f;
    if (!CALIB && p.gate_mode == kGateThreshold) {
      const int pos = qi_s < p.thr_positions - 1 ? qi_s : p.thr_positions - 1;
      T = p.thr[(long long)hq * p.thr_positions + pos];
    }

    const float lam = p.gate_lambda;
    float m_true = -INFINITY;  // exact running row max (RunningMaxGate), raw units
    float m_ref = -INFINITY;  // raw (unscaled) reference max of this row over its kept tiles
    float l_sum = 0.f;        // row sum relative to m_ref
    bool o_valid = false;     // tile-uniform: O_s holds data
    unsigned dn = 0;
    unsigned long long kept_tiles = 0;

    // turn barriers 5 + s: group s may start its phase once the other group
    // finished the same phase of the previous (s = 0) / same (s = 1) step
    constexpr bool kTurn = !CALIB && NQ == 2 && BSFA_TURN != 0;
    auto turn_wait = [&](int j) {
      if (kTurn && !(s == 0 && j == 0)) named_bar_sync(5 + s, 256);
    };
    auto turn_pass = [&]() {
      if (kTurn) named_bar_arrive(5 + (s ^ 1), 256);
    };
    for (int j = 0; j < nst; ++j) {
      if (BSFA_TURN == 2) turn_wait(j);
      if constexpr (CALIB)
        mbar_wait((j & 1) ? (o_full + 8 * (s)) : (s_full + 8 * (s)), (j >> 1) & 1);
      else
        mbar_wait((s_full + 8 * (s)), j & 1);
      if (tr0 && j < kTraceSteps) p.trace[(kEvSReady * 2 + s) * kTraceSteps + j] = clock64();
      tc_fence_after();
      uint32_t sv[128];
      const uint32_t s_buf = CALIB ? tmem + lane_off + (2 * s + (j & 1)) * 128 : s_row;
#pragma unroll
      for (int c = 0; c < 128; c += 32) tmem_ld32(s_buf + c, &sv[c]);
      tmem_wait_ld();

      const int sb = CALIB ? -1 : step_static_bits<GT>(gate_mode, window, j, qi_s);
      if (!CALIB) {
        if (j == qi_s && causal) {  // frontier step: key offset c vs row r inside block i
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (c > r) sv[c] = __float_as_uint(-INFINITY);
        }
        if (!causal && (j + 1) * 128 > valid_len) {
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (j * 128 + c >= valid_len) sv[c] = __float_as_uint(-INFINITY);
        }
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
      // gate-tile maxima: b_n = 64 -> the halves; b_n = 128 -> the whole row
      float mx[GT];
      if constexpr (GT == 2) {
        mx[0] = mh[0];
        mx[1] = mh[1];
      } else {
        mx[0] = fmaxf(mh[0], mh[1]);
      }

      if constexpr (CALIB) {
#pragma unroll
        for (int x = 0; x < GT; ++x) {
          // warp max in one REDUX on the order-preserving integer image of the scaled max
          const int m = __reduce_max_sync(0xffffffffu, float_to_ordered(mx[x] * scale));
          if (lane == 0) atomicMax(&cvals[s * C::MAXA + j * GT + x], m);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive((p_half + 8 * (j & 1)));  // buffer j & 1 may take QK_s(j+2)
        continue;
      } else {
        // ---- gate decision; votes are OR-reduced over the tile's 128 rows in the
        //      barrier hardware (BAR.RED.OR)
        uint32_t bits;
        if (sb >= 0) {
          bits = uint32_t(sb);
        } else if (gate_mode == kGateThreshold) {
          // ThresholdGate: keep iff tile max (scaled) > T (gates.py:77-78)
          bits = 0;
#pragma unroll
          for (int x = 0; x < GT; ++x) bits |= named_bar_red_or(1 + s, 128, mx[x] * scale > T ? 1u : 0u) << x;
        } else {
          // RunningMaxGate: keep iff max over rows of (local row max - running
          // row max) >= lambda, judged before the tile is merged; tiles in key
          // order, so gate tile 1 sees tile 0 merged if it was kept
          // (gates.py:101-118; -inf running max gives +inf: keep)
          bits = 0;
          float mrun = m_true;
#pragma unroll
          for (int x = 0; x < GT; ++x) {
            const uint32_t k = named_bar_red_or(1 + s, 128, (mx[x] - mrun) * scale >= lam ? 1u : 0u);
            bits |= k << x;
            if (k) mrun = fmaxf(mrun, mx[x]);
          }
        }
        if (gate_mode == kGateRunMax) {
#pragma unroll
          for (int x = 0; x < GT; ++x)
            if ((bits >> x) & 1u) m_true = fmaxf(m_true, mx[x]);
        }
        if (tr0 && j < kTraceSteps) p.trace[(kEvVoted * 2 + s) * kTraceSteps + j] = clock64();
        if (r == 0) {
          if (sb < 0) {
            const int di = int(dn % DQ);
            mbar_wait((dec_empty + 8 * (s * DQ + di)), ((dn / DQ) & 1) ^ 1);
            sts_u32(dec_sm + (s * DQ + di) * 4, bits);
            mbar_arrive((dec_full + 8 * (s * DQ + di)));
          }
          sts_u32(decm_sm + s * 4, bits);
          kept_tiles += __popc(bits);
          if (p.decisions) {
            int8_t* drow = p.decisions + (((long long)b * p.heads_q + hq) * p.num_q_tiles + qi_s) * p.gate_cols;
#pragma unroll
            for (int x = 0; x < GT; ++x)
              drow[j * GT + x] = j == qi_s ? int8_t(2) : (((bits >> x) & 1u) ? int8_t(3) : int8_t(1));
          }
        }
        if (sb < 0) ++dn;
        if (bits == 0) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive((p_half + 8 * (0)));
          if (lane == 0 && !C::PSM) mbar_arrive((p_half + 8 * (1)));  // PSM: kept second halves only
          if (tr0 && j < kTraceSteps) p.trace[(kEvPDone * 2 + s) * kTraceSteps + j] = clock64();
          if (BSFA_TURN == 1) turn_wait(j);
          turn_pass();
          continue;
        }
        if (BSFA_TURN == 1) turn_wait(j);

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
        // O_s is quiescent here (S_s(j) committed after PV_s(j-1); PSM: after the
        // first-half PV, pv_done certifies the second): rescale the rows whose
        // reference max moved by more than 2^8, before any P release
        if (__any_sync(0xffffffffu, rescale)) {
          if (C::PSM && j > 0) mbar_wait((pv_done + 8 * (s)), (j - 1) & 1);
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

        // P = exp2(s * scale*log2e - m * scale*log2e), per 64-key half, bf16-packed
        // over S_s columns [32hh, 32hh + 32); released to the MMA warp per half
        const float neg = (m_ref == -INFINITY) ? 0.f : -m_ref * sl2;
        const uint64_t sl2x2 = f2_pack(sl2, sl2);
        const uint64_t negx2 = f2_pack(neg, neg);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const bool kept_h = ((bits >> (GT == 2 ? hh : 0)) & 1u) != 0;
          // PSM: p_full[s][1] is released for kept second halves only (the MMA
          // warp knows the decision); the previous step's second-half PV must
          // have landed first -- it frees the P buffer and keeps p_full[s][1]
          // at most one phase ahead of the MMA warp
          if (C::PSM && hh == 1 && kept_h && j > 0) mbar_wait((pv_done + 8 * (s)), (j - 1) & 1);
          if (kept_h) {
            uint32_t pk[32];
#pragma unroll
            for (int c = 0; c < 64; c += 4) {
              const int e = hh * 64 + c;
              const uint64_t x0 = ffma2(f2_pack(__uint_as_float(sv[e]), __uint_as_float(sv[e + 1])), sl2x2, negx2);
              const uint64_t x1 =
                  ffma2(f2_pack(__uint_as_float(sv[e + 2]), __uint_as_float(sv[e + 3])), sl2x2, negx2);
              const float p0 = ex2_approx(f2_lo(x0)), p1 = ex2_approx(f2_hi(x0));
              float p2, p3;
              // offload part of the exponentials from the MUFU to the FMA pipe
              if (BSFA_EXP_EMU == 2 || (BSFA_EXP_EMU == 1 && ((c >> 2) & 1))) {
                // x1 += 0 * (p0, p1): a data dependency on this group's MUFU
                // results, so the scheduler interleaves the polynomial work with
                // the (8-cycle) MUFU issue slots instead of clustering the MUFUs
                const uint64_t x1d = BSFA_EXP_CHAIN ? ffma2(f2_pack(p0, p1), 0ull, x1) : x1;
                const uint64_t e1 = exp2_poly_x2(x1d);
                p2 = f2_lo(e1);
                p3 = f2_hi(e1);
              } else {
                p2 = ex2_approx(f2_lo(x1));
                p3 = ex2_approx(f2_hi(x1));
              }
              sv[e] = __float_as_uint(p0);
              sv[e + 1] = __float_as_uint(p1);
              sv[e + 2] = __float_as_uint(p2);
              sv[e + 3] = __float_as_uint(p3);
              pk[c / 2] = pack_bf16x2(p0, p1);
              pk[c / 2 + 1] = pack_bf16x2(p2, p3);
            }
            if (C::PSM && hh == 1) {
              // second half -> shared memory, K-major SW128 (16-byte chunk c of
              // row r at chunk c ^ (r & 7)); the buffer is free (pv_done waited below)
              const uint32_t prow = sP + s * C::P_TILE + r * 128;
#pragma unroll
              for (int c16 = 0; c16 < 8; ++c16)
                sts_u128(prow + ((c16 ^ (r & 7)) << 4), pk[4 * c16], pk[4 * c16 + 1], pk[4 * c16 + 2],
                         pk[4 * c16 + 3]);
              fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core
            } else {
              tmem_st32(s_row + hh * 32, pk);
              tmem_wait_st();
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0 && !(C::PSM && hh == 1 && !kept_h)) mbar_arrive((p_half + 8 * (hh)));
          if (tr0 && hh == 0 && j < kTraceSteps) p.trace[(kEvExpDone * 2 + s) * kTraceSteps + j] = clock64();
        }
        if (tr0 && j < kTraceSteps) p.trace[(kEvPDone * 2 + s) * kTraceSteps + j] = clock64();
        turn_pass();

        // row sum of the kept exponentials (off the MMA critical path)
        uint64_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if (((bits >> (GT == 2 ? hh : 0)) & 1u) != 0) {
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
    }
    if (kTurn && s == 0 && nsteps > 0) named_bar_sync(5, 256);  // group 1's last pass

    if constexpr (CALIB) {
      // ---- order statistics of this row of gate-tile maxima (calibration.py:116-153)
      const int A = nst * GT;
      named_bar_sync(3 + s, 128);
      int* vals = cvals + s * C::MAXA;
      if (p.c_maxima) {
        float* out = p.c_maxima + ((long long)hq * p.num_q_tiles + qi_s) * p.gate_cols;
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
        const long long idx = (((long long)r * p.c_num_layers + p.c_layer) * p.heads_q + hq) * p.c_positions + qi_s;
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
      // ---- epilogue: O = O~ / l, lse = m * scale + ln l (engine.py:178-182)
      mbar_wait((o_full + 8 * (s)), 0);
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
      if (r == 0 && p.counters) {
        atomicAdd(&p.counters[0], (unsigned long long)nst * GT);
        atomicAdd(&p.counters[1], kept_tiles);
      }
    }
    tc_fence_before();
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  } else {
    // idle warp (completes the last warpgroup for setmaxnreg); issues query
    // tile 1's tcgen05 work in split-issue builds
    if constexpr (C::SPLIT_REGS) setmaxnreg_dec<C::REG_OTHER>();
    if constexpr (C::SPLIT && NQ == 2) {
      if (nsteps > 0) split_issue(1);
      __syncwarp();
    }
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  }
}

}  // namespace bsfa
