// K2: calibration block maxima for sm_100a, fused with the cutoff selection.
//
// Reference: calibration.py:93-123 collect_block_maxima (the max of the scaled
// scores over every off-frontier tile j < A_p of the causal prefix, per
// (layer, head, query position p)), calibration.py:126-153
// thresholds_from_maxima / _tie_count (the (k+1)-th largest maximum, +inf for
// k = 0, -inf when fewer than k+1 tiles, tie iff vals[k-1] == vals[k]) and the
// per-sample accumulation of calibration.py:185-196 (fp64 sum of finite
// cutoffs, counts of finite / -inf / +inf).  The 512 MiB-per-sample block-max
// tensor of the reference never exists: each CTA keeps its rows' maxima in
// shared memory and accumulates the cutoffs of this (sample, layer).
//
// One CTA = two query tiles (two q heads of a GQA group at query block i, or
// blocks 2m+1 and 2m of one q head for odd groups) over the off-frontier
// prefix j < i, in 128-key steps (GT = 128 / b_n gate tiles per step).  With
// no O accumulator, TMEM holds two score buffers per query tile, so QK(j+2) is
// issued as soon as the softmax warps have read S(j) and the tensor core never
// waits for them.
//
// Warp roles (384 threads): warps 0-3 / 4-7 reduce query tile 0 / 1 (thread r
// = row r = TMEM lane r), warp 8 = TMA producer (Q once, K per step), warp 9 =
// tcgen05 issuer + TMEM owner, warps 10-11 idle (complete the warpgroup).
#pragma once

#include "bsfa_common.cuh"

namespace bsfa {

template <int D, int GT, int BM = 128>
struct CCfg {
  static constexpr int NCH = D / 64;           // 64-column swizzle atoms along head_dim
  static constexpr int NQ = D == 256 ? 1 : 2;  // query tiles per CTA (head_dim 256: one)
  static constexpr int Q_TILE = 128 * D * 2;
  static constexpr int K_TILE = 128 * D * 2;   // one 128-key step
  static constexpr int KS = D == 256 ? 2 : 3;  // K ring stages
  static constexpr int MAXA = 4096;            // max off-frontier gate tiles per row
  static constexpr int NBLK = 128 / BM;        // query blocks per 128-row tile
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + NQ * Q_TILE;
  static constexpr int OFF_CAL = OFF_K + KS * K_TILE;      // int [NQ tiles][NBLK][MAXA] ordered maxima
  static constexpr int OFF_BAR = OFF_CAL + NQ * NBLK * MAXA * 4;
  // bar_q, k_full/empty[KS], s_full[2][2 buffers], s_read[2][2 buffers]
  static constexpr int NUM_BARS = 1 + 2 * KS + 4 + 4;
  static constexpr int OFF_TMEMPTR = OFF_BAR + NUM_BARS * 8;
  static constexpr int SMEM_BYTES = OFF_TMEMPTR + 16 + 1024;  // + alignment slack
  static constexpr int TMEM_COLS = 512;                        // S_{s,b} at (2s + b) * 128
  static constexpr int NUM_THREADS = 12 * 32;
  static constexpr int KPROD_WARP = 8, MMA_WARP = 9;
  static constexpr int REG_OTHER = 56;
  static constexpr int REG_LAUNCH = (65536 / NUM_THREADS) / 8 * 8;
  static constexpr int REG_SOFT = (NUM_THREADS * REG_LAUNCH - 128 * REG_OTHER) / 256 / 8 * 8;
  static_assert(GT == 1 || GT == 2, "b_n in {64, 128}");
  static_assert(BM == 128 || BM == 64, "b_m in {64, 128}");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
};

// BM = 64: a 128-row tile holds query blocks 2t (rows 0-63) and 2t+1 (rows
// 64-127); each block has its own off-frontier prefix A = blk * 64 / b_n, its
// own maxima row (warps 0-1 / 2-3 of the tile) and its own cutoffs.
template <int D, int GT, int BM = 128>
__global__ void __launch_bounds__(CCfg<D, GT, BM>::NUM_THREADS, 1)
    bsfa_calib_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const KernelParams p) {
  using C = CCfg<D, GT, BM>;
  constexpr int KS = C::KS, NCH = C::NCH, NBLK = C::NBLK;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = opaque_u32((sraw + 1023u) & ~1023u);
  uint8_t* smem = smem_raw + (sbase - sraw);
  const uint32_t sQ = sbase + C::OFF_Q;
  const uint32_t sK = sbase + C::OFF_K;
  int* cvals = reinterpret_cast<int*>(smem + C::OFF_CAL);
  const uint32_t bar_q = sbase + C::OFF_BAR;
  const uint32_t k_full = bar_q + 8;
  const uint32_t k_empty = k_full + 8 * KS;
  const uint32_t s_full = k_empty + 8 * KS;   // [2 tiles][2 buffers] QK landed
  const uint32_t s_read = s_full + 32;        // [2 tiles][2 buffers] the 4 warps read it
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEMPTR);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- work unit: (kv head) major, heaviest query block first (as the forward)
  int qi_a[2], hq_a[2], ns_a[2];
  int g_;
  {
    const int unit = blockIdx.x;
    if constexpr (C::NQ == 1) {
      // head_dim 256: one query tile per CTA
      const int per_g = p.num_q_tiles * p.group;
      g_ = unit / per_g;
      const int rem = unit - g_ * per_g;
      qi_a[0] = p.num_q_tiles - 1 - rem / p.group;
      qi_a[1] = -1;
      hq_a[0] = hq_a[1] = g_ * p.group + rem % p.group;
    } else if (p.block_pair) {
      const int per_g = ((p.num_q_tiles + 1) / 2) * p.group;
      g_ = unit / per_g;
      const int rem = unit - g_ * per_g;
      const int m = rem / p.group;
      const int qi = p.num_q_tiles - 1 - 2 * m;
      qi_a[0] = qi;
      qi_a[1] = qi - 1;  // -1: no second block (odd block count)
      hq_a[0] = hq_a[1] = g_ * p.group + (rem - m * p.group);
    } else {
      const int pairs = p.group / 2;
      const int per_g = p.num_q_tiles * pairs;
      g_ = unit / per_g;
      const int rem = unit - g_ * per_g;
      const int qi = p.num_q_tiles - 1 - rem / pairs;
      const int pr = rem - (rem / pairs) * pairs;
      qi_a[0] = qi_a[1] = qi;
      hq_a[0] = g_ * p.group + 2 * pr;
      hq_a[1] = hq_a[0] + 1;
    }
  }
  const int g = g_;
  // the off-frontier causal prefix (calibration.py:110-113): j < i for b_m =
  // 128; for b_m = 64 the 128-key steps holding the prefix of block 2t+1
  constexpr int BN = 128 / GT;
  auto a_of = [](int blk) { return blk * BM / BN; };  // A_blk, tiling.py:63-65
#pragma unroll
  for (int t = 0; t < 2; ++t)
    ns_a[t] = qi_a[t] < 0 ? 0 : (BM == 128 ? qi_a[t] : (a_of(2 * qi_a[t] + 1) + GT - 1) / GT);
  const int nsteps = ns_a[0];

  // ---- setup
  if (warp == C::KPROD_WARP && lane == 0) {
    mbar_init(bar_q, 1);
    for (int i = 0; i < KS; ++i) {
      mbar_init(k_full + 8 * i, 1);
      mbar_init(k_empty + 8 * i, 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(s_full + 8 * i, 1);
      mbar_init(s_read + 8 * i, 4);
    }
    fence_mbarrier_init();
  }
  for (int i = threadIdx.x; i < C::NQ * NBLK * C::MAXA; i += blockDim.x) cvals[i] = float_to_ordered(-INFINITY);
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
    // ======================= TMA producer: Q once, K per 128-key step =========
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
          tma_load_4d_w(sQ + s * C::Q_TILE + c * 128 * 128, &tm_q, bar_q, c * 64, (qi_a[s] < 0 ? 0 : qi_a[s]) * 128,
                        hq_a[s], 0, kEvictFirst);
      for (int j = 0; j < nsteps; ++j) {
        const int st = j % KS;
        mbar_wait(k_empty + 8 * st, ((j / KS) & 1) ^ 1);
        mbar_arrive_expect_tx_w(k_full + 8 * st, C::K_TILE);
#pragma unroll
        for (int c = 0; c < NCH; ++c)
          tma_load_4d_w(sK + st * C::K_TILE + c * 128 * 128, &tm_k, k_full + 8 * st, c * 64, j * 128, g, 0, kEvictLast);
      }
    }
    __syncwarp();
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  } else if (warp == C::MMA_WARP) {
    setmaxnreg_dec<C::REG_OTHER>();
    // ======================= tcgen05 issuer: QK(j) into buffer j & 1 ===========
    if (nsteps > 0) {
      constexpr uint32_t IDESC_QK = make_idesc_bf16(128, 128, 0, 0);
      const uint64_t dq0 = make_sdesc_sw128(sQ, 16, 1024);
      const uint64_t dk0 = make_sdesc_sw128(sK, 16, 1024);
      mbar_wait(bar_q, 0);
      auto issue_qk = [&](int s, int j) {
        const int st = j % KS;
        if (s == 0) mbar_wait(k_full + 8 * st, (j / KS) & 1);
        tc_fence_after();
        if constexpr (D == 256) {  // K = 256: four 64-column atoms, accumulating
#pragma unroll
          for (int c = 0; c < NCH; ++c)
            umma_qk_chunk_w(tmem + (2 * s + (j & 1)) * 128, dq0 + uint64_t((s * C::Q_TILE + c * 128 * 128) >> 4),
                            dk0 + uint64_t((st * C::K_TILE + c * 128 * 128) >> 4), IDESC_QK, c > 0 ? 1u : 0u);
        } else {
          umma_qk_tile_w<D, 128>(tmem + (2 * s + (j & 1)) * 128, dq0 + uint64_t((s * C::Q_TILE) >> 4),
                                 dk0 + uint64_t((st * C::K_TILE) >> 4), IDESC_QK);
        }
        // the stage is released by the last query tile reading it (tile 1 of a
        // block pair stops one step early)
        if (s == (j < ns_a[1] ? 1 : 0)) umma_commit_w(k_empty + 8 * st);
        umma_commit_w(s_full + 8 * (2 * s + (j & 1)));
      };
      for (int j = 0; j < 2 && j < nsteps; ++j)
#pragma unroll
        for (int s = 0; s < 2; ++s)
          if (j < ns_a[s]) issue_qk(s, j);
      // QK_s(j+2) goes into the buffer the softmax released after step j
      for (int j = 0; j + 2 < nsteps; ++j) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (j + 2 >= ns_a[s]) continue;
          mbar_wait(s_read + 8 * (2 * s + (j & 1)), (j >> 1) & 1);
          issue_qk(s, j + 2);
        }
      }
    }
    __syncwarp();
    named_bar_sync(15, C::NUM_THREADS);
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
    return;
  } else if (warp < 8) {
    setmaxnreg_inc<C::REG_SOFT>();
    // ======================= per-row tile maxima of query tile s ===============
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
    const float scale = p.scale;
    const int hf = BM == 64 ? (r >> 6) : 0;          // this thread's query block in the tile
    const int blk = BM == 64 ? 2 * qi_s + hf : qi_s;
    const int A = BM == 64 ? a_of(blk) : nst * GT;   // this block's off-frontier prefix (gate tiles)
    int* vals = cvals + (s * NBLK + hf) * C::MAXA;
    for (int j = 0; j < nst; ++j) {
      const int buf = 2 * s + (j & 1);
      mbar_wait(s_full + 8 * buf, (j >> 1) & 1);
      tc_fence_after();
      uint32_t sv[128];
#pragma unroll
      for (int c = 0; c < 128; c += 32) tmem_ld32(tmem + lane_off + buf * 128 + c, &sv[c]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_read + 8 * buf);  // the buffer may take QK_s(j+2)
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
      // tile max over the 128 rows: one REDUX.MAX per warp on the order-preserving
      // integer image of the scaled max (max(x * scale) == max(x) * scale), then
      // one shared atomicMax per warp
#pragma unroll
      for (int x = 0; x < GT; ++x) {
        const int m = __reduce_max_sync(0xffffffffu, float_to_ordered(mx[x] * scale));
        if (lane == 0 && (BM == 128 || j * GT + x < A)) atomicMax(&vals[j * GT + x], m);
      }
    }

    // ---- order statistics of this row of gate-tile maxima (calibration.py:116-153)
    // (b_m = 64: each block sorts its own row with its 64 threads)
    constexpr int NT = BM;  // threads per query block
    const int rt = BM == 64 ? (r & 63) : r;
    const int bar_id = BM == 64 ? 6 + 2 * s + hf : 3 + s;
    // query blocks past the sample's reference grid (the kernel pads to 128 rows) add nothing
    const int blk_valid = p.valid_len / BM;  // valid_len = the sample's padded length (a multiple of lcm(b_m, b_n))
    const bool live = blk < blk_valid;
    named_bar_sync(bar_id, NT);
    if (p.c_maxima && live) {
      float* out = p.c_maxima + ((long long)hq * (p.num_q_tiles * NBLK) + blk) * p.gate_cols;
      for (int x = rt; x < A; x += NT) out[x] = ordered_to_float(vals[x]);
    }
    int n2 = 1;
    while (n2 < A) n2 <<= 1;
    for (int kk = 2; kk <= n2; kk <<= 1) {
      for (int jj = kk >> 1; jj > 0; jj >>= 1) {
        for (int x = rt; x < n2; x += NT) {
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
        named_bar_sync(bar_id, NT);
      }
    }
    if (live && rt < p.c_num_levels) {
      const int k = p.c_levels[rt];
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
      const long long idx = (((long long)rt * p.c_num_layers + p.c_layer) * p.heads_q + hq) * p.c_positions + blk;
      if (isfinite(cut)) {
        p.c_sum[idx] += (double)cut;
        p.c_fin[idx] += 1;
      } else if (cut < 0.f) {
        p.c_neg[idx] += 1;
      } else {
        p.c_pos[idx] += 1;
      }
      if (tie) atomicAdd(&p.c_ties[rt], 1ull);
    }
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  } else {
    setmaxnreg_dec<C::REG_OTHER>();
    named_bar_arrive(15, C::NUM_THREADS);
    return;
  }
}

}  // namespace bsfa
