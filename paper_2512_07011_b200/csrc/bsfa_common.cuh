// Shared definitions of the sm_100a BSFA kernels: launch parameters (filled by
// bsfa_capi.cu from the C-ABI argument structs), gate modes, the statically
// known decision bits of a step, and the O store with its peer copies.
#pragma once

#include "ptx.cuh"

// Debug timeline (bsfa_debug_trace); compiled out of the production library.
#ifndef BSFA_TRACE
#define BSFA_TRACE 0
#endif
// Fraction of exponentials computed by polynomial on the FMA pipe instead of
// the MUFU: 0 = none (measured fastest), 1 = 1/4, 2 = 1/2.
#ifndef BSFA_EXP_EMU
#define BSFA_EXP_EMU 0
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

// b_m = 64 (a 128-row query tile holds query blocks 2t and 2t+1): the gate
// tiles x of step j for 64-row query block `blk` (tiling.py:50-65, engine.py:
// 152-174): `reach` = causally reachable, `front` = frontier (always kept,
// causal mask on its elements), `smask` = decided without a vote, `sval` =
// their keep bits.  Gate columns / blocks past the reference's padded grid
// (kernel padding to 128 rows) are computed like any other and only left out
// of the counters and the cropped trace.
struct StepBits64 {
  uint32_t reach, front, smask, sval;
};
template <int GT>
__device__ __forceinline__ StepBits64 step_bits64(int gate_mode, int window, bool causal, int j, int blk) {
  constexpr int BN = 128 / GT;
  const int f_lo = (blk * 64) / BN, f_hi = (blk * 64 + 64 + BN - 1) / BN;
  StepBits64 r{0u, 0u, 0u, 0u};
#pragma unroll
  for (int x = 0; x < GT; ++x) {
    const int g = j * GT + x;
    const uint32_t bit = 1u << x;
    if (causal && g >= f_hi) {  // unreachable: statically not kept
      r.smask |= bit;
      continue;
    }
    r.reach |= bit;
    if (g >= f_lo && g < f_hi) {
      r.front |= bit;
      r.smask |= bit;
      r.sval |= bit;
    } else if (gate_mode == kGateDense) {
      r.smask |= bit;
      r.sval |= bit;
    } else if (gate_mode == kGateFrontier) {
      r.smask |= bit;
    } else if (gate_mode == kGateWindow) {  // gates.py:96-98 with b_m = 64
      r.smask |= bit;
      if ((g + 1) * BN > blk * 64 - window && g * BN < (blk + 1) * 64) r.sval |= bit;
    }  // ThresholdGate / RunningMaxGate: voted
  }
  return r;
}

}  // namespace bsfa
