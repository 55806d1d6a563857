/*
 * bsfa_b200.h -- C ABI of the B200-native Block-Sparse FlashAttention path.
 *
 * Plain pointers and sizes only (no torch / numpy types).  Every device
 * pointer is a CUDA global-memory address on the current device; `stream` is
 * a cudaStream_t (NULL = legacy default stream).  All entry points are
 * asynchronous w.r.t. the host and return 0 on success or a negative
 * BSFA_ERR_* code; bsfa_last_error() returns a message for the calling thread.
 *
 * Which reference interface each entry point replaces (paths relative to the
 * reference package, pkg/src/bsfa/):
 *
 *   bsfa_fwd              engine.py:117-193  flash_forward(inp, tiles, gate, ctx)
 *                         with gates.py:41-78 ThresholdGate / DenseGate /
 *                         FrontierOnlyGate compiled into the kernel and the
 *                         threshold lookup thresholds.py:75-88 done per CTA.
 *                         Batched over (batch, q head) with GQA; the trace
 *                         codes of engine.py:22-25 are written to `decisions`.
 *   bsfa_calib_blockmax   calibration.py:93-123 collect_block_maxima (tile
 *                         maxima of the off-frontier causal prefix), fused with
 *                         calibration.py:126-153 thresholds_from_maxima /
 *                         _tie_count and the per-sample accumulation loop of
 *                         calibration.py:185-196.
 *   bsfa_calib_finalize   calibration.py:201-205 (finite mean in fp64, sentinel
 *                         rules, float32 cast).
 *   bsfa_calib_select     calibration.py:126-153 thresholds_from_maxima /
 *                         _tie_count over an explicit tile-maxima grid (the
 *                         torch.ops.bsfa.calib_select operator).
 */
#ifndef BSFA_B200_H
#define BSFA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSFA_ABI_VERSION 6

/* error codes */
#define BSFA_OK 0
#define BSFA_ERR_INVALID (-1)     /* bad argument: shape, alignment, unsupported config */
#define BSFA_ERR_CUDA (-2)        /* CUDA runtime / driver failure                       */
#define BSFA_ERR_UNSUPPORTED (-3) /* device is not sm_100                                */

/* gate modes (reference gates.py) */
#define BSFA_GATE_THRESHOLD 0 /* ThresholdGate: keep iff tile max (scaled) > T   gates.py:59-78 */
#define BSFA_GATE_DENSE 1     /* DenseGate: keep every reachable tile            gates.py:41-47 */
#define BSFA_GATE_FRONTIER 2  /* FrontierOnlyGate: skip every off-frontier tile  gates.py:50-56 */
#define BSFA_GATE_WINDOW 3    /* SlidingWindowGate(gate_window tokens)          gates.py:81-98  */
#define BSFA_GATE_RUNMAX 4    /* RunningMaxGate(gate_lambda)                    gates.py:101-118 */

/* counters written by bsfa_fwd (accumulated with atomics, caller zeroes) */
#define BSFA_CNT_REACHABLE 0 /* reachable gate tiles (frontier included)        */
#define BSFA_CNT_KEPT 1      /* processed gate tiles (frontier + kept)          */
#define BSFA_CNT_VLOADS 2    /* V gate tiles fetched by TMA (one fetch serves    */
                             /* every query tile of a CTA that kept the tile)  */
#define BSFA_CNT_VUNITS 3    /* V gate tiles a CTA could have fetched           */

#define BSFA_MAX_O_PEERS 7 /* a gather over up to 8 GPUs */

typedef struct bsfa_fwd_args {
  /* inputs: bf16 [batch][heads][seq][head_dim], arbitrary element strides with
     unit stride on head_dim and 16-byte aligned rows */
  const void* q;
  const void* k;
  const void* v;
  int64_t q_stride_b, q_stride_h, q_stride_n;
  int64_t k_stride_b, k_stride_h, k_stride_n;
  int64_t v_stride_b, v_stride_h, v_stride_n;
  /* outputs */
  void* o; /* bf16, layout given by o_stride_* */
  int64_t o_stride_b, o_stride_h, o_stride_n;
  float* lse;        /* fp32 [batch][heads_q][seq_len], natural log, scaled-score units */
  int8_t* decisions; /* optional int8 [batch][heads_q][seq_len/b_m][seq_len/b_n]; caller zeroes */
  /* tiles: b_m in {64, 128}, b_n in {64, 128}; seq_len a multiple of 128 (pad
     by repeating the last row); valid_len = unpadded length.  With b_m = 64 the
     counters count only the reference grid padded to lcm(b_m, b_n).  head_dim
     in {64, 128, 256} (zero-pad narrower heads; scale from the original d). */
  unsigned long long* counters; /* optional [4], see BSFA_CNT_* */
  int* status; /* optional; bit 0 set if any row has a non-finite accumulator or l <= 0 */
  /* gate */
  const float* thresholds; /* fp32 [heads_q][thr_positions] (one level, one layer) */
  int thr_positions;
  int gate_mode;
  /* geometry */
  int batch, heads_q, heads_kv, seq_len, valid_len, head_dim;
  int b_m, b_n;
  int causal;
  float scale; /* fp32(1/sqrt(original head_dim)) */
  int inject_fault;
  int gate_window;   /* BSFA_GATE_WINDOW: trailing window w >= 0 (tokens) */
  float gate_lambda; /* BSFA_GATE_RUNMAX: keep iff max_rows(local - running max) >= lambda */
  /* extra O destinations written by the epilogue with o's strides and the same
     element offsets (e.g. other GPUs' gathered-O buffers mapped over NVLink), so
     a head-sharded forward needs no separate all-gather; 0..BSFA_MAX_O_PEERS */
  int num_o_peers;
  void* o_peers[BSFA_MAX_O_PEERS];
} bsfa_fwd_args;

typedef struct bsfa_calib_args {
  /* one layer of one calibration sample: bf16 q [heads_q][seq][d], k [heads_kv][seq][d] */
  const void* q;
  const void* k;
  int64_t q_stride_h, q_stride_n;
  int64_t k_stride_h, k_stride_n;
  int heads_q, heads_kv, seq_len, head_dim; /* seq_len: this sample's padded length */
  int b_m, b_n;
  float scale;
  /* accumulator geometry: [num_levels][num_layers][heads_q][num_positions] */
  int layer, num_layers, num_positions;
  int num_levels;
  int k_levels[16];
  double* finite_sum;
  int32_t* finite_cnt;
  int32_t* neg_cnt;
  int32_t* pos_cnt;
  unsigned long long* tie_counts; /* [num_levels] */
  /* optional raw tile maxima fp32 [heads_q][seq_len/b_m][seq_len/b_n] (unsorted,
     scaled units); entries outside the off-frontier prefix are left untouched */
  float* block_maxima;
  /* the sample's padded length in the reference grid (a multiple of b_m and b_n,
     <= seq_len; 0 = seq_len): query blocks past it (seq_len is padded further
     to a multiple of 128 for the kernel) contribute nothing.  ABI 6. */
  int valid_len;
} bsfa_calib_args;

int bsfa_abi_version(void);
const char* bsfa_last_error(void);
/* 1 if the current device can run the kernels (sm_100 family), else 0. */
int bsfa_device_supported(void);

int bsfa_fwd(const bsfa_fwd_args* args, void* stream);
/* Debug: in a library built with -DBSFA_TRACE=1, subsequent bsfa_fwd launches
   record per-step clock64 timestamps of CTA `cta` into dev_buf
   (int64 [6 events][2 query tiles][2048 steps]); NULL disables.  The
   production build ignores the buffer. */
int bsfa_debug_trace(long long* dev_buf, int cta);
int bsfa_calib_blockmax(const bsfa_calib_args* args, void* stream);
int bsfa_calib_finalize(const double* finite_sum, const int32_t* finite_cnt, const int32_t* neg_cnt,
                        const int32_t* pos_cnt, float* values, int64_t count, void* stream);
/* Per (row, query position p) of a tile-maxima grid bm fp32 [rows][m_q][m_kv]
   (scaled units, e.g. the block_maxima of bsfa_calib_blockmax), take the first
   A_p = p * b_m / b_n entries (the off-frontier causal prefix, tiling.py:63-65),
   and for each level k write the (k+1)-th largest (+inf for k = 0, -inf when
   A_p <= k) to thr fp32 [num_levels][rows][m_q]; ties[s] (zeroed by the
   caller) += positions where vals[k-1] == vals[k] (calibration.py:126-153).
   m_kv <= 4096; 1 <= num_levels <= 16. */
int bsfa_calib_select(const float* bm, int64_t rows, int m_q, int m_kv, int b_m, int b_n, const int32_t* k_levels,
                      int num_levels, float* thr, unsigned long long* ties, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BSFA_B200_H */
