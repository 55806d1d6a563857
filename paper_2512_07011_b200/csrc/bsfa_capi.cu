// C ABI (include/bsfa_b200.h): argument checking, TMA descriptor encoding and
// kernel dispatch.  No torch types cross this boundary.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/bsfa_b200.h"
#include "bsfa_calib.cuh"    // K2: calibration block maxima + cutoffs
#include "bsfa_fwd3.cuh"     // K1: forward (two query tiles per CTA, one shared S, P in TMEM)
#define BSFA_FWD_KERNEL bsfa_fwd3_kernel
#define BSFA_FWD_CFG FCfg3
// Measurement builds only (-DBSFA_FWD_PAIR=1, tools/build_variants.sh): head_dim
// 128 with an even GQA group on CTA pairs, experimental/csrc/bsfa_fwd7.cuh
// (measured 45 % slower); the production library does
// not contain it.
#ifndef BSFA_FWD_PAIR
#define BSFA_FWD_PAIR 0
#endif
#if BSFA_FWD_PAIR
#include "../../experimental/csrc/bsfa_fwd7.cuh"
#endif
// Measurement builds only (-DBSFA_FWD8=1): ThresholdGate at 128x64 on 64-key
// steps with a per-tile score buffer, experimental/csrc/bsfa_fwd8.cuh
#ifndef BSFA_FWD8
#define BSFA_FWD8 0
#endif
#if BSFA_FWD8
#include "../../experimental/csrc/bsfa_fwd8.cuh"
#endif
// The round-1 forward and the other measured alternatives live in
// experimental/csrc (not built); DESIGN.md section 5 has their numbers.

static_assert(BSFA_MAX_O_PEERS == sizeof(bsfa::KernelParams::o_peer) / sizeof(void*), "peer slots");

using namespace bsfa;

namespace {

thread_local std::string g_last_error;
long long* g_trace = nullptr;  // debug timeline buffer (bsfa_debug_trace)
int g_trace_cta = -1;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(BSFA_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point, so the
// library does not link libcuda directly.
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

// 4-D bf16 view (head_dim, seq, heads, batch) with a {64, rows, 1, 1} box and
// 128-byte swizzle -- the canonical K-major SW128 UMMA operand layout.
int make_map(CUtensorMap* m, const void* base, int d, int n, int h, int bsz, int64_t sn, int64_t sh, int64_t sb,
             int box_rows, const char* name) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return fail(BSFA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the CUDA driver");
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0) return fail(BSFA_ERR_INVALID, "%s: base not 16-byte aligned", name);
  if ((sn * 2) % 16 || (sh * 2) % 16 || (sb * 2) % 16)
    return fail(BSFA_ERR_INVALID, "%s: strides must be multiples of 8 elements", name);
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)n, (cuuint64_t)h, (cuuint64_t)bsz};
  // dims of size 1 still need a valid stride
  cuuint64_t strides[3] = {(cuuint64_t)(sn * 2), (cuuint64_t)((h > 1 ? sh : (int64_t)n * sn) * 2),
                           (cuuint64_t)((bsz > 1 ? sb : (int64_t)h * (h > 1 ? sh : (int64_t)n * sn)) * 2)};
  cuuint32_t box[4] = {64u, (cuuint32_t)box_rows, 1u, 1u};
  cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BSFA_ERR_CUDA, "%s: cuTensorMapEncodeTiled failed (CUresult %d)", name, (int)r);
  return BSFA_OK;
}

// The dynamic shared-memory opt-in is a per-device function attribute: set it
// once per (kernel instantiation, device).
template <auto Kern>
int ensure_smem_attr(int bytes) {
  static bool done[64] = {};  // one array per kernel (template argument)
  auto kern = Kern;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev >= 0 && dev < 64 && done[dev]) return BSFA_OK;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
  if (dev >= 0 && dev < 64) done[dev] = true;
  return BSFA_OK;
}

// calibration kernel K2 (bsfa_calib.cuh)
template <int D, int GT, int BM>
int launch_calib(const CUtensorMap& tq, const CUtensorMap& tk, const KernelParams& p, int grid, cudaStream_t st) {
  using C = CCfg<D, GT, BM>;
  auto kern = bsfa_calib_kernel<D, GT, BM>;
  if (int rc = ensure_smem_attr<bsfa_calib_kernel<D, GT, BM>>(C::SMEM_BYTES)) return rc;
  if (grid == 0) return BSFA_OK;
  kern<<<grid, C::NUM_THREADS, C::SMEM_BYTES, st>>>(tq, tk, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bsfa calibration launch");
  return BSFA_OK;
}

// forward K1 (bsfa_fwd3.cuh)
template <int D, int GT, int BM>
int launch_fwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const KernelParams& p, int grid,
               cudaStream_t st) {
  // gate class and causality are template parameters of the forward kernel;
  // the shared-memory rings (hence the size) depend on the gate class
  const int gm = p.gate_mode == BSFA_GATE_THRESHOLD ? 0 : (p.gate_mode == BSFA_GATE_RUNMAX ? 2 : 1);
  void (*kern)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const KernelParams) = nullptr;
  int rc = BSFA_OK;
  int smem = 0;
  constexpr int threads = BSFA_FWD_CFG<D, GT>::NUM_THREADS;
#define BSFA_GM(GM_, CA_)                                                                     \
  if (gm == GM_ && (p.causal != 0) == CA_) {                                                  \
    kern = BSFA_FWD_KERNEL<D, GT, GM_, CA_, BM>;                                              \
    smem = BSFA_FWD_CFG<D, GT, GM_>::SMEM_BYTES;                                              \
    rc = ensure_smem_attr<BSFA_FWD_KERNEL<D, GT, GM_, CA_, BM>>(smem);                        \
  }
  BSFA_GM(0, true)
  BSFA_GM(0, false)
  BSFA_GM(1, true)
  BSFA_GM(1, false)
  BSFA_GM(2, true)
  BSFA_GM(2, false)
#undef BSFA_GM
  if (rc) return rc;
  if (grid == 0) return BSFA_OK;
  kern<<<grid, threads, smem, st>>>(tq, tk, tv, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bsfa forward launch");
  return BSFA_OK;
}

#if BSFA_FWD_PAIR
// forward K1 on CTA pairs (bsfa_fwd7.cuh): clusters of two, grid = 2 x units
template <int GT>
int launch_fwd7(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const KernelParams& p, int grid,
                cudaStream_t st) {
  using C = FCfg7<GT>;
  const int gm = p.gate_mode == BSFA_GATE_THRESHOLD ? 0 : (p.gate_mode == BSFA_GATE_RUNMAX ? 2 : 1);
  void (*kern)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const KernelParams) = nullptr;
  int rc = BSFA_OK;
#define BSFA_GM7(GM_, CA_)                                                  \
  if (gm == GM_ && (p.causal != 0) == CA_) {                               \
    kern = bsfa_fwd7_kernel<GT, GM_, CA_>;                                 \
    rc = ensure_smem_attr<bsfa_fwd7_kernel<GT, GM_, CA_>>(C::SMEM_BYTES);  \
  }
  BSFA_GM7(0, true)
  BSFA_GM7(0, false)
  BSFA_GM7(1, true)
  BSFA_GM7(1, false)
  BSFA_GM7(2, true)
  BSFA_GM7(2, false)
#undef BSFA_GM7
  if (rc) return rc;
  if (grid == 0) return BSFA_OK;
  kern<<<grid, C::NUM_THREADS, C::SMEM_BYTES, st>>>(tq, tk, tv, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bsfa forward (CTA pair) launch");
  return BSFA_OK;
}

#endif

#if BSFA_FWD8
template <int D>
int launch_fwd8(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const KernelParams& p, int grid,
                cudaStream_t st) {
  using C = FCfg8<D>;
  void (*kern)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const KernelParams) =
      p.causal ? bsfa_fwd8_kernel<D, true> : bsfa_fwd8_kernel<D, false>;
  int rc = p.causal ? ensure_smem_attr<bsfa_fwd8_kernel<D, true>>(C::SMEM_BYTES)
                    : ensure_smem_attr<bsfa_fwd8_kernel<D, false>>(C::SMEM_BYTES);
  if (rc) return rc;
  if (grid == 0) return BSFA_OK;
  kern<<<grid, C::NUM_THREADS, C::SMEM_BYTES, st>>>(tq, tk, tv, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bsfa forward (v8) launch");
  return BSFA_OK;
}
#endif

int dispatch_fwd(int d, int b_m, int b_n, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                 const KernelParams& p, int grid, cudaStream_t st) {
#define BSFA_FWD(D_, BM_, BN_) \
  if (d == D_ && b_m == BM_ && b_n == BN_) return launch_fwd<D_, 128 / BN_, BM_>(tq, tk, tv, p, grid, st);
  BSFA_FWD(64, 128, 64)
  BSFA_FWD(128, 128, 64)
  BSFA_FWD(64, 128, 128)
  BSFA_FWD(128, 128, 128)
  BSFA_FWD(64, 64, 64)
  BSFA_FWD(128, 64, 64)
  BSFA_FWD(64, 64, 128)
  BSFA_FWD(128, 64, 128)
  BSFA_FWD(256, 128, 64)
  BSFA_FWD(256, 128, 128)
  BSFA_FWD(256, 64, 64)
  BSFA_FWD(256, 64, 128)
#undef BSFA_FWD
  return fail(BSFA_ERR_INVALID, "no kernel for head_dim=%d tiles %dx%d", d, b_m, b_n);
}

int dispatch_calib(int d, int b_m, int b_n, const CUtensorMap& tq, const CUtensorMap& tk, const KernelParams& p,
                   int grid, cudaStream_t st) {
#define BSFA_CAL(D_, BM_, BN_) \
  if (d == D_ && b_m == BM_ && b_n == BN_) return launch_calib<D_, 128 / BN_, BM_>(tq, tk, p, grid, st);
  BSFA_CAL(64, 128, 64)
  BSFA_CAL(128, 128, 64)
  BSFA_CAL(64, 128, 128)
  BSFA_CAL(128, 128, 128)
  BSFA_CAL(64, 64, 64)
  BSFA_CAL(128, 64, 64)
  BSFA_CAL(64, 64, 128)
  BSFA_CAL(128, 64, 128)
  BSFA_CAL(256, 128, 64)
  BSFA_CAL(256, 128, 128)
  BSFA_CAL(256, 64, 64)
  BSFA_CAL(256, 64, 128)
#undef BSFA_CAL
  return fail(BSFA_ERR_INVALID, "no calibration kernel for head_dim=%d tiles %dx%d", d, b_m, b_n);
}

// b_m in {64, 128} x b_n in {64, 128}: the reference's 128x64 default and the
// 64x64 / 64x128 / 128x128 tilings of its tests (tiling.py:26-32 admits any pair
// where one size divides the other)
int check_tiles(int b_m, int b_n) {
  if ((b_m != 128 && b_m != 64) || (b_n != 64 && b_n != 128))
    return fail(BSFA_ERR_INVALID,
                "unsupported tiles %dx%d: the sm_100a kernel implements b_m in {64,128}, b_n in {64,128}", b_m, b_n);
  return BSFA_OK;
}

}  // namespace

extern "C" {

int bsfa_abi_version(void) { return BSFA_ABI_VERSION; }

const char* bsfa_last_error(void) { return g_last_error.c_str(); }

int bsfa_device_supported(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return 0;
  return prop.major == 10 && prop.minor == 0 ? 1 : 0;
}

#if BSFA_WATCHDOG_RECORD
// debug builds only: stuck waits recorded by the watchdog (count, then records)
extern "C" int bsfa_debug_stuck(unsigned long long* host_out, int n) {
  unsigned cnt = 0;
  cudaMemcpyFromSymbol(&cnt, bsfa_stuck_n, sizeof(cnt));
  cudaMemcpyFromSymbol(host_out, bsfa_stuck, sizeof(unsigned long long) * (n < 64 ? n : 64));
  return (int)cnt;
}
#endif

int bsfa_debug_trace(long long* dev_buf, int cta) {
  g_trace = dev_buf;
  g_trace_cta = cta;
  return BSFA_OK;
}

int bsfa_fwd(const bsfa_fwd_args* a, void* stream) {
  if (!a) return fail(BSFA_ERR_INVALID, "null args");
  if (int rc = check_tiles(a->b_m, a->b_n)) return rc;
  if (a->head_dim != 64 && a->head_dim != 128 && a->head_dim != 256)
    return fail(BSFA_ERR_INVALID, "head_dim %d unsupported (64, 128 or 256; pad smaller heads)", a->head_dim);
  if (a->batch < 1 || a->heads_q < 1 || a->heads_kv < 1 || a->heads_q % a->heads_kv)
    return fail(BSFA_ERR_INVALID, "bad head counts q=%d kv=%d batch=%d", a->heads_q, a->heads_kv, a->batch);
  if (a->seq_len < 128 || a->seq_len % 128)
    return fail(BSFA_ERR_INVALID, "seq_len %d must be a positive multiple of 128 (pad first)", a->seq_len);
  if (a->valid_len < 1 || a->valid_len > a->seq_len) return fail(BSFA_ERR_INVALID, "bad valid_len %d", a->valid_len);
  if (a->gate_mode < 0 || a->gate_mode > 4) return fail(BSFA_ERR_INVALID, "bad gate_mode %d", a->gate_mode);
  if (a->gate_mode == BSFA_GATE_WINDOW && a->gate_window < 0)
    return fail(BSFA_ERR_INVALID, "window must be >= 0, got %d", a->gate_window);
  if (a->gate_mode == BSFA_GATE_THRESHOLD && (!a->thresholds || a->thr_positions < 1))
    return fail(BSFA_ERR_INVALID, "threshold gate needs a [heads_q][positions] threshold array");
  if (!a->q || !a->k || !a->v || !a->o || !a->lse) return fail(BSFA_ERR_INVALID, "null tensor pointer");
  if (reinterpret_cast<uintptr_t>(a->o) % 16 || (a->o_stride_n * 2) % 16)
    return fail(BSFA_ERR_INVALID, "o must be 16-byte aligned per row");

  const int d = a->head_dim, n = a->seq_len;
  CUtensorMap tq, tk, tv;
  if (int rc = make_map(&tq, a->q, d, n, a->heads_q, a->batch, a->q_stride_n, a->q_stride_h, a->q_stride_b, 128, "q"))
    return rc;
  // (measurement builds) CTA pairs, d = 128, even GQA group: each CTA stages 64 keys of a step
  const bool pair = BSFA_FWD_PAIR && d == 128 && (a->heads_q / a->heads_kv) % 2 == 0;
  // (measurement builds) v8: ThresholdGate, 128x64 tiles, 64-key K boxes
  const bool v8 = BSFA_FWD8 && a->gate_mode == BSFA_GATE_THRESHOLD && a->b_m == 128 && a->b_n == 64;
  if (int rc = make_map(&tk, a->k, d, n, a->heads_kv, a->batch, a->k_stride_n, a->k_stride_h, a->k_stride_b,
                        (pair || v8) ? 64 : 128, "k"))
    return rc;
  if (int rc =
          make_map(&tv, a->v, d, n, a->heads_kv, a->batch, a->v_stride_n, a->v_stride_h, a->v_stride_b,
                   64, "v"))
    return rc;

  KernelParams p;
  memset(&p, 0, sizeof(p));
  p.batch = a->batch;
  p.heads_q = a->heads_q;
  p.heads_kv = a->heads_kv;
  p.group = a->heads_q / a->heads_kv;
  p.seq_len = n;
  p.valid_len = a->valid_len;
  p.num_q_tiles = n / 128;
  p.num_steps = n / 128;  // 128-key MMA steps
  p.gate_cols = n / a->b_n;
  p.causal = a->causal ? 1 : 0;
  p.gate_mode = a->gate_mode;
  p.thr_positions = a->thr_positions;
  p.scale = a->scale;
  p.scale_log2 = a->scale * 1.4426950408889634f;
  p.rescale_raw = 8.0f / p.scale_log2;
  p.inject_fault = a->inject_fault;
  p.gate_window = a->gate_window;
  p.gate_lambda = a->gate_lambda;
  p.thr = a->thresholds;
  p.o = reinterpret_cast<__nv_bfloat16*>(a->o);
  p.o_sb = a->o_stride_b;
  p.o_sh = a->o_stride_h;
  p.o_sn = a->o_stride_n;
  if (a->num_o_peers < 0 || a->num_o_peers > BSFA_MAX_O_PEERS)
    return fail(BSFA_ERR_INVALID, "num_o_peers %d outside [0, %d]", a->num_o_peers, BSFA_MAX_O_PEERS);
  p.num_o_peers = a->num_o_peers;
  for (int i = 0; i < a->num_o_peers; ++i) {
    if (!a->o_peers[i] || reinterpret_cast<uintptr_t>(a->o_peers[i]) % 16)
      return fail(BSFA_ERR_INVALID, "o_peers[%d] must be a 16-byte aligned device pointer", i);
    p.o_peer[i] = reinterpret_cast<__nv_bfloat16*>(a->o_peers[i]);
  }
  p.lse = a->lse;
  p.trace = g_trace;
  p.trace_cta = g_trace_cta;
  p.decisions = a->decisions;
  p.counters = a->counters;
  p.status = a->status;

  // two query tiles per CTA: two q heads of one GQA group (even groups), or
  // query blocks 2m+1 and 2m of one q head (odd groups, MHA included)
  p.block_pair = p.group % 2 == 1 ? 1 : 0;
  const int nq = 2;
  // head_dim 256: one query tile per CTA
  const long long grid = d == 256 ? (long long)a->batch * a->heads_q * p.num_q_tiles
                       : p.block_pair ? (long long)a->batch * a->heads_q * ((p.num_q_tiles + 1) / 2)
                                      : (long long)a->batch * (a->heads_q / nq) * p.num_q_tiles;
  if (grid > 0x7fffffffLL) return fail(BSFA_ERR_INVALID, "grid too large");
  (void)nq;
#if BSFA_FWD8
  if (v8) return d == 128 ? launch_fwd8<128>(tq, tk, tv, p, (int)grid, reinterpret_cast<cudaStream_t>(stream))
                          : launch_fwd8<64>(tq, tk, tv, p, (int)grid, reinterpret_cast<cudaStream_t>(stream));
#endif
#if BSFA_FWD_PAIR
  if (pair) {
    if (2 * grid > 0x7fffffffLL) return fail(BSFA_ERR_INVALID, "grid too large");
    if (a->b_n == 64) return launch_fwd7<2>(tq, tk, tv, p, (int)(2 * grid), reinterpret_cast<cudaStream_t>(stream));
    return launch_fwd7<1>(tq, tk, tv, p, (int)(2 * grid), reinterpret_cast<cudaStream_t>(stream));
  }
#endif
  return dispatch_fwd(d, a->b_m, a->b_n, tq, tk, tv, p, (int)grid, reinterpret_cast<cudaStream_t>(stream));
}

int bsfa_calib_blockmax(const bsfa_calib_args* a, void* stream) {
  if (!a) return fail(BSFA_ERR_INVALID, "null args");
  if (int rc = check_tiles(a->b_m, a->b_n)) return rc;
  if (a->head_dim != 64 && a->head_dim != 128 && a->head_dim != 256)
    return fail(BSFA_ERR_INVALID, "head_dim %d unsupported (64, 128 or 256; pad smaller heads)", a->head_dim);
  if (a->heads_q < 1 || a->heads_kv < 1 || a->heads_q % a->heads_kv)
    return fail(BSFA_ERR_INVALID, "bad head counts q=%d kv=%d", a->heads_q, a->heads_kv);
  if (a->seq_len < 128 || a->seq_len % 128)
    return fail(BSFA_ERR_INVALID, "seq_len %d must be a positive multiple of 128 (pad first)", a->seq_len);
  if (a->seq_len / a->b_n > CCfg<64, 2>::MAXA)
    return fail(BSFA_ERR_INVALID, "calibration supports at most %d key blocks per row", CCfg<64, 2>::MAXA);
  if (a->num_levels < 1 || a->num_levels > 16) return fail(BSFA_ERR_INVALID, "1..16 k levels supported");
  if (a->layer < 0 || a->layer >= a->num_layers) return fail(BSFA_ERR_INVALID, "bad layer %d", a->layer);
  const int valid = a->valid_len > 0 ? a->valid_len : a->seq_len;
  if (valid > a->seq_len || valid % a->b_m || valid % a->b_n)
    return fail(BSFA_ERR_INVALID, "valid_len %d must be <= seq_len %d and a multiple of b_m and b_n", valid,
                a->seq_len);
  if (valid / a->b_m > a->num_positions)
    return fail(BSFA_ERR_INVALID, "sample has %d positions > accumulator %d", valid / a->b_m, a->num_positions);
  if (!a->q || !a->k || !a->finite_sum || !a->finite_cnt || !a->neg_cnt || !a->pos_cnt || !a->tie_counts)
    return fail(BSFA_ERR_INVALID, "null pointer");

  const int d = a->head_dim, n = a->seq_len;
  CUtensorMap tq, tk;
  if (int rc = make_map(&tq, a->q, d, n, a->heads_q, 1, a->q_stride_n, a->q_stride_h, 0, 128, "q")) return rc;
  if (int rc = make_map(&tk, a->k, d, n, a->heads_kv, 1, a->k_stride_n, a->k_stride_h, 0,
                       128, "k"))
    return rc;

  KernelParams p;
  memset(&p, 0, sizeof(p));
  p.batch = 1;
  p.heads_q = a->heads_q;
  p.heads_kv = a->heads_kv;
  p.group = a->heads_q / a->heads_kv;
  p.seq_len = n;
  p.valid_len = valid;  // the sample's reference grid; rows past it are kernel padding
  p.num_q_tiles = n / 128;
  p.num_steps = n / 128;
  p.gate_cols = n / a->b_n;
  p.causal = 1;
  p.scale = a->scale;
  p.scale_log2 = a->scale * 1.4426950408889634f;
  p.c_layer = a->layer;
  p.c_num_layers = a->num_layers;
  p.c_positions = a->num_positions;
  p.c_num_levels = a->num_levels;
  for (int i = 0; i < a->num_levels; ++i) {
    if (a->k_levels[i] < 0) return fail(BSFA_ERR_INVALID, "k levels must be >= 0");
    p.c_levels[i] = a->k_levels[i];
  }
  p.c_sum = a->finite_sum;
  p.c_fin = a->finite_cnt;
  p.c_neg = a->neg_cnt;
  p.c_pos = a->pos_cnt;
  p.c_ties = a->tie_counts;
  p.c_maxima = a->block_maxima;

  // odd groups (MHA included): two query blocks of one head per CTA, as in the forward
  p.block_pair = p.group % 2 == 1 ? 1 : 0;
  const int nq = 2;
  const int grid = d == 256       ? a->heads_q * p.num_q_tiles  // one query tile per CTA
                   : p.block_pair ? a->heads_q * ((p.num_q_tiles + 1) / 2)
                                  : (a->heads_q / nq) * p.num_q_tiles;
  (void)nq;
  return dispatch_calib(d, a->b_m, a->b_n, tq, tk, p, grid, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"

// ---------------------------------------------------------------- finalize (K4)
namespace {
__global__ void calib_finalize_kernel(const double* __restrict__ sum, const int32_t* __restrict__ fin,
                                      const int32_t* __restrict__ neg, const int32_t* __restrict__ pos,
                                      float* __restrict__ out, long long count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    float v;
    if (fin[i] > 0)
      v = (float)(sum[i] / (double)fin[i]);
    else if (neg[i] > 0)
      v = -INFINITY;
    else if (pos[i] > 0)
      v = INFINITY;
    else
      v = 0.f;
    out[i] = v;
  }
}
}  // namespace

extern "C" int bsfa_calib_finalize(const double* finite_sum, const int32_t* finite_cnt, const int32_t* neg_cnt,
                                   const int32_t* pos_cnt, float* values, int64_t count, void* stream) {
  if (count < 0 || (count > 0 && (!finite_sum || !finite_cnt || !neg_cnt || !pos_cnt || !values)))
    return fail(BSFA_ERR_INVALID, "bad finalize arguments");
  if (count == 0) return BSFA_OK;
  const int threads = 256;
  long long blocks = (count + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  calib_finalize_kernel<<<(int)blocks, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      finite_sum, finite_cnt, neg_cnt, pos_cnt, values, count);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "finalize launch");
  return BSFA_OK;
}

// ---------------------------------------------------------------- selection (K3)
namespace {
// One CTA per (row, position p): bitonic sort of the A_p tile maxima (order-
// preserving integer image, descending) in shared memory, then per level the
// (k+1)-th largest with the reference's sentinels and tie test.
__global__ void __launch_bounds__(256) calib_select_kernel(const float* __restrict__ bm, int m_q, int m_kv, int b_m,
                                                           int b_n, KernelParams lv, float* __restrict__ thr,
                                                           unsigned long long* __restrict__ ties, long long rows) {
  __shared__ int vals[4096];
  const long long rp = blockIdx.x;  // row * m_q + p
  const int p = int(rp % m_q);
  const long long row = rp / m_q;
  const int a = (int)(((long long)p * b_m) / b_n);
  const float* src = bm + rp * m_kv;
  int n2 = 1;
  while (n2 < a) n2 <<= 1;
  for (int x = threadIdx.x; x < n2; x += blockDim.x)
    vals[x] = x < a ? float_to_ordered(src[x]) : float_to_ordered(-INFINITY);
  __syncthreads();
  for (int kk = 2; kk <= n2; kk <<= 1) {
    for (int jj = kk >> 1; jj > 0; jj >>= 1) {
      for (int x = threadIdx.x; x < n2; x += blockDim.x) {
        const int y = x ^ jj;
        if (y > x) {
          const int u = vals[x], w = vals[y];
          const bool desc = (x & kk) == 0;
          if (desc ? (u < w) : (u > w)) {
            vals[x] = w;
            vals[y] = u;
          }
        }
      }
      __syncthreads();
    }
  }
  if ((int)threadIdx.x < lv.c_num_levels) {
    const int k = lv.c_levels[threadIdx.x];
    float cut;
    bool tie = false;
    if (k == 0) {
      cut = INFINITY;
    } else if (a <= k) {
      cut = -INFINITY;
    } else {
      cut = ordered_to_float(vals[k]);
      tie = vals[k - 1] == vals[k];
    }
    thr[((long long)threadIdx.x * rows + row) * m_q + p] = cut;
    if (tie) atomicAdd(&ties[threadIdx.x], 1ull);
  }
}
}  // namespace

extern "C" int bsfa_calib_select(const float* bm, int64_t rows, int m_q, int m_kv, int b_m, int b_n,
                                 const int32_t* k_levels, int num_levels, float* thr, unsigned long long* ties,
                                 void* stream) {
  if (rows < 0 || m_q < 0 || m_kv < 0 || m_kv > 4096) return fail(BSFA_ERR_INVALID, "bad grid %lld x %d x %d", (long long)rows, m_q, m_kv);
  if (b_m < 1 || b_n < 1 || (b_m % b_n && b_n % b_m)) return fail(BSFA_ERR_INVALID, "bad tiles %dx%d", b_m, b_n);
  if (num_levels < 1 || num_levels > 16 || !k_levels) return fail(BSFA_ERR_INVALID, "1..16 k levels supported");
  if ((long long)(m_q - 1) * b_m / b_n > m_kv) return fail(BSFA_ERR_INVALID, "grid narrower than the causal prefix");
  if (rows * (long long)m_q == 0) return BSFA_OK;
  if (!bm || !thr || !ties) return fail(BSFA_ERR_INVALID, "null pointer");
  KernelParams lv;
  memset(&lv, 0, sizeof(lv));
  lv.c_num_levels = num_levels;
  for (int i = 0; i < num_levels; ++i) {
    if (k_levels[i] < 0) return fail(BSFA_ERR_INVALID, "k levels must be >= 0");
    lv.c_levels[i] = k_levels[i];
  }
  const long long grid = rows * (long long)m_q;
  if (grid > 0x7fffffffLL) return fail(BSFA_ERR_INVALID, "grid too large");
  calib_select_kernel<<<(int)grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(bm, m_q, m_kv, b_m, b_n, lv, thr,
                                                                                     ties, rows);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "calib_select launch");
  return BSFA_OK;
}
