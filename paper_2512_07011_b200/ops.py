"""``torch.ops.bsfa`` custom operators over the C ABI (SURVEY §8(b) op contract).

* ``bsfa::fwd(q, k, v, thr, causal, b_m, b_n, scale, want_trace)
  -> (o, lse, counters, decisions)``: one ``bsfa_fwd`` launch.  ``thr`` is the
  fp32 [Hq, P] slice ``values[level, layer]`` of a ThresholdTensor (one
  threshold per (q head, query block), clamped at P - 1 as thresholds.py:87),
  or an empty tensor for the DenseGate.  ``counters`` is int64 [4] (reachable,
  kept, V tiles loaded, V tiles loadable); ``decisions`` the int8 code grid
  [B, Hq, M_q, M_kv] (engine.py:22-25) when ``want_trace``, else empty.
* ``bsfa::blockmax(q, k, b_m, b_n) -> bm``: fp32 [B, Hq, M_q, M_kv] of scaled
  tile maxima over the off-frontier causal prefix j < A_i
  (calibration.py:93-123), -inf elsewhere -- the calibration kernel (K2).
* ``bsfa::calib_select(bm, k_levels) -> (thr, ties)``: per (head, position)
  the (k+1)-th largest tile maximum with the reference's sentinels
  (calibration.py:126-153): thr fp32 [S, B, Hq, M_q], ties int64 [S] -- one
  ``bsfa_calib_select`` launch (K3: a bitonic sort per (head, position) in
  shared memory).

The ops carry fake (meta) implementations, so they trace under
``torch.compile`` / ``torch.export`` without running the kernel.  Only CUDA
kernels are registered: the dispatcher refuses CPU tensors (no fallback).
The calibration path itself (``calibrate`` / ``Calibrator``) fuses maxima,
selection and accumulation in one kernel (K2); ``blockmax`` + ``calib_select``
expose the two halves separately.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .attention import _check_inputs, _forward
from .calibration import Calibrator
from .errors import ConfigurationError, InvalidInputError
from .tiling import TileConfig, kernel_len, require_kernel_tiles

Tensor = torch.Tensor


@torch.library.custom_op("bsfa::fwd", mutates_args=(), device_types="cuda")
def fwd(q: Tensor, k: Tensor, v: Tensor, thr: Tensor, causal: bool, b_m: int, b_n: int, scale: float,
        want_trace: bool) -> tuple[Tensor, Tensor, Tensor, Tensor]:
    _check_inputs(q, k, v)
    tiles = TileConfig(b_m, b_n)
    require_kernel_tiles(tiles)
    if thr.numel() == 0:
        thr_dev, mode = None, _lib.GATE_DENSE
    else:
        if thr.dim() != 2 or thr.shape[0] != q.shape[1] or thr.dtype != torch.float32 or thr.device != q.device:
            raise InvalidInputError(f"thr must be fp32 [Hq={q.shape[1]}, P] on {q.device}, got "
                                    f"{thr.dtype} {tuple(thr.shape)} on {thr.device}")
        thr_dev, mode = thr.contiguous(), _lib.GATE_THRESHOLD
    res = _forward(q, k, v, thr_dev, mode, 0, 0.0, causal=causal, tiles=tiles, return_trace=want_trace,
                   scale=scale)
    o = res.o if res.o.is_contiguous() else res.o.contiguous()
    lse = res.lse if res.lse.is_contiguous() else res.lse.contiguous()
    dec = res.decisions if want_trace else q.new_empty((0,), dtype=torch.int8)
    return o, lse, res.counters, dec


@fwd.register_fake
def _fwd_fake(q, k, v, thr, causal, b_m, b_n, scale, want_trace):
    b, h, n, d = q.shape
    n_pad = TileConfig(b_m, b_n).padded_len(n)
    o = q.new_empty((b, h, n, d), dtype=torch.bfloat16)
    lse = q.new_empty((b, h, n), dtype=torch.float32)
    counters = q.new_empty((4,), dtype=torch.int64)
    dec = (q.new_empty((b, h, n_pad // b_m, n_pad // b_n), dtype=torch.int8) if want_trace
           else q.new_empty((0,), dtype=torch.int8))
    return o, lse, counters, dec


@torch.library.custom_op("bsfa::blockmax", mutates_args=(), device_types="cuda")
def blockmax(q: Tensor, k: Tensor, b_m: int, b_n: int) -> Tensor:
    _check_inputs(q, k, k)
    tiles = TileConfig(b_m, b_n)
    require_kernel_tiles(tiles)
    b, h, n, d = q.shape
    n_pad, n_kern = tiles.padded_len(n), kernel_len(n, tiles)
    out = torch.full((b, h, n_kern // b_m, n_kern // b_n), float("-inf"), dtype=torch.float32, device=q.device)
    for bi in range(b):
        cal = Calibrator([0], tiles, 1, h, n, d, device=q.device)
        cal.add_layer(0, 0, q[bi], k[bi], seq_len=n, block_maxima=out[bi])
    if n_kern != n_pad:  # the reference grid (b_m = 64, odd block count)
        out = out[:, :, : n_pad // b_m, : n_pad // b_n].contiguous()
    return out


@blockmax.register_fake
def _blockmax_fake(q, k, b_m, b_n):
    b, h, n, _ = q.shape
    n_pad = TileConfig(b_m, b_n).padded_len(n)
    return q.new_empty((b, h, n_pad // b_m, n_pad // b_n), dtype=torch.float32)


@torch.library.custom_op("bsfa::calib_select", mutates_args=(), device_types="cuda")
def calib_select(bm: Tensor, k_levels: list[int], b_m: int, b_n: int) -> tuple[Tensor, Tensor]:
    if bm.dim() != 4 or bm.dtype != torch.float32:
        raise InvalidInputError(f"bm must be fp32 [B, H, M_q, M_kv], got {bm.dtype} {tuple(bm.shape)}")
    if not k_levels or any(x < 0 for x in k_levels) or any(a >= c for a, c in zip(k_levels, k_levels[1:])):
        raise ConfigurationError(f"k levels must be non-negative and strictly increasing: {list(k_levels)}")
    if not bm.is_cuda:
        raise InvalidInputError("calib_select runs on CUDA tensors only (no CPU fallback)")
    if len(k_levels) > 16:
        raise ConfigurationError("at most 16 sparsity levels")
    b, h, m_q, m_kv = bm.shape
    src = bm.contiguous()
    thr = torch.empty((len(k_levels), b, h, m_q), dtype=torch.float32, device=bm.device)
    ties = torch.zeros(len(k_levels), dtype=torch.int64, device=bm.device)
    levels = (ctypes.c_int32 * len(k_levels))(*[int(x) for x in k_levels])
    with torch.cuda.device(bm.device):
        stream = torch.cuda.current_stream(bm.device).cuda_stream
        _lib.check(_lib.load_library().bsfa_calib_select(
            src.data_ptr(), b * h, m_q, m_kv, b_m, b_n, levels, len(k_levels), thr.data_ptr(), ties.data_ptr(),
            ctypes.c_void_p(stream)), "bsfa_calib_select")
    return thr, ties


@calib_select.register_fake
def _calib_select_fake(bm, k_levels, b_m, b_n):
    return (bm.new_empty((len(k_levels),) + tuple(bm.shape[:3]), dtype=torch.float32),
            bm.new_empty((len(k_levels),), dtype=torch.int64))
