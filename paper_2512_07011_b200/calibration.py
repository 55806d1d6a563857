"""Threshold calibration on sm_100a.

Reference pkg/src/bsfa/calibration.py:93-222: for every (layer, head,
query-block position p) take the off-frontier tile maxima of the causal
prefix (j < A_p), sort descending, cut at the (k+1)-th largest value
(sentinels: k = 0 -> +inf, fewer than k+1 tiles -> -inf), average the
cutoffs over samples in sample-id order in fp64 (a position whose samples
are all sentinels takes -inf if any is -inf, else +inf), cast to float32.

Here the tile maxima, the per-row selection, the tie test and the fp64
accumulation are one kernel launch per (sample, layer) (``bsfa_calib_blockmax``,
same QK^T / rowmax code as the forward kernel, so calibration and inference
see bit-identical block maxima on the GPU), and the mean/sentinel rule is
``bsfa_calib_finalize``.  Samples may be GQA-shaped (k with fewer heads); q
head h then reads kv head h // (Hq/Hkv).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .attention import head_dim_pad, reference_scale
from .errors import ConfigurationError, InvalidInputError
from .thresholds import ThresholdTensor
from .tiling import TileConfig, kernel_len, off_frontier_count, require_kernel_tiles


def _to_array(x):
    if isinstance(x, torch.Tensor):
        return x
    if isinstance(x, np.ndarray) and x.dtype == np.float32:
        return x  # views (e.g. memory-mapped dump blobs) stay lazy; uploads copy per layer
    return np.ascontiguousarray(x, dtype=np.float32)


@dataclass
class CalibrationSample:
    """One calibration input: q (L, Hq, N, d), k (L, Hkv, N, d) (calibration.py:26-50).

    Arrays may be numpy (uploaded per layer) or torch tensors (used in place
    when already on the GPU).
    """

    sample_id: int
    q: object
    k: object
    v: object | None = None

    def __post_init__(self):
        self.q = _to_array(self.q)
        self.k = _to_array(self.k)
        if self.v is not None:
            self.v = _to_array(self.v)
        qs, ks = tuple(self.q.shape), tuple(self.k.shape)
        if len(qs) != 4 or len(ks) != 4 or qs[0] != ks[0] or qs[2:] != ks[2:] \
                or ks[1] < 1 or qs[1] % ks[1]:
            raise InvalidInputError(
                f"sample {self.sample_id}: q/k must be 4-D (L, H, N, d) with matching L, N, d "
                f"and Hq a multiple of Hkv, got {qs} and {ks}")
        if self.v is not None and tuple(self.v.shape) != ks:
            raise InvalidInputError(f"sample {self.sample_id}: v shape {tuple(self.v.shape)} differs from k")

    @property
    def seq_len(self) -> int:
        return int(self.q.shape[2])


@dataclass
class CalibrationDump:
    num_layers: int
    num_heads: int
    head_dim: int
    samples: list = field(default_factory=list)

    def __post_init__(self):
        for s in self.samples:
            L, H, _, d = s.q.shape
            if (L, H, d) != (self.num_layers, self.num_heads, self.head_dim):
                raise ConfigurationError(
                    f"sample {s.sample_id} shape {tuple(s.q.shape)} inconsistent with dump "
                    f"(L={self.num_layers}, H={self.num_heads}, d={self.head_dim})")


@dataclass
class BlockMaximaProfile:
    """Descending tile maxima per (layer, head, position) (calibration.py:70-77)."""

    num_layers: int
    num_heads: int
    num_positions: int
    maxima: dict


@dataclass
class CalibrationDiagnostics:
    num_samples: int
    tie_counts: dict
    threshold_stats: dict


def _head_operand(x, n_pad: int, d_pad: int, device) -> torch.Tensor:
    """[H, N, d] numpy/torch -> bf16 [H, n_pad, d_pad] on `device` (rows repeated, d zero-padded).

    A bf16 device tensor of the padded shape with 16-byte aligned rows is used
    as is (no copy); anything else is rounded to bf16 once (RNE, as the
    forward does) and padded.
    """
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    t = t.to(device=device, non_blocking=True).to(torch.bfloat16)
    n = t.shape[1]
    if n != n_pad:
        t = torch.cat([t, t[:, n - 1:n].expand(-1, n_pad - n, -1)], dim=1)
    if t.shape[2] != d_pad:
        t = torch.nn.functional.pad(t, (0, d_pad - t.shape[2]))
    if t.stride(2) != 1 or (t.stride(1) * 2) % 16 or (t.stride(0) * 2) % 16 or t.data_ptr() % 16:
        t = t.contiguous()
    return t


class Calibrator:
    """Streaming GPU calibration: feed (sample, layer) slices in sample-id order.

    ``calibrate`` uses this for in-memory dumps; large synthetic or on-device
    calibration sets call :meth:`add_layer` directly so a full sample never
    has to exist on the host.
    """

    def __init__(self, k_levels, tiles: TileConfig, num_layers: int, num_heads: int, n_max: int,
                 head_dim: int, device=None):
        k_levels = [int(k) for k in k_levels]
        if not k_levels:
            raise ConfigurationError("need at least one sparsity level")
        if any(b <= a for a, b in zip(k_levels, k_levels[1:])):
            raise ConfigurationError(f"k levels must be strictly increasing: {k_levels}")
        if k_levels[0] < 0:
            raise ConfigurationError(f"k must be >= 0, got {k_levels[0]}")
        if len(k_levels) > 16:
            raise ConfigurationError("at most 16 sparsity levels per calibration")
        require_kernel_tiles(tiles)
        self.k_levels = k_levels
        self.tiles = tiles
        self.num_layers = num_layers
        self.num_heads = num_heads
        self.head_dim = head_dim
        self.n_max = tiles.padded_len(n_max)
        self.num_positions = self.n_max // tiles.b_m
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        shape = (len(k_levels), num_layers, num_heads, self.num_positions)
        dev = self.device
        self.sum = torch.zeros(shape, dtype=torch.float64, device=dev)
        self.fin = torch.zeros(shape, dtype=torch.int32, device=dev)
        self.neg = torch.zeros(shape, dtype=torch.int32, device=dev)
        self.pos = torch.zeros(shape, dtype=torch.int32, device=dev)
        self.ties = torch.zeros(len(k_levels), dtype=torch.int64, device=dev)
        self.nonfinite = torch.zeros((), dtype=torch.bool, device=dev)
        self.covered = np.zeros((num_layers, self.num_positions), dtype=bool)  # per (layer, position)
        self.sample_ids = []
        self._last = None

    def add_layer(self, sample_id: int, layer: int, q, k, seq_len: int | None = None,
                  block_maxima: torch.Tensor | None = None) -> None:
        """q [Hq, N, d], k [Hkv, N, d] of one (sample, layer); any float dtype/device.

        ``block_maxima`` (optional) receives the raw tile maxima on the kernel
        grid, fp32 [Hq, n_kern / b_m, n_kern / b_n], n_kern = kernel_len(N).
        """
        key = (int(sample_id), int(layer))
        if self._last is not None and key[0] < self._last[0]:
            raise ConfigurationError("samples must be added in non-decreasing sample-id order")
        self._last = key
        if not self.sample_ids or self.sample_ids[-1] != key[0]:
            self.sample_ids.append(key[0])
        n = int(q.shape[1]) if seq_len is None else int(seq_len)
        n_pad = self.tiles.padded_len(n)   # the reference grid of this sample
        n_kern = kernel_len(n, self.tiles)  # rounded up to the kernel's 128 rows
        if n_pad > self.n_max:
            raise ConfigurationError(f"sample length {n} exceeds calibrator n_max {self.n_max}")
        d_pad = head_dim_pad(self.head_dim)
        qd = _head_operand(q, n_kern, d_pad, self.device)
        kd = _head_operand(k, n_kern, d_pad, self.device)
        if qd.shape[0] != self.num_heads:
            raise ConfigurationError(f"layer has {qd.shape[0]} q heads, calibrator expects {self.num_heads}")
        self.nonfinite |= ~(torch.isfinite(qd).all() & torch.isfinite(kd).all())
        if not 0 <= layer < self.num_layers:
            raise ConfigurationError(f"layer {layer} outside the calibrator's {self.num_layers} layers")
        self.covered[layer, : n_pad // self.tiles.b_m] = True
        a = _lib.CalibArgs()
        a.q, a.k = qd.data_ptr(), kd.data_ptr()
        a.q_stride_h, a.q_stride_n = qd.stride(0), qd.stride(1)
        a.k_stride_h, a.k_stride_n = kd.stride(0), kd.stride(1)
        a.heads_q, a.heads_kv, a.seq_len, a.head_dim = qd.shape[0], kd.shape[0], n_kern, d_pad
        a.valid_len = n_pad
        a.b_m, a.b_n = self.tiles.b_m, self.tiles.b_n
        a.scale = reference_scale(self.head_dim)
        a.layer, a.num_layers, a.num_positions = layer, self.num_layers, self.num_positions
        a.num_levels = len(self.k_levels)
        for i, kv in enumerate(self.k_levels):
            a.k_levels[i] = kv
        a.finite_sum, a.finite_cnt = self.sum.data_ptr(), self.fin.data_ptr()
        a.neg_cnt, a.pos_cnt = self.neg.data_ptr(), self.pos.data_ptr()
        a.tie_counts = self.ties.data_ptr()
        if block_maxima is not None:
            want = (qd.shape[0], n_kern // self.tiles.b_m, n_kern // self.tiles.b_n)
            if (tuple(block_maxima.shape) != want or block_maxima.dtype != torch.float32
                    or block_maxima.device != qd.device or not block_maxima.is_contiguous()):
                raise InvalidInputError(f"block_maxima must be contiguous fp32 {want} on {qd.device}, got "
                                        f"{block_maxima.dtype} {tuple(block_maxima.shape)} on {block_maxima.device}")
        a.block_maxima = block_maxima.data_ptr() if block_maxima is not None else None
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device).cuda_stream
            _lib.check(_lib.load_library().bsfa_calib_blockmax(ctypes.byref(a), ctypes.c_void_p(stream)),
                       "bsfa_calib_blockmax")
        # keep operands alive until the stream has consumed them
        self._keep = (qd, kd)

    def finish(self) -> ThresholdTensor:
        if not self.sample_ids:
            raise ConfigurationError("calibration dump has no samples")
        if bool(self.nonfinite.item()):
            raise InvalidInputError("non-finite activations in a calibration sample")
        if not self.covered.all():
            missing = sorted({int(x) for x in np.nonzero(~self.covered.all(axis=1))[0]})
            raise ConfigurationError(
                f"some calibrated (layer, position) pairs are covered by no sample (layers {missing[:8]})")
        vals = torch.empty(self.sum.shape, dtype=torch.float32, device=self.device)
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device).cuda_stream
            _lib.check(_lib.load_library().bsfa_calib_finalize(
                self.sum.data_ptr(), self.fin.data_ptr(), self.neg.data_ptr(), self.pos.data_ptr(),
                vals.data_ptr(), vals.numel(), ctypes.c_void_p(stream)), "bsfa_calib_finalize")
        values = vals.cpu().numpy()
        ties = self.ties.cpu().numpy()
        # a larger budget must never raise the cutoff (calibration.py:207-208)
        assert not (values[1:] > values[:-1]).any(), "threshold monotonicity violated"
        stats = {}
        for si, k in enumerate(self.k_levels):
            fv = values[si][np.isfinite(values[si])]
            stats[k] = (float(fv.min()), float(fv.mean()), float(fv.max())) if fv.size else (None, None, None)
        diag = CalibrationDiagnostics(num_samples=len(self.sample_ids),
                                      tie_counts={k: int(ties[i]) for i, k in enumerate(self.k_levels)},
                                      threshold_stats=stats)
        return ThresholdTensor(values=values, k_levels=tuple(self.k_levels), n_max=self.n_max,
                               b_m=self.tiles.b_m, b_n=self.tiles.b_n, diagnostics=diag)


def calibrate(dump: CalibrationDump, k_levels, tiles: TileConfig, device=None) -> ThresholdTensor:
    """Reference-signature calibration (calibration.py:156-222) on the GPU."""
    if not dump.samples:
        raise ConfigurationError("calibration dump has no samples")
    k_levels = [int(k) for k in k_levels]
    if not k_levels:
        raise ConfigurationError("need at least one sparsity level")
    if any(a >= b for a, b in zip(k_levels, k_levels[1:])):
        raise ConfigurationError(f"k levels must be strictly increasing: {k_levels}")
    samples = sorted(dump.samples, key=lambda s: s.sample_id)
    n_max = max(tiles.padded_len(s.seq_len) for s in samples)
    cal = Calibrator(k_levels, tiles, dump.num_layers, dump.num_heads, n_max, dump.head_dim, device=device)
    for s in samples:
        for layer in range(dump.num_layers):
            cal.add_layer(s.sample_id, layer, s.q[layer], s.k[layer], seq_len=s.seq_len)
    return cal.finish()


def collect_block_maxima(sample: CalibrationSample, tiles: TileConfig, device=None) -> BlockMaximaProfile:
    """Sorted off-frontier tile maxima per (layer, head, position) (calibration.py:93-123)."""
    require_kernel_tiles(tiles)
    n_pad = tiles.padded_len(sample.seq_len)
    n_kern = kernel_len(sample.seq_len, tiles)
    L, H, _, d = sample.q.shape
    num_p = n_pad // tiles.b_m
    cal = Calibrator([0], tiles, L, H, n_pad, d, device=device)
    maxima = {}
    for layer in range(L):
        bm = torch.full((H, n_kern // tiles.b_m, n_kern // tiles.b_n), float("nan"), dtype=torch.float32,
                        device=cal.device)
        cal.add_layer(sample.sample_id, layer, sample.q[layer], sample.k[layer], seq_len=sample.seq_len,
                      block_maxima=bm)
        bm_sorted = torch.sort(torch.nan_to_num(bm, nan=-float("inf")), dim=2, descending=True).values.cpu().numpy()
        for h in range(H):
            for p in range(num_p):
                a = off_frontier_count(p, tiles)
                maxima[(layer, h, p)] = np.ascontiguousarray(bm_sorted[h, p, :a])
    if bool(cal.nonfinite.item()):
        raise InvalidInputError(f"sample {sample.sample_id}: non-finite activations")
    return BlockMaximaProfile(num_layers=L, num_heads=H, num_positions=num_p, maxima=maxima)
