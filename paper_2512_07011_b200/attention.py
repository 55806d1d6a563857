"""BSFA forward on sm_100a: the batched entry point and the reference drop-in.

* :func:`attention` -- batched/GQA entry point on CUDA tensors
  (q [B, Hq, N, d], k/v [B, Hkv, N, d], bf16).  One launch of the
  ``bsfa_fwd`` C-ABI kernel; returns O (bf16), LSE (fp32) and optionally the
  per-tile decision trace and kept/skipped/V-load counters.
* :func:`flash_forward` -- the reference signature
  ``flash_forward(inp, tiles, gate, ctx=None, threads=1, inject_fault=False)
  -> (AttentionOutput, GateTrace)`` (reference engine.py:117-193), numpy in,
  numpy out, one head, executed by the same kernel.

Semantics kept from the reference engine:
  - sequences are padded to lcm(b_m, b_n) by repeating the last row
    (engine.py:99-114), then to the kernels' 128-row tiles
    (``tiling.kernel_len``), and outputs / the trace are sliced back to the
    valid length / the reference grid;
  - head_dim d <= 256 is zero-padded to 64, 128 or 256 columns with the
    scale of the original d;
  - frontier tiles are always processed with the element-wise causal mask,
    off-frontier tiles go through the gate (engine.py:157-175);
  - keep iff max(QK^T * scale over the tile) > T, strictly (gates.py:77-78);
  - scale = float32(1/sqrt(d)) (engine.py:144); LSE = m + ln(l) in scaled
    natural-log units (engine.py:182);
  - a row with a non-finite accumulator or l <= 0 raises NumericError
    (engine.py:178-179) when ``check_numerics`` is on (the default, as in
    the reference; always on in the drop-in, which synchronises anyway).
Numerics differ by design: inputs are rounded to bf16, P is bf16 on the
tensor cores, O is emitted in bf16 (tolerance documented in DESIGN.md).
"""

from __future__ import annotations

import ctypes
import weakref
import zlib
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import AttentionOutput, HeadInput
from .errors import ConfigurationError, InvalidInputError, NumericError
from .gates import GateContext, ThresholdGate, gate_params, kernel_gate_mode
from .thresholds import ThresholdTensor
from .tiling import TileConfig, kernel_len, require_kernel_tiles
from .trace import GateTrace


@dataclass
class AttentionResult:
    o: torch.Tensor                  # [B, Hq, N, d] bf16
    lse: torch.Tensor                # [B, Hq, N] fp32
    decisions: torch.Tensor | None   # [B, Hq, M_q, M_kv] int8 (padded grid) or None
    counters: torch.Tensor           # int64 [4]: reachable, kept, V tiles loaded, V tiles loadable
    status: torch.Tensor             # int32 [1]; non-zero = numeric failure


def _scale_for(d: int) -> float:
    return float(np.float32(1.0) / np.sqrt(np.float32(d)))


def reference_scale(d: int) -> float:
    """float32(1/sqrt(d)) exactly as reference engine.py:144 computes it."""
    return float(np.float32(1.0 / np.sqrt(d)))


def _pad_rows(x: torch.Tensor, target: int) -> torch.Tensor:
    n = x.shape[2]
    if n == target:
        return x
    tail = x[:, :, n - 1:n, :].expand(-1, -1, target - n, -1)
    return torch.cat([x, tail], dim=2)


def _pad_dim(x: torch.Tensor, dp: int) -> torch.Tensor:
    d = x.shape[3]
    if d == dp:
        return x
    return torch.nn.functional.pad(x, (0, dp - d))


def _check_inputs(q, k, v):
    for name, t in (("q", q), ("k", k), ("v", v)):
        if not isinstance(t, torch.Tensor):
            raise InvalidInputError(f"{name} must be a torch tensor")
        if t.dim() != 4:
            raise InvalidInputError(f"{name} must be 4-D [B, H, N, d], got {tuple(t.shape)}")
        if not t.is_cuda:
            raise InvalidInputError(f"{name} must be on a CUDA device (no CPU fallback)")
    if k.shape != v.shape:
        raise InvalidInputError(f"k/v shapes differ: {tuple(k.shape)} vs {tuple(v.shape)}")
    b, hq, n, d = q.shape
    if k.shape[0] != b or k.shape[2] != n or k.shape[3] != d:
        raise InvalidInputError(f"q {tuple(q.shape)} and k {tuple(k.shape)} disagree")
    hkv = k.shape[1]
    if hkv < 1 or hq % hkv:
        raise InvalidInputError(f"query heads {hq} must be a multiple of kv heads {hkv}")
    if n < 1 or d < 1:
        raise InvalidInputError("empty sequence or head dimension")
    if d > 256:
        raise InvalidInputError(f"head_dim {d} > 256 is not supported by the kernels")


def head_dim_pad(d: int) -> int:
    """The kernels' head_dim for a head of width d: 64, 128 or 256 (zero-padded columns)."""
    return 64 if d <= 64 else (128 if d <= 128 else 256)


def _as_kernel_operand(x: torch.Tensor, n_pad: int, d_pad: int) -> torch.Tensor:
    x = x.to(torch.bfloat16)
    x = _pad_dim(_pad_rows(x, n_pad), d_pad)
    if x.stride(3) != 1 or (x.stride(2) * 2) % 16 or x.data_ptr() % 16:
        x = x.contiguous()
    return x


_THR_CACHE: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _device_thresholds(thresholds: ThresholdTensor, k_level, layer: int, head_offset: int, hq: int,
                       device) -> torch.Tensor:
    """fp32 [Hq, P] threshold rows on ``device``, uploaded once per (tensor, level, layer, heads, device).

    The cache is keyed on the ThresholdTensor object and re-validated by a
    CRC of the slice, so repeated calls (every layer of every forward) do not
    pay a synchronous host-to-device copy, and an in-place edit of ``values``
    is still picked up.
    """
    sl = np.ascontiguousarray(thresholds.layer_slice(k_level, layer)[head_offset:head_offset + hq])
    crc = zlib.crc32(sl.view(np.uint8))
    per = _THR_CACHE.setdefault(thresholds, {})
    key = (k_level, layer, head_offset, hq, str(device))
    hit = per.get(key)
    if hit is not None and hit[0] == crc:
        return hit[1]
    t = torch.from_numpy(sl).to(device)
    per[key] = (crc, t)
    return t


def attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, causal: bool = True,
              gate=None, thresholds: ThresholdTensor | None = None, layer: int = 0,
              k_level: int | None = None, head_offset: int = 0,
              tiles: TileConfig = TileConfig(), return_trace: bool = False,
              inject_fault: bool = False, check_numerics: bool = True,
              scale: float | None = None, out: torch.Tensor | None = None,
              o_peers=()) -> AttentionResult:
    """Block-sparse (or dense) causal/non-causal GQA attention forward.

    Gate selection: ``thresholds`` + ``k_level`` (+ ``layer``) runs the
    ThresholdGate with per-(head, query block) thresholds
    ``values[level, layer, head_offset + h, min(i, P-1)]``; otherwise ``gate``
    may be a DenseGate / FrontierOnlyGate / ThresholdGate object; with
    neither the run is dense.

    ``check_numerics`` (default on, like the reference engine.py:178-179)
    reads the kernel's status word after the launch -- one device sync -- and
    raises :class:`NumericError` if any row had a non-finite accumulator or a
    zero normaliser.  Pass ``False`` in stream-ordered serving loops (or use
    :class:`BsfaPlan`) and inspect ``result.status`` when convenient.

    ``out`` (bf16 [B, Hq, n_kern, d_pad], n_kern = ``tiling.kernel_len(n, tiles)``, unit head_dim stride, 16-byte aligned
    rows) receives O instead of a fresh tensor; ``o_peers`` are device
    addresses of further copies with ``out``'s strides (peer GPUs' slots of a
    gathered-O buffer mapped over NVLink) that the kernel epilogue writes
    alongside ``out`` -- the head-sharded all-gather without a collective.
    """
    _check_inputs(q, k, v)
    require_kernel_tiles(tiles)
    hq = q.shape[1]

    thr_dev = None
    if thresholds is None and isinstance(gate, ThresholdGate):
        thresholds = gate.tensor
    if thresholds is not None:
        ThresholdGate(thresholds).validate(tiles, GateContext(layer=layer, k_level=k_level))
        thresholds.check_site(layer, head_offset)
        if head_offset + hq > thresholds.num_heads:
            raise ConfigurationError(
                f"heads [{head_offset}, {head_offset + hq}) outside calibrated {thresholds.num_heads}")
        thr_dev = _device_thresholds(thresholds, k_level, layer, head_offset, hq, q.device)
        mode = _lib.GATE_THRESHOLD
    elif gate is not None:
        mode = kernel_gate_mode(gate)
        if mode == _lib.GATE_THRESHOLD:  # pragma: no cover - handled above
            raise ConfigurationError("threshold gate without thresholds")
    else:
        mode = _lib.GATE_DENSE
    window, lam = gate_params(gate) if thr_dev is None else (0, 0.0)
    res = _forward(q, k, v, thr_dev, mode, window, lam, causal=causal, tiles=tiles, return_trace=return_trace,
                   inject_fault=inject_fault, scale=scale, out=out, o_peers=o_peers)
    if check_numerics and int(res.status.item()) != 0:
        raise NumericError("non-finite accumulator or zero normaliser in at least one query row")
    return res


def _forward(q, k, v, thr_dev, mode: int, window: int, lam: float, *, causal: bool, tiles: TileConfig,
             return_trace: bool, inject_fault: bool = False, scale: float | None = None,
             out: torch.Tensor | None = None, o_peers=()) -> AttentionResult:
    """One ``bsfa_fwd`` launch on validated inputs; ``thr_dev`` fp32 [Hq, P] on q's device or None."""
    bsz, hq, n, d = q.shape
    hkv = k.shape[1]
    thr_positions = int(thr_dev.shape[1]) if thr_dev is not None else 0
    n_pad = tiles.padded_len(n)  # the reference grid
    n_kern = kernel_len(n, tiles)  # n_pad rounded up to the kernels' 128 rows
    d_pad = head_dim_pad(d)
    sc = reference_scale(d) if scale is None else float(np.float32(scale))

    dev = q.device
    with torch.cuda.device(dev):
        qk = _as_kernel_operand(q, n_kern, d_pad)
        kk = _as_kernel_operand(k, n_kern, d_pad)
        vk = _as_kernel_operand(v, n_kern, d_pad)
        o_peers = [int(x) for x in o_peers]
        if out is not None:
            if (tuple(out.shape) != (bsz, hq, n_kern, d_pad) or out.dtype != torch.bfloat16 or out.device != dev
                    or out.stride(3) != 1 or (out.stride(2) * 2) % 16 or out.data_ptr() % 16):
                raise InvalidInputError(
                    f"out must be bf16 {(bsz, hq, n_kern, d_pad)} on {dev} with unit head_dim stride and "
                    "16-byte aligned rows")
            o = out
        elif o_peers:
            raise InvalidInputError("o_peers mirror out's layout: pass out as well")
        else:
            o = torch.empty((bsz, hq, n_kern, d_pad), dtype=torch.bfloat16, device=dev)
        if len(o_peers) > _lib.MAX_O_PEERS:
            raise ConfigurationError(f"at most {_lib.MAX_O_PEERS} peer copies of O")
        lse = torch.empty((bsz, hq, n_kern), dtype=torch.float32, device=dev)
        m_q, m_kv = n_kern // tiles.b_m, n_kern // tiles.b_n
        dec = torch.zeros((bsz, hq, m_q, m_kv), dtype=torch.int8, device=dev) if return_trace else None
        counters = torch.zeros(4, dtype=torch.int64, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)

        a = _lib.FwdArgs()
        a.q, a.k, a.v = qk.data_ptr(), kk.data_ptr(), vk.data_ptr()
        a.q_stride_b, a.q_stride_h, a.q_stride_n = qk.stride(0), qk.stride(1), qk.stride(2)
        a.k_stride_b, a.k_stride_h, a.k_stride_n = kk.stride(0), kk.stride(1), kk.stride(2)
        a.v_stride_b, a.v_stride_h, a.v_stride_n = vk.stride(0), vk.stride(1), vk.stride(2)
        a.o = o.data_ptr()
        a.o_stride_b, a.o_stride_h, a.o_stride_n = o.stride(0), o.stride(1), o.stride(2)
        a.lse = lse.data_ptr()
        a.decisions = dec.data_ptr() if dec is not None else None
        a.counters = counters.data_ptr()
        a.status = status.data_ptr()
        a.thresholds = thr_dev.data_ptr() if thr_dev is not None else None
        a.thr_positions = thr_positions
        a.gate_mode = mode
        a.batch, a.heads_q, a.heads_kv = bsz, hq, hkv
        a.seq_len, a.valid_len, a.head_dim = n_kern, n, d_pad
        a.b_m, a.b_n = tiles.b_m, tiles.b_n
        a.causal = 1 if causal else 0
        a.scale = sc
        a.inject_fault = 1 if inject_fault else 0
        a.gate_window, a.gate_lambda = window, lam
        a.num_o_peers = len(o_peers)
        for i, ptr in enumerate(o_peers):
            a.o_peers[i] = ptr
        stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(_lib.load_library().bsfa_fwd(ctypes.byref(a), ctypes.c_void_p(stream)), "bsfa_fwd")

    if n_kern != n or d_pad != d:
        o = o[:, :, :n, :d]
        lse = lse[:, :, :n]
    if dec is not None and n_kern != n_pad:  # the reference grid (b_m = 64, odd block count)
        dec = dec[:, :, :n_pad // tiles.b_m, :n_pad // tiles.b_n]
    return AttentionResult(o=o, lse=lse, decisions=dec, counters=counters, status=status)


def flash_forward(inp, tiles: TileConfig, gate, ctx: GateContext | None = None, threads: int = 1,
                  inject_fault: bool = False, device=None) -> tuple[AttentionOutput, GateTrace]:
    """Reference-signature single-head forward (engine.py:117-124) on the GPU.

    ``threads`` is accepted for signature compatibility and ignored (the
    kernel parallelises over query blocks by construction, bitwise
    deterministically).  ``inp`` is a HeadInput (this package's or any object
    with q/k/v/causal); values are rounded to bf16 on upload.
    """
    if ctx is None:
        ctx = GateContext()
    gate.validate(tiles, ctx)
    mode = kernel_gate_mode(gate)
    require_kernel_tiles(tiles)
    if not isinstance(inp, HeadInput):
        inp = HeadInput(inp.q, inp.k, inp.v, causal=bool(inp.causal))
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())

    def up(m):
        return torch.from_numpy(m).to(dev).to(torch.bfloat16)[None, None]

    kw = {}
    if mode == _lib.GATE_THRESHOLD:
        kw = dict(thresholds=gate.tensor, layer=ctx.layer, k_level=ctx.k_level, head_offset=ctx.head)
    else:
        kw = dict(gate=gate)
    res = attention(up(inp.q), up(inp.k), up(inp.v), causal=inp.causal, tiles=tiles,
                    return_trace=True, inject_fault=inject_fault, **kw)
    if int(res.status.item()) != 0:
        raise NumericError("non-finite accumulator in at least one query block")
    o = res.o[0, 0].float().cpu().numpy()
    lse = res.lse[0, 0].cpu().numpy()
    trace = GateTrace(decisions=res.decisions[0, 0].cpu().numpy(), tiles=tiles,
                      causal=inp.causal, layer=ctx.layer, head=ctx.head)
    return AttentionOutput(o=o, logsumexp=lse), trace


class BsfaPlan:
    """Pre-built launch for a fixed shape: device buffers and C-ABI arguments made once.

    ``run(q, k, v)`` is then one ``bsfa_fwd`` launch (plus a counter reset)
    on the current stream -- the form used by serving loops, CUDA graphs and
    the benchmark.  q/k/v must already have the padded shape the plan was
    built for ([B, Hq, n_pad, d] bf16, d in {64, 128}, row stride 16-B aligned).
    """

    def __init__(self, batch: int, heads_q: int, heads_kv: int, seq_len: int, head_dim: int, *,
                 causal: bool = True, tiles: TileConfig = TileConfig(), thresholds: ThresholdTensor | None = None,
                 layer: int = 0, k_level: int | None = None, head_offset: int = 0, gate=None,
                 return_trace: bool = False, device=None, out: torch.Tensor | None = None, o_peers=(),
                 scale: float | None = None):
        """``out`` / ``o_peers``: as in :func:`attention` (caller-owned O, extra peer copies).

        ``scale`` defaults to float32(1/sqrt(head_dim)) (engine.py:144).  Heads
        narrower than 64/128 that the caller zero-pads to a plan width must pass
        the ORIGINAL head's scale (``reference_scale(d)``), or the softmax and
        the threshold comparisons use the padded width's.
        """
        require_kernel_tiles(tiles)
        if head_dim not in (64, 128, 256):
            raise InvalidInputError("plans take head_dim 64, 128 or 256 (pad smaller heads and pass their scale)")
        if heads_q % heads_kv:
            raise InvalidInputError(f"query heads {heads_q} must be a multiple of kv heads {heads_kv}")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.tiles = tiles
        self.n = seq_len
        self.n_pad = kernel_len(seq_len, tiles)  # the reference padding rounded up to 128 rows
        self.shape_q = (batch, heads_q, self.n_pad, head_dim)
        self.shape_kv = (batch, heads_kv, self.n_pad, head_dim)
        dev = self.device
        self.thr = None
        if thresholds is None and isinstance(gate, ThresholdGate):
            thresholds = gate.tensor
        if thresholds is not None:
            ThresholdGate(thresholds).validate(tiles, GateContext(layer=layer, k_level=k_level))
            thresholds.check_site(layer, head_offset)
            if head_offset + heads_q > thresholds.num_heads:
                raise ConfigurationError("plan heads exceed the calibrated head range")
            sl = thresholds.layer_slice(k_level, layer)[head_offset:head_offset + heads_q]
            self.thr = torch.from_numpy(np.ascontiguousarray(sl)).to(dev)
            mode = _lib.GATE_THRESHOLD
        elif gate is not None:
            mode = kernel_gate_mode(gate)
        else:
            mode = _lib.GATE_DENSE
        o_peers = [int(x) for x in o_peers]
        if out is not None:
            if (tuple(out.shape) != self.shape_q or out.dtype != torch.bfloat16 or out.device != dev
                    or out.stride(3) != 1 or (out.stride(2) * 2) % 16 or out.data_ptr() % 16):
                raise InvalidInputError(f"out must be bf16 {self.shape_q} on {dev} with 16-byte aligned rows")
            self.o = out
        elif o_peers:
            raise InvalidInputError("o_peers mirror out's layout: pass out as well")
        else:
            self.o = torch.empty(self.shape_q, dtype=torch.bfloat16, device=dev)
        if len(o_peers) > _lib.MAX_O_PEERS:
            raise ConfigurationError(f"at most {_lib.MAX_O_PEERS} peer copies of O")
        self.lse = torch.empty((batch, heads_q, self.n_pad), dtype=torch.float32, device=dev)
        m_q, m_kv = self.n_pad // tiles.b_m, self.n_pad // tiles.b_n
        self.decisions = (torch.zeros((batch, heads_q, m_q, m_kv), dtype=torch.int8, device=dev)
                          if return_trace else None)
        self.counters = torch.zeros(4, dtype=torch.int64, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        a = _lib.FwdArgs()
        a.o = self.o.data_ptr()
        a.o_stride_b, a.o_stride_h, a.o_stride_n = self.o.stride(0), self.o.stride(1), self.o.stride(2)
        a.lse = self.lse.data_ptr()
        a.decisions = self.decisions.data_ptr() if self.decisions is not None else None
        a.counters = self.counters.data_ptr()
        a.status = self.status.data_ptr()
        a.thresholds = self.thr.data_ptr() if self.thr is not None else None
        a.thr_positions = self.thr.shape[1] if self.thr is not None else 0
        a.gate_mode = mode
        a.batch, a.heads_q, a.heads_kv = batch, heads_q, heads_kv
        a.seq_len, a.valid_len, a.head_dim = self.n_pad, seq_len, head_dim
        a.b_m, a.b_n = tiles.b_m, tiles.b_n
        a.causal = 1 if causal else 0
        a.scale = reference_scale(head_dim) if scale is None else float(np.float32(scale))
        a.inject_fault = 0
        a.gate_window, a.gate_lambda = gate_params(gate) if self.thr is None else (0, 0.0)
        a.num_o_peers = len(o_peers)
        for i, ptr in enumerate(o_peers):
            a.o_peers[i] = ptr
        self.args = a
        self.lib = _lib.load_library()

    def run(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, reset_counters: bool = True) -> torch.Tensor:
        if tuple(q.shape) != self.shape_q or tuple(k.shape) != self.shape_kv or tuple(v.shape) != self.shape_kv:
            raise InvalidInputError(f"plan built for q{self.shape_q} kv{self.shape_kv}")
        if q.dtype != torch.bfloat16 or k.dtype != torch.bfloat16 or v.dtype != torch.bfloat16:
            raise InvalidInputError("plan inputs must be bf16")
        a = self.args
        a.q, a.k, a.v = q.data_ptr(), k.data_ptr(), v.data_ptr()
        a.q_stride_b, a.q_stride_h, a.q_stride_n = q.stride(0), q.stride(1), q.stride(2)
        a.k_stride_b, a.k_stride_h, a.k_stride_n = k.stride(0), k.stride(1), k.stride(2)
        a.v_stride_b, a.v_stride_h, a.v_stride_n = v.stride(0), v.stride(1), v.stride(2)
        with torch.cuda.device(self.device):
            if reset_counters:
                self.counters.zero_()
            stream = torch.cuda.current_stream(self.device).cuda_stream
            _lib.check(self.lib.bsfa_fwd(ctypes.byref(a), ctypes.c_void_p(stream)), "bsfa_fwd")
        return self.o

    # ------------------------------------------------------------------ host-resident inputs
    def run_host(self, q_h: torch.Tensor, k_h: torch.Tensor, v_h: torch.Tensor, o_h: torch.Tensor,
                 chunks: int | None = None) -> torch.Tensor:
        """End-to-end forward from pinned host tensors into a pinned host output.

        The q heads are cut into ``chunks`` equal groups (each within one kv
        head or covering whole kv heads); streams pipeline the host->device
        copy of group c+1, the kernel on group c (two compute streams, so one
        launch's tail overlaps the next launch) and the device->host copy of
        group c-1, so PCIe transfers overlap the attention instead of
        bracketing it.  K/V of a kv head are copied with its first group.
        Inputs are bf16 [B, H, n_pad, d] pinned host tensors of the plan's
        shape.  Returns ``o_h``; the caller synchronises (or waits on
        ``self.done``).
        """
        if tuple(q_h.shape) != self.shape_q or tuple(k_h.shape) != self.shape_kv or tuple(v_h.shape) != self.shape_kv:
            raise InvalidInputError(f"plan built for q{self.shape_q} kv{self.shape_kv}")
        if tuple(o_h.shape) != self.shape_q:
            raise InvalidInputError("o_h must have the q shape")
        for t in (q_h, k_h, v_h, o_h):
            if t.is_cuda or t.dtype != torch.bfloat16 or not t.is_contiguous():
                raise InvalidInputError("run_host takes contiguous bf16 host tensors (pinned for async copies)")
        bsz, hq, n, d = self.shape_q
        hkv = self.shape_kv[1]
        grp = hq // hkv

        def valid(c):
            qp = hq // c
            return hq % c == 0 and (qp % grp == 0 or grp % qp == 0)

        if chunks is None:
            # two q heads per launch (a full CTA pair) when the group allows,
            # at most 16 launches (l32k e2e: 16 groups 9.4 ms, 8 groups 9.5, serial 18.3)
            qmin = 2 if grp % 2 == 0 else grp
            chunks = max(c for c in range(1, min(16, hq // qmin) + 1) if valid(c))
        if chunks < 1 or not valid(chunks):
            raise ConfigurationError(f"{hq} q heads ({hkv} kv heads) cannot be cut into {chunks} chunks")
        with torch.cuda.device(self.device):
            return self._run_host(q_h, k_h, v_h, o_h, chunks, grp)

    def _run_host(self, q_h, k_h, v_h, o_h, chunks, grp):
        bsz, hq, n, d = self.shape_q
        dev = self.device
        if getattr(self, "_host_bufs", None) is None:
            self._host_bufs = (torch.empty(self.shape_q, dtype=torch.bfloat16, device=dev),
                               torch.empty(self.shape_kv, dtype=torch.bfloat16, device=dev),
                               torch.empty(self.shape_kv, dtype=torch.bfloat16, device=dev))
            self._streams = tuple(torch.cuda.Stream(dev) for _ in range(4))
        qd, kd, vd = self._host_bufs
        s_in, s_out, c0, c1 = self._streams
        current = torch.cuda.current_stream(dev)
        q_per = hq // chunks
        self.counters.zero_()
        start = torch.cuda.Event()
        start.record(current)
        for st in self._streams:
            st.wait_event(start)
        base = self.args
        kv_copied = 0
        for c in range(chunks):
            h0 = c * q_per
            g0, g1 = h0 // grp, (h0 + q_per - 1) // grp + 1
            with torch.cuda.stream(s_in):
                qd[:, h0:h0 + q_per].copy_(q_h[:, h0:h0 + q_per], non_blocking=True)
                if g1 > kv_copied:
                    kd[:, kv_copied:g1].copy_(k_h[:, kv_copied:g1], non_blocking=True)
                    vd[:, kv_copied:g1].copy_(v_h[:, kv_copied:g1], non_blocking=True)
                    kv_copied = g1
                ready = torch.cuda.Event()
                ready.record(s_in)
            compute = c0 if c % 2 == 0 else c1
            compute.wait_event(ready)
            for bi in range(bsz):  # one launch per batch element: LSE / trace rows stay [b, h] addressed
                a = _lib.FwdArgs.from_buffer_copy(base)
                a.q = qd[bi, h0].data_ptr()
                a.k, a.v = kd[bi, g0].data_ptr(), vd[bi, g0].data_ptr()
                a.q_stride_b, a.q_stride_h, a.q_stride_n = qd.stride(0), qd.stride(1), qd.stride(2)
                a.k_stride_b, a.k_stride_h, a.k_stride_n = kd.stride(0), kd.stride(1), kd.stride(2)
                a.v_stride_b, a.v_stride_h, a.v_stride_n = vd.stride(0), vd.stride(1), vd.stride(2)
                a.o = self.o[bi, h0].data_ptr()
                a.lse = self.lse[bi, h0].data_ptr()
                a.batch, a.heads_q, a.heads_kv = 1, q_per, g1 - g0
                a.num_o_peers = 0  # the host path returns O to the host; no peer copies
                if self.thr is not None:
                    a.thresholds = self.thr[h0].data_ptr()
                if self.decisions is not None:
                    a.decisions = self.decisions[bi, h0].data_ptr()
                _lib.check(self.lib.bsfa_fwd(ctypes.byref(a), ctypes.c_void_p(compute.cuda_stream)), "bsfa_fwd")
            done = torch.cuda.Event()
            done.record(compute)
            s_out.wait_event(done)
            with torch.cuda.stream(s_out):
                o_h[:, h0:h0 + q_per].copy_(self.o[:, h0:h0 + q_per], non_blocking=True)
        # s_out follows every kernel (it waited on each); the caller's stream follows s_out
        self.done = torch.cuda.Event()
        self.done.record(s_out)
        current.wait_event(self.done)
        return o_h
