"""Multi-GPU BSFA: one process per GPU, heads sharded by kv-head group.

The forward is embarrassingly parallel over (batch, kv head): every q head
reads only its own kv head, and thresholds are per (layer, head).  Rank r of
W owns kv heads [r*Hkv/W, (r+1)*Hkv/W) and the q heads of those groups
(a contiguous range, since q head h reads kv head h // (Hq/Hkv)), runs the
ordinary kernel on them with ``head_offset`` selecting its threshold rows,
and never talks to the other ranks during compute.  When the caller needs the
full [B, Hq, N, d] tensor on every rank there are two ways to assemble it:

* ``gather="nccl"``: an all-gather of O after the kernel (NCCL over NVLink);
* ``gather="peer"``: a :class:`PeerGatherBuffer` in symmetric memory -- the
  kernel epilogue stores each rank's O rows into its own slot of every
  rank's buffer over NVLink (``bsfa_fwd_args.o_peers``), so the exchange
  overlaps the attention tile by tile and only a barrier follows.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .errors import ConfigurationError


@dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    q_lo: int
    q_hi: int
    kv_lo: int
    kv_hi: int

    @property
    def num_q(self) -> int:
        return self.q_hi - self.q_lo

    @property
    def num_kv(self) -> int:
        return self.kv_hi - self.kv_lo


def shard_heads(heads_q: int, heads_kv: int, world: int, rank: int) -> HeadShard:
    """Contiguous kv-group partition; requires Hkv divisible by the world size."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigurationError(f"bad rank {rank} of {world}")
    if heads_q % heads_kv:
        raise ConfigurationError(f"q heads {heads_q} not a multiple of kv heads {heads_kv}")
    if heads_kv % world:
        raise ConfigurationError(
            f"{heads_kv} kv heads cannot be split evenly over {world} ranks; shard the batch instead")
    g = heads_q // heads_kv
    per = heads_kv // world
    kv_lo = rank * per
    return HeadShard(rank, world, kv_lo * g, (kv_lo + per) * g, kv_lo, kv_lo + per)


def gather_heads(o_local: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """All-gather per-rank [B, Hq/W, N, d] head shards into [B, Hq, N, d]."""
    if world == 1:
        return o_local
    b, hl, n, d = o_local.shape
    src = o_local.contiguous()
    buf = torch.empty((world, b, hl, n, d), dtype=o_local.dtype, device=o_local.device)
    backend = dist.get_backend(group)
    if backend == "nccl":
        dist.all_gather_into_tensor(buf.view(world * b, hl, n, d), src.view(b, hl, n, d), group=group)
    else:
        dist.all_gather(list(buf.unbind(0)), src, group=group)
    return gathered_view(buf)  # head-major for B = 1: rank shards are already contiguous


def peer_slot_pointers(buffer_ptrs, rank: int, slot_bytes: int) -> list[int]:
    """Addresses of rank ``rank``'s slot in every OTHER rank's gathered-O buffer.

    ``buffer_ptrs[p]`` is rank p's buffer base as mapped into this process
    (symmetric memory); the buffer is rank-major [W, B, Hq/W, N, d].
    """
    return [int(base) + rank * slot_bytes for p, base in enumerate(buffer_ptrs) if p != rank]


def gathered_view(buf: torch.Tensor) -> torch.Tensor:
    """Rank-major [W, B, Hq/W, N, d] -> [B, Hq, N, d] (a view for B = 1)."""
    world, b, hl, n, d = buf.shape
    if b == 1:
        return buf.view(1, world * hl, n, d)
    return buf.permute(1, 0, 2, 3, 4).reshape(b, world * hl, n, d)


class PeerGatherBuffer:
    """Gathered O, rank-major [W, B, Hq/W, N, d], filled by the kernel epilogues of all ranks.

    ``out`` is this rank's slot (pass it as ``attention(out=...)``) and
    ``peers`` the addresses of this rank's slot in the other ranks' buffers
    (``attention(o_peers=...)``).  After every rank's launch, :meth:`barrier`
    orders the remote stores before anyone reads :meth:`gathered`.
    Build it with :meth:`symmetric` (torch symmetric memory over NVLink);
    the constructor takes any mapping of the W buffers (tests use shared CPU
    memory and gloo).
    """

    def __init__(self, buf: torch.Tensor, buffer_ptrs, rank: int, barrier):
        world = buf.shape[0]
        if len(buffer_ptrs) != world or not 0 <= rank < world:
            raise ConfigurationError(f"{len(buffer_ptrs)} buffers for rank {rank} of {world}")
        if world - 1 > 7:
            raise ConfigurationError("peer stores reach at most 7 other GPUs")
        self.buf, self.rank, self.world = buf, rank, world
        self.out = buf[rank]
        self.peers = peer_slot_pointers(buffer_ptrs, rank, self.out.numel() * self.out.element_size())
        self._barrier = barrier

    @classmethod
    def symmetric(cls, batch: int, heads_q: int, seq_len: int, head_dim: int, *, rank: int, world: int,
                  group=None, device=None) -> "PeerGatherBuffer":
        from torch.distributed import _symmetric_memory as symm_mem

        if heads_q % world:
            raise ConfigurationError(f"{heads_q} q heads cannot be split over {world} ranks")
        device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        buf = symm_mem.empty((world, batch, heads_q // world, seq_len, head_dim), dtype=torch.bfloat16,
                             device=device)
        grp = group if group is not None else dist.group.WORLD
        handle = symm_mem.rendezvous(buf, grp.group_name)
        self = cls(buf, [int(x) for x in handle.buffer_ptrs], rank, lambda: handle.barrier())
        self.handle = handle
        return self

    def barrier(self) -> None:
        self._barrier()

    def gathered(self) -> torch.Tensor:
        return gathered_view(self.buf)


def sharded_attention(q, k, v, *, rank: int, world: int, thresholds=None, layer: int = 0,
                      k_level=None, gather=False, group=None, compute=None, peer_buffer=None, **kw):
    """Run this rank's heads of a full [B, Hq, N, d] problem.

    Without ``heads_q``/``heads_kv`` keywords, ``q``/``k``/``v`` are the FULL
    tensors and this rank's heads are sliced out here.  To pass only the local
    shard, give the full head counts: ``heads_q=Hq, heads_kv=Hkv`` -- then
    ``q.shape[1]`` must be Hq (sliced here) or Hq/W (used as is); anything else
    raises.  ``gather``: False, True/"nccl" (all-gather after the kernel) or
    "peer" (epilogue stores into ``peer_buffer``, a :class:`PeerGatherBuffer`;
    the returned gathered view aliases that buffer and is valid until the next
    call that uses it).  ``compute`` defaults to :func:`attention`; tests
    substitute a CPU checker to exercise the partition/gather logic without a GPU.
    """
    from .attention import attention

    compute = compute or attention
    full_q = kw.pop("heads_q", None)
    full_kv = kw.pop("heads_kv", None)
    if (full_q is None) != (full_kv is None):
        raise ConfigurationError("give both heads_q and heads_kv (the full head counts) or neither")
    hq = full_q if full_q is not None else q.shape[1]
    hkv = full_kv if full_kv is not None else k.shape[1]
    sh = shard_heads(hq, hkv, world, rank)
    if q.shape[1] == hq and k.shape[1] == hkv:
        if world > 1:
            q = q[:, sh.q_lo:sh.q_hi]
            k = k[:, sh.kv_lo:sh.kv_hi]
            v = v[:, sh.kv_lo:sh.kv_hi]
    elif q.shape[1] != sh.num_q or k.shape[1] != sh.num_kv:
        raise ConfigurationError(
            f"q/k carry {q.shape[1]}/{k.shape[1]} heads: neither the full problem ({hq}/{hkv}) "
            f"nor rank {rank}'s shard ({sh.num_q}/{sh.num_kv})")
    if gather == "peer":
        if peer_buffer is None:
            raise ConfigurationError('gather="peer" needs a PeerGatherBuffer')
        # write-after-read: a faster rank's epilogue must not overwrite slots a
        # peer is still reading from the previous call's gathered view
        peer_buffer.barrier()
        res = compute(q, k, v, thresholds=thresholds, layer=layer, k_level=k_level, head_offset=sh.q_lo,
                      out=peer_buffer.out, o_peers=peer_buffer.peers, **kw)
        peer_buffer.barrier()
        return res, peer_buffer.gathered()
    res = compute(q, k, v, thresholds=thresholds, layer=layer, k_level=k_level, head_offset=sh.q_lo, **kw)
    if gather:
        return res, gather_heads(res.o, world, group)
    return res, None


def sharded_calibrate(dump, k_levels, tiles, *, rank: int, world: int, group=None, calibrate_fn=None):
    """Threshold calibration sharded like the forward: rank r
    calibrates the q heads of its kv-head groups over every layer and sample,
    then the per-rank [S, L, H/W, P] slices are all-gathered into the full
    ThresholdTensor -- identical on every rank to a single-process calibrate().

    ``calibrate_fn(dump, k_levels, tiles)`` defaults to the GPU
    :func:`~paper_2512_07011_b200.calibration.calibrate`; tests substitute a
    CPU checker to exercise the partition and gather on gloo.
    """
    import numpy as np

    from .calibration import CalibrationDiagnostics, CalibrationDump, CalibrationSample, calibrate
    from .thresholds import ThresholdTensor

    calibrate_fn = calibrate_fn or calibrate
    if not dump.samples:
        raise ConfigurationError("calibration dump has no samples")
    hq, hkv = dump.samples[0].q.shape[1], dump.samples[0].k.shape[1]
    sh = shard_heads(hq, hkv, world, rank)
    local = CalibrationDump(dump.num_layers, sh.num_q, dump.head_dim, [
        CalibrationSample(s.sample_id, s.q[:, sh.q_lo:sh.q_hi], s.k[:, sh.kv_lo:sh.kv_hi]) for s in dump.samples])
    part = calibrate_fn(local, k_levels, tiles)
    if world == 1:
        return part
    vals = torch.from_numpy(np.ascontiguousarray(part.values))
    dev = None
    if dist.get_backend(group) == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
        vals = vals.to(dev)
    out = [torch.empty_like(vals) for _ in range(world)]
    dist.all_gather(out, vals, group=group)
    values = torch.cat(out, dim=2).cpu().numpy()  # ranks own consecutive head ranges
    ties = {}
    if getattr(part, "diagnostics", None) is not None:
        local_ties = torch.tensor([part.diagnostics.tie_counts[k] for k in part.k_levels], dtype=torch.int64,
                                  device=dev)
        dist.all_reduce(local_ties, group=group)
        ties = {k: int(v) for k, v in zip(part.k_levels, local_ties.cpu().tolist())}
        stats = {}
        for si, k in enumerate(part.k_levels):
            fv = values[si][np.isfinite(values[si])]
            stats[k] = (float(fv.min()), float(fv.mean()), float(fv.max())) if fv.size else (None, None, None)
        diag = CalibrationDiagnostics(num_samples=part.diagnostics.num_samples, tie_counts=ties,
                                      threshold_stats=stats)
    else:
        diag = None
    return ThresholdTensor(values=values, k_levels=part.k_levels, n_max=part.n_max, b_m=part.b_m, b_n=part.b_n,
                           diagnostics=diag)
