"""Multi-GPU BSFA: one process per GPU, heads sharded by kv-head group.

The forward is embarrassingly parallel over (batch, kv head): every q head
reads only its own kv head, and thresholds are per (layer, head).  Rank r of
W owns kv heads [r*Hkv/W, (r+1)*Hkv/W) and the q heads of those groups
(a contiguous range, since q head h reads kv head h // (Hq/Hkv)), runs the
ordinary kernel on them with ``head_offset`` selecting its threshold rows,
and never talks to the other ranks during compute.  The only collective is
an optional all-gather of O (NCCL over NVLink) when the caller needs the full
[B, Hq, N, d] tensor on every rank.
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
    if b == 1:
        return buf.view(1, world * hl, n, d)  # head-major: rank shards are already contiguous
    return buf.permute(1, 0, 2, 3, 4).reshape(b, world * hl, n, d)


def sharded_attention(q, k, v, *, rank: int, world: int, thresholds=None, layer: int = 0,
                      k_level=None, gather: bool = False, group=None, compute=None, **kw):
    """Run this rank's heads of a full [B, Hq, N, d] problem.

    ``q``/``k``/``v`` may be the full tensors (sliced here) or already the
    local shard (``q.shape[1] == Hq/W``).  ``compute`` defaults to
    :func:`attention`; tests substitute a CPU checker to exercise the
    partition/gather logic without a GPU.
    """
    from .attention import attention

    compute = compute or attention
    full_q = kw.pop("heads_q", None)
    full_kv = kw.pop("heads_kv", None)
    hq = full_q if full_q is not None else q.shape[1]
    hkv = full_kv if full_kv is not None else k.shape[1]
    sh = shard_heads(hq, hkv, world, rank)
    if q.shape[1] == hq and world > 1:
        q = q[:, sh.q_lo:sh.q_hi]
        k = k[:, sh.kv_lo:sh.kv_hi]
        v = v[:, sh.kv_lo:sh.kv_hi]
    res = compute(q, k, v, thresholds=thresholds, layer=layer, k_level=k_level, head_offset=sh.q_lo, **kw)
    if gather:
        return res, gather_heads(res.o, world, group)
    return res, None
