"""Synthetic Llama-shaped attention inputs generated on the GPU.

The reference generators (pkg/src/bsfa/workloads.py:58-77 gen_random,
:139-172 gen_structured, :185-216 gen_model_dump) draw N(0, 1) q/k/v per
(sample, layer, head) from numpy and, for "structured" heads, add a shared
bias of norm sqrt(6 * sqrt(d)) along a per-(layer, head) unit direction to
every query row and to the elevated key rows (a 64-key sink, a 128-key
trailing window and 2 heavy hitters), so those blocks dominate the
block-maxima profile.  The model dump alternates structured / random heads
over (layer * H + head).

This module restates that distribution on the device for full Llama scale
(32 layers x 32 q heads x 32K tokens would be 16 GiB per tensor per sample
as host fp32).  GQA-shaped: the structure is a property of the kv head g
(layer * Hkv + g even -> structured), its direction biases the q heads of
that group and the elevated rows of k_g.  Torch's generator replaces numpy's,
so values are distributed like the reference's, not bit-identical; parity
tests use the numpy oracle on the exact tensors produced here.
"""

from __future__ import annotations

import math

import torch

ELEVATION = 6.0  # reference workloads.py _ELEVATION


def _gen(seed: int, sample: int, layer: int, tag: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((((seed * 1_000_003 + sample) * 1_000_033 + layer) * 1_009 + tag) & 0x7FFF_FFFF_FFFF_FFFF)
    return g


def model_dump_layer(sample: int, layer: int, heads_q: int, heads_kv: int, n: int, d: int, *, seed: int = 0,
                     device=None, dtype=torch.bfloat16, sink: int = 64, window: int = 128, heavy: int = 2,
                     with_v: bool = True):
    """q [Hq, n, d], k/v [Hkv, n, d] of one (sample, layer) of a model-dump-style workload."""
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    group = heads_q // heads_kv
    q = torch.randn((heads_q, n, d), generator=_gen(seed, sample, layer, 0, device), device=device)
    k = torch.randn((heads_kv, n, d), generator=_gen(seed, sample, layer, 1, device), device=device)
    v = torch.randn((heads_kv, n, d), generator=_gen(seed, sample, layer, 2, device), device=device) \
        if with_v else None
    amp = math.sqrt(ELEVATION * math.sqrt(d))
    for gk in range(heads_kv):
        if (layer * heads_kv + gk) % 2:
            continue  # random head
        # direction and heavy hitters are properties of (layer, kv head), stable across samples
        aux = _gen(seed, 0, layer, 3 + 10 * gk, device)
        direction = torch.randn(d, generator=aux, device=device)
        direction = direction / direction.norm()
        elevated = torch.zeros(n, dtype=torch.bool, device=device)
        elevated[:sink] = True
        if window:
            elevated[n - window:] = True
        if heavy:
            elevated[torch.randperm(n, generator=aux, device=device)[:heavy]] = True
        bias = amp * direction
        q[gk * group:(gk + 1) * group] += bias
        k[gk, elevated] += bias
    out = (q.to(dtype), k.to(dtype))
    return out + (v.to(dtype),) if with_v else out
