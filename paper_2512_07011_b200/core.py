"""Single-head input/output records of the drop-in API.

Same fields and validation as reference pkg/src/bsfa/core.py:20-101
(HeadInput / AttentionOutput / BlockMask).  The fp64 oracle functions of that
module are *not* part of the product; they live in ``oracle/`` as test
infrastructure.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InvalidInputError
from .tiling import TileConfig, frontier_blocks


@dataclass
class HeadInput:
    """One head's Q/K/V (n, d), stored as contiguous float32 (core.py:20-56)."""

    q: np.ndarray
    k: np.ndarray
    v: np.ndarray
    causal: bool = True

    def __post_init__(self):
        arrs = []
        for name in ("q", "k", "v"):
            m = np.ascontiguousarray(getattr(self, name), dtype=np.float32)
            if m.ndim != 2:
                raise InvalidInputError(f"{name} must be 2-D (n, d), got shape {m.shape}")
            arrs.append(m)
            setattr(self, name, m)
        if not (arrs[0].shape == arrs[1].shape == arrs[2].shape):
            raise InvalidInputError(
                f"q/k/v shapes differ: {arrs[0].shape}, {arrs[1].shape}, {arrs[2].shape}")
        for name, m in zip("qkv", arrs):
            if not np.isfinite(m).all():
                raise InvalidInputError(f"{name} contains non-finite entries")
        n, d = self.q.shape
        if n < 1 or d < 1:
            raise InvalidInputError(f"need n >= 1 and d >= 1, got n={n}, d={d}")

    @property
    def seq_len(self) -> int:
        return self.q.shape[0]

    @property
    def head_dim(self) -> int:
        return self.q.shape[1]


@dataclass
class AttentionOutput:
    o: np.ndarray          # (n, d)
    logsumexp: np.ndarray  # (n,)  m + ln(l), scaled-score units


@dataclass
class BlockMask:
    """Boolean (query block x key block) grid of processed blocks."""

    allowed: np.ndarray

    def __post_init__(self):
        self.allowed = np.asarray(self.allowed, dtype=bool)
        if self.allowed.ndim != 2:
            raise InvalidInputError(f"block mask must be 2-D, got {self.allowed.shape}")

    @classmethod
    def frontier_only(cls, n: int, tiles: TileConfig) -> "BlockMask":
        grid = np.zeros((tiles.num_q_blocks(n), tiles.num_kv_blocks(n)), dtype=bool)
        for i in range(grid.shape[0]):
            fr = frontier_blocks(i, tiles, n)
            grid[i, fr.start:fr.stop] = True
        return cls(grid)
