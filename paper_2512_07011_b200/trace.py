"""Per-tile keep/skip record of a gated run (reference engine.py:22-25, 71-96).

Codes: UNREACHABLE=0, SKIPPED=1, FRONTIER=2, KEPT=3, one int8 per
(query block, key block) of the padded grid.  The kernel writes the same
codes (``decisions`` output of ``bsfa_fwd``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import BlockMask
from .tiling import TileConfig

UNREACHABLE = 0
SKIPPED = 1
FRONTIER = 2
KEPT = 3


@dataclass
class GateTrace:
    decisions: np.ndarray  # (m_q, m_kv) int8
    tiles: TileConfig
    causal: bool
    layer: int = 0
    head: int = 0

    def to_mask(self) -> BlockMask:
        return BlockMask(self.decisions >= FRONTIER)

    def kept_blocks(self) -> int:
        return int(np.count_nonzero(self.decisions >= FRONTIER))

    def reachable_blocks(self) -> int:
        return int(np.count_nonzero(self.decisions != UNREACHABLE))

    def retained_off_frontier(self) -> np.ndarray:
        return np.count_nonzero(self.decisions == KEPT, axis=1)

    def density(self) -> float:
        return self.kept_blocks() / self.reachable_blocks()
