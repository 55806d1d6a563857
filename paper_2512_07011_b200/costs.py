"""FLOP / byte / density accounting used for measurement.

Restates reference pkg/src/bsfa/costs.py:45-125 (tile counts, predicted
density under a top-k budget, executed matmul FLOPs, K/V traffic) and adds
the conversion from the kernel's own counters (BSFA_CNT_*) to the roofline
numerators reported by ``bench.py``:

    F_exec = 2 * b_m * b_n * d * (reachable + kept)    QK for every reachable
                                                       tile, PV for kept ones
    F_dense = 2 * b_m * b_n * d * 2 * reachable        the same kernel at T=-inf
"""

from __future__ import annotations

from .errors import InvalidInputError
from .tiling import TileConfig, frontier_count, off_frontier_count


def tile_counts(n: int, tiles: TileConfig, causal: bool = True) -> tuple[int, int]:
    """(reachable tiles incl. frontier, frontier tiles) per head (costs.py:45-55)."""
    n = tiles.padded_len(n)
    m_q, m_kv = n // tiles.b_m, n // tiles.b_n
    fr = sum(frontier_count(i, tiles, n) for i in range(m_q))
    if not causal:
        return m_q * m_kv, fr
    return sum(off_frontier_count(i, tiles) for i in range(m_q)) + fr, fr


def predicted_density(n: int, tiles: TileConfig, k: int) -> float:
    """sum_i (min(k, A_i) + F_i) / sum_i (A_i + F_i)  (costs.py:58-75)."""
    if k < 0:
        raise InvalidInputError(f"k must be >= 0, got {k}")
    n = tiles.padded_len(n)
    kept = total = 0
    for i in range(n // tiles.b_m):
        a, f = off_frontier_count(i, tiles), frontier_count(i, tiles, n)
        kept += min(k, a) + f
        total += a + f
    return kept / total


def k_for_density(n: int, tiles: TileConfig, density: float) -> int:
    """Smallest top-k budget whose predicted density reaches ``density``."""
    lo, hi = 0, tiles.padded_len(n) // tiles.b_n
    while lo < hi:
        mid = (lo + hi) // 2
        if predicted_density(n, tiles, mid) >= density:
            hi = mid
        else:
            lo = mid + 1
    return lo


def per_tile_flops(tiles: TileConfig, d: int) -> int:
    return 2 * tiles.b_m * tiles.b_n * d


def executed_flops(reachable: int, kept: int, tiles: TileConfig, d: int) -> int:
    """QK on every reachable tile + PV on every processed (frontier or kept) tile."""
    return per_tile_flops(tiles, d) * (int(reachable) + int(kept))


def dense_flops(reachable: int, tiles: TileConfig, d: int) -> int:
    return per_tile_flops(tiles, d) * 2 * int(reachable)


def kv_bytes(reachable: int, v_tiles: int, tiles: TileConfig, d: int, elem_bytes: int = 2) -> int:
    """K tile bytes streamed for every reachable tile + V bytes for fetched tiles (costs.py:119-125)."""
    return tiles.b_n * d * elem_bytes * (int(reachable) + int(v_tiles))
