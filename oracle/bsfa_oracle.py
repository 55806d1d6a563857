"""CPU oracle for the BSFA hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in numpy, the reference algorithm of the path the
CUDA kernels implement.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it,
and only as the checker / CPU baseline -- never as a product code path.

Pinned: ``tests/golden/*.npz`` were produced by running the *reference*
package (/root/reference/pkg/src/bsfa, imported in the build container by
``tests/golden/make_golden.py``) on seeded inputs; ``tests/test_oracle.py``
checks every function below against those vectors and against the
reference's own known-answer tests.

Reference citations are ``pkg/src/bsfa/<file>:<lines>``.
"""

from __future__ import annotations

import math

import numpy as np

UNREACHABLE, SKIPPED, FRONTIER, KEPT = 0, 1, 2, 3


# ----------------------------------------------------------------- geometry
# tiling.py:19-69
def alignment(b_m: int, b_n: int) -> int:
    return math.lcm(b_m, b_n)


def padded_len(n: int, b_m: int, b_n: int) -> int:
    a = alignment(b_m, b_n)
    return -(-n // a) * a


def frontier(i: int, b_m: int, b_n: int, n: int | None = None) -> range:
    lo = (i * b_m) // b_n
    hi = -(-((i + 1) * b_m) // b_n)
    if n is not None:
        hi = min(hi, -(-n // b_n))
    return range(lo, hi)


def off_frontier(i: int, b_m: int, b_n: int) -> int:
    return (i * b_m) // b_n


def pad_rows(m: np.ndarray, target: int) -> np.ndarray:
    """Repeat the last row up to ``target`` rows (engine.py:99-114, calibration.py:87-90)."""
    if m.shape[0] == target:
        return m
    return np.concatenate([m, np.repeat(m[-1:], target - m.shape[0], axis=0)])


def scale_for(d: int) -> np.float32:
    return np.float32(1.0 / np.sqrt(d))  # engine.py:144


# ----------------------------------------------------------------- fp64 oracle
# core.py:104-142
def reference_attention(q, k, v, allow) -> tuple[np.ndarray, np.ndarray]:
    """Restricted softmax attention in float64 over an explicit (n, n) key mask."""
    if not allow.any(axis=1).all():
        raise ValueError("a query row has an empty allowed key set")
    q64, k64, v64 = (np.asarray(x, dtype=np.float64) for x in (q, k, v))
    s = (q64 @ k64.T) / np.sqrt(np.float64(q64.shape[1]))
    s = np.where(allow, s, -np.inf)
    m = s.max(axis=1)
    p = np.exp(s - m[:, None])
    l = p.sum(axis=1)
    return (p @ v64) / l[:, None], m + np.log(l)


def causal_allow(n: int) -> np.ndarray:
    idx = np.arange(n)
    return idx[None, :] <= idx[:, None]


def dense_attention(q, k, v, causal=True):
    n = q.shape[0]
    allow = causal_allow(n) if causal else np.ones((n, n), dtype=bool)
    return reference_attention(q, k, v, allow)


def masked_dense_attention(q, k, v, decisions, b_m, b_n, causal=True):
    """Dense attention restricted to blocks with code >= FRONTIER (core.py:133-142)."""
    n = q.shape[0]
    rb = np.arange(n) // b_m
    kb = np.arange(n) // b_n
    allow = (np.asarray(decisions) >= FRONTIER)[rb][:, kb]
    if causal:
        allow &= causal_allow(n)
    return reference_attention(q, k, v, allow)


def max_rel_err(actual, expected) -> float:
    a = np.asarray(actual, dtype=np.float64)
    e = np.asarray(expected, dtype=np.float64)
    return float(np.max(np.abs(a - e)) / (1.0 + np.max(np.abs(e))))  # core.py:145-149


# ----------------------------------------------------------------- gates
# gates.py:41-118 as plain callables  keep = gate(s_tile, i, j, m_running)
def dense_gate(s, i, j, m):
    return True


def frontier_only_gate(s, i, j, m):
    return False


def threshold_gate(thresholds_per_block):
    """Keep iff tile max > T[min(i, P-1)], strict (gates.py:77-78, thresholds.py:87)."""
    t = np.asarray(thresholds_per_block, dtype=np.float32)

    def gate(s, i, j, m):
        return float(s.max()) > float(t[min(i, t.shape[0] - 1)])
    return gate


def replay_gate(decisions):
    """Replays an externally produced decision grid (e.g. the GPU's)."""
    dec = np.asarray(decisions)

    def gate(s, i, j, m):
        return bool(dec[i, j] == KEPT)
    return gate


def sliding_window_gate(window, b_m, b_n):
    def gate(s, i, j, m):  # gates.py:81-98
        return (j + 1) * b_n > i * b_m - window and j * b_n < (i + 1) * b_m
    return gate


def running_max_gate(lam):
    def gate(s, i, j, m):  # gates.py:101-118
        return bool((s.max(axis=1) - m).max() >= lam)
    return gate


# ----------------------------------------------------------------- engine
# engine.py:117-193, tile by tile
def flash_forward(q, k, v, causal, b_m, b_n, gate, record=None, q_blocks=None):
    """Tiled online-softmax forward with a per-off-frontier-tile gate.

    Returns (o, lse, decisions) with decisions on the padded grid.  If
    ``record`` is a dict, ``record[(i, j)] = s_max`` for every gated tile.
    ``q_blocks`` restricts the run to those query blocks (query blocks are
    independent; rows of other blocks are left uninitialised).
    """
    q = np.ascontiguousarray(q, dtype=np.float32)
    k = np.ascontiguousarray(k, dtype=np.float32)
    v = np.ascontiguousarray(v, dtype=np.float32)
    valid = q.shape[0]
    n = padded_len(valid, b_m, b_n)
    q, k, v = pad_rows(q, n), pad_rows(k, n), pad_rows(v, n)
    d = q.shape[1]
    m_q, m_kv = n // b_m, n // b_n
    scale = scale_for(d)
    out = np.empty((n, d), dtype=np.float32)
    lse = np.empty(n, dtype=np.float32)
    dec = np.zeros((m_q, m_kv), dtype=np.int8)
    neg_inf = np.float32(-np.inf)
    for i in (range(m_q) if q_blocks is None else q_blocks):
        fr = frontier(i, b_m, b_n)
        last = fr.stop - 1 if causal else m_kv - 1
        m = np.full(b_m, -np.inf, dtype=np.float32)
        l = np.zeros(b_m, dtype=np.float32)
        acc = np.zeros((b_m, d), dtype=np.float32)
        qi = q[i * b_m:(i + 1) * b_m]
        rows = np.arange(i * b_m, (i + 1) * b_m)
        for j in range(last + 1):
            s = (qi @ k[j * b_n:(j + 1) * b_n].T) * scale
            cols = np.arange(j * b_n, (j + 1) * b_n)
            if not causal and (j + 1) * b_n > valid:
                s[:, cols >= valid] = neg_inf
            if j in fr:
                if causal:
                    s[rows[:, None] < cols[None, :]] = neg_inf
                dec[i, j] = FRONTIER
            else:
                if record is not None:
                    record[(i, j)] = float(s.max())
                keep = gate(s, i, j, m)
                dec[i, j] = KEPT if keep else SKIPPED
                if not keep:
                    continue
            # RunningStats.update, engine.py:57-68
            m_new = np.maximum(m, s.max(axis=1))
            m_safe = np.where(np.isneginf(m_new), np.float32(0.0), m_new)
            p = np.exp(s - m_safe[:, None])
            alpha = np.exp(m - m_safe)
            acc *= alpha[:, None]
            acc += p @ v[j * b_n:(j + 1) * b_n]
            l = l * alpha + p.sum(axis=1)
            m = m_new
        if not np.isfinite(acc).all() or not (l > 0).all():
            raise ArithmeticError(f"non-finite accumulator in query block {i}")
        out[i * b_m:(i + 1) * b_m] = acc / l[:, None]
        lse[i * b_m:(i + 1) * b_m] = m + np.log(l)
    return out[:valid], lse[:valid], dec


def flash_forward_fast(q, k, v, causal, b_m, b_n, keep_fn, record=None, q_blocks=None):
    """Same algorithm as :func:`flash_forward`, vectorised over query blocks.

    Processes key block j for every query block that reaches it in one
    sgemm, so a 32K-token head takes seconds instead of minutes.  Per row the
    arithmetic is the reference's (same tile scores, same update order);
    only BLAS blocking differs.  ``keep_fn(i_idx, j, smax) -> bool array``
    decides the gated tiles; ``record`` (dict) receives smax arrays per j.
    ``q_blocks`` restricts the run to those query blocks (rows of the other
    blocks come back NaN), e.g. the longest rows of a 128K head.
    """
    q = np.ascontiguousarray(q, dtype=np.float32)
    k = np.ascontiguousarray(k, dtype=np.float32)
    v = np.ascontiguousarray(v, dtype=np.float32)
    valid = q.shape[0]
    n = padded_len(valid, b_m, b_n)
    q, k, v = pad_rows(q, n), pad_rows(k, n), pad_rows(v, n)
    d = q.shape[1]
    m_q, m_kv = n // b_m, n // b_n
    scale = scale_for(d)
    neg_inf = np.float32(-np.inf)
    m = np.full((m_q, b_m), -np.inf, dtype=np.float32)
    l = np.zeros((m_q, b_m), dtype=np.float32)
    acc = np.zeros((m_q, b_m, d), dtype=np.float32)
    dec = np.zeros((m_q, m_kv), dtype=np.int8)
    fr_lo = np.array([frontier(i, b_m, b_n).start for i in range(m_q)])
    fr_hi = np.array([frontier(i, b_m, b_n).stop for i in range(m_q)])
    last = fr_hi - 1 if causal else np.full(m_q, m_kv - 1)
    q3 = q.reshape(m_q, b_m, d)
    rows = np.arange(n).reshape(m_q, b_m)
    active = np.ones(m_q, dtype=bool)
    if q_blocks is not None:
        active[:] = False
        active[list(q_blocks)] = True
    for j in range(m_kv):
        idx = np.nonzero((last >= j) & active)[0]
        if idx.size == 0:
            continue
        kj = k[j * b_n:(j + 1) * b_n]
        s = (q3[idx].reshape(-1, d) @ kj.T).reshape(idx.size, b_m, b_n) * scale
        cols = np.arange(j * b_n, (j + 1) * b_n)
        if not causal and (j + 1) * b_n > valid:
            s[:, :, cols >= valid] = neg_inf
        is_fr = (fr_lo[idx] <= j) & (j < fr_hi[idx])
        if causal and is_fr.any():
            fi = np.nonzero(is_fr)[0]
            mask = rows[idx[fi]][:, :, None] < cols[None, None, :]
            sf = s[fi]
            sf[mask] = neg_inf
            s[fi] = sf
        smax = s.reshape(idx.size, -1).max(axis=1)
        gated = ~is_fr
        keep = np.ones(idx.size, dtype=bool)
        if gated.any():
            gk = np.asarray(keep_fn(idx[gated], j, smax[gated]), dtype=bool)
            keep[gated] = gk
            if record is not None:
                record[j] = (idx[gated], smax[gated])
        dec[idx, j] = np.where(is_fr, FRONTIER, np.where(keep, KEPT, SKIPPED))
        ki = idx[keep]
        if ki.size == 0:
            continue
        sk = s[keep]
        mk = m[ki]
        m_new = np.maximum(mk, sk.max(axis=2))
        m_safe = np.where(np.isneginf(m_new), np.float32(0.0), m_new)
        p = np.exp(sk - m_safe[:, :, None])
        alpha = np.exp(mk - m_safe)
        pv = (p.reshape(-1, b_n) @ v[j * b_n:(j + 1) * b_n]).reshape(ki.size, b_m, d)
        acc[ki] = acc[ki] * alpha[:, :, None] + pv
        l[ki] = l[ki] * alpha + p.sum(axis=2)
        m[ki] = m_new
    if not np.isfinite(acc[active]).all() or not (l[active] > 0).all():
        raise ArithmeticError("non-finite accumulator")
    with np.errstate(divide="ignore", invalid="ignore"):
        out = (acc / l[:, :, None])
        lse = m + np.log(l)
    out[~active] = np.nan
    lse[~active] = np.nan
    return out.reshape(n, d)[:valid], lse.reshape(n)[:valid], dec


# engine.py:157-171: s_max of every gated (off-frontier, causal) tile, without the softmax
def tile_maxima_grid(q, k, b_m, b_n):
    """(m_q, m_kv) grid of max(q_i k_j^T * scale) over each off-frontier causal tile; NaN elsewhere.

    The statistic ThresholdGate compares (gates.py:77-78) for every gated tile of
    a causal head, one sgemm per query block: the mask-parity checker for
    sequences whose full forward oracle is too slow (128K tokens).
    """
    q = np.ascontiguousarray(q, dtype=np.float32)
    k = np.ascontiguousarray(k, dtype=np.float32)
    n = padded_len(q.shape[0], b_m, b_n)
    q, k = pad_rows(q, n), pad_rows(k, n)
    scale = scale_for(q.shape[1])
    m_q, m_kv = n // b_m, n // b_n
    grid = np.full((m_q, m_kv), np.nan, dtype=np.float32)
    for i in range(m_q):
        a = off_frontier(i, b_m, b_n)
        if a == 0:
            continue
        s = (q[i * b_m:(i + 1) * b_m] @ k[:a * b_n].T) * scale
        grid[i, :a] = s.reshape(b_m, a, b_n).max(axis=(0, 2))
    return grid


# ----------------------------------------------------------------- thresholds
# thresholds.py:75-88
def threshold_lookup(values, level_idx, layer, head, query_block):
    p = min(query_block, values.shape[3] - 1)
    return float(values[level_idx, layer, head, p])


# ----------------------------------------------------------------- calibration
# calibration.py:93-123 (maxima of the off-frontier causal prefix, descending)
def block_maxima(q, k, b_m, b_n):
    """q, k: (n, d) one head.  Returns list over positions p of descending arrays."""
    q = np.ascontiguousarray(q, dtype=np.float32)
    k = np.ascontiguousarray(k, dtype=np.float32)
    n_pad = padded_len(q.shape[0], b_m, b_n)
    q, k = pad_rows(q, n_pad), pad_rows(k, n_pad)
    scale = scale_for(q.shape[1])
    out = []
    for p in range(n_pad // b_m):
        a = off_frontier(p, b_m, b_n)
        qp = q[p * b_m:(p + 1) * b_m]
        if a == 0:
            out.append(np.empty(0, dtype=np.float32))
            continue
        s = (qp @ k[:a * b_n].T) * scale
        vals = s.reshape(b_m, a, b_n).max(axis=(0, 2)).astype(np.float32)
        out.append(np.sort(vals)[::-1].copy())
    return out


# calibration.py:126-153
def cutoff(vals: np.ndarray, k: int) -> float:
    if k == 0:
        return np.inf
    if len(vals) <= k:
        return -np.inf
    return float(np.float64(vals[k]))


def is_tie(vals: np.ndarray, k: int) -> bool:
    return k > 0 and len(vals) > k and vals[k - 1] == vals[k]


# calibration.py:156-222
def calibrate(samples, k_levels, b_m, b_n):
    """samples: list of (sample_id, q (L,H,N,d), k (L,Hkv,N,d)).

    Returns (values float32 (S,L,H,P), n_max, tie_counts dict).  GQA samples
    map q head h to kv head h // (H / Hkv) (the reference requires H == Hkv).
    """
    k_levels = [int(x) for x in k_levels]
    if not samples:
        raise ValueError("no samples")
    if not k_levels or any(a >= b for a, b in zip(k_levels, k_levels[1:])):
        raise ValueError("k levels must be non-empty and strictly increasing")
    samples = sorted(samples, key=lambda s: s[0])
    n_max = max(padded_len(s[1].shape[2], b_m, b_n) for s in samples)
    L, H = samples[0][1].shape[:2]
    P = n_max // b_m
    shape = (len(k_levels), L, H, P)
    fsum = np.zeros(shape)
    fcnt = np.zeros(shape, dtype=np.int64)
    ncnt = np.zeros(shape, dtype=np.int64)
    pcnt = np.zeros(shape, dtype=np.int64)
    ties = {kk: 0 for kk in k_levels}
    for _, sq, sk in samples:
        group = sq.shape[1] // sk.shape[1]
        for l in range(L):
            for h in range(H):
                prof = block_maxima(sq[l, h], sk[l, h // group], b_m, b_n)
                for si, kk in enumerate(k_levels):
                    for p, vals in enumerate(prof):
                        c = cutoff(vals, kk)
                        ties[kk] += int(is_tie(vals, kk))
                        if np.isfinite(c):
                            fsum[si, l, h, p] += c
                            fcnt[si, l, h, p] += 1
                        elif c < 0:
                            ncnt[si, l, h, p] += 1
                        else:
                            pcnt[si, l, h, p] += 1
    with np.errstate(invalid="ignore", divide="ignore"):
        vals = np.where(fcnt > 0, fsum / np.maximum(fcnt, 1), 0.0)
    vals = np.where((fcnt == 0) & (ncnt > 0), -np.inf, vals)
    vals = np.where((fcnt == 0) & (ncnt == 0) & (pcnt > 0), np.inf, vals)
    return vals.astype(np.float32), n_max, ties


# ----------------------------------------------------------------- workloads
# workloads.py:58-77 (seeded per (seed, sample, layer, head, tag) streams)
def rng_for(seed, sample, layer, head, tag):
    return np.random.default_rng(np.random.SeedSequence([seed, sample, layer, head, tag]))


def gen_random(n, d, seed=0, sample=0, layer=0, head=0):
    q = rng_for(seed, sample, layer, head, 0).standard_normal((n, d)).astype(np.float32)
    k = rng_for(seed, sample, layer, head, 1).standard_normal((n, d)).astype(np.float32)
    v = rng_for(seed, sample, layer, head, 2).standard_normal((n, d)).astype(np.float32)
    return q, k, v


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 to the nearest bf16 value (ties to even), returned as float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    out = r.astype(np.uint32).view(np.float32)
    return np.where(np.isfinite(x), out, x).astype(np.float32)
