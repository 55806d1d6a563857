"""GPU parity for the b_m = 64 tilings (64x64, 64x128) against the CPU oracle.

The reference admits any tiling where one block size divides the other
(tiling.py:26-32); its own tests run 64x64 and 64x128 next to the 128x64
default (test_engine.py, test_calibration.py, golden engine_09).  The kernels
run 128-row query tiles, so with b_m = 64 a tile holds query blocks 2t and
2t+1, each with its own threshold, frontier and decisions (engine.py:151-182);
a reference grid with an odd number of 64-blocks is padded to 128 rows and the
extra block is cropped (tiling.kernel_len).

Same tolerances as tests/test_gpu_parity.py: decisions equal to the oracle's
except gated tiles whose block max lies within EPS of the threshold; outputs
against the oracle engine replaying the GPU's decisions (max-abs, per-row
relative, LSE); calibration within 1e-4 of the oracle with identical sentinel
positions and tie counts.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import bsfa_oracle as orc  # noqa: E402
from test_gpu_parity import ATOL, EPS, LSE_ATOL, ROW_RTOL, _lse_err, _mask_parity, _row_rel_err, _smax_grid  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bsfa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_07011_b200 as m
    return m


def _inputs(rng, n, d, heads=None):
    shape = (n, d) if heads is None else heads + (n, d)
    return orc.round_bf16(rng.standard_normal(shape).astype(np.float32))


def _median_thresholds(q, k, b_m, b_n, rng, n_pad):
    """Per query block: the median of the oracle's off-frontier tile maxima, jittered (~50 % skip)."""
    grid = orc.tile_maxima_grid(q, k, b_m, b_n)
    fin = grid[np.isfinite(grid)]
    base = float(np.median(fin)) if fin.size else 0.0
    return (base + 0.05 * rng.standard_normal(n_pad // b_m)).astype(np.float32)


def _check_forward(out, trace, q, k, v, causal, b_m, b_n, gate_ref, thr=None):
    rec = {}
    o_ref, lse_ref, dec_ref = orc.flash_forward(q, k, v, causal, b_m, b_n, gate_ref, record=rec)
    assert trace.decisions.shape == dec_ref.shape
    if thr is None:
        np.testing.assert_array_equal(trace.decisions, dec_ref)
    else:
        smax = _smax_grid(rec, dec_ref.shape)
        bad = _mask_parity(trace.decisions, dec_ref, smax, lambda i: thr[min(i, len(thr) - 1)])
        assert not bad, bad[:5]
    o_rep, lse_rep, _ = orc.flash_forward(q, k, v, causal, b_m, b_n, orc.replay_gate(trace.decisions))
    assert np.abs(out.o - o_rep).max() <= ATOL
    assert _row_rel_err(out.o, o_rep) <= ROW_RTOL
    assert _lse_err(out.logsumexp, lse_rep) <= LSE_ATOL
    return dec_ref


# (n, d, causal, b_n): odd and even 64-block counts, ragged lengths, both head dims
FWD_CASES = [(1024, 128, True, 64), (448, 128, True, 64), (300, 64, True, 64), (500, 128, False, 64),
             (1024, 128, True, 128), (320, 64, True, 128), (200, 128, False, 128), (1984, 128, True, 64)]


@pytest.mark.parametrize("n,d,causal,b_n", FWD_CASES)
def test_bm64_threshold_forward(bsfa, n, d, causal, b_n):
    rng = np.random.default_rng(n * 7 + d + b_n + causal)
    q, k, v = (_inputs(rng, n, d) for _ in range(3))
    tiles = bsfa.TileConfig(64, b_n)
    n_pad = tiles.padded_len(n)
    thr = _median_thresholds(q, k, 64, b_n, rng, n_pad)
    t = bsfa.ThresholdTensor(values=thr[None, None, None], k_levels=(4,), n_max=n_pad, b_m=64, b_n=b_n)
    out, trace = bsfa.flash_forward(bsfa.HeadInput(q, k, v, causal=causal), tiles, bsfa.threshold_gate(t),
                                    bsfa.GateContext(k_level=4))
    dec = _check_forward(out, trace, q, k, v, causal, 64, b_n, orc.threshold_gate(thr), thr)
    gated = (dec == orc.KEPT) | (dec == orc.SKIPPED)
    if gated.sum() >= 20:  # the thresholds really split the gated tiles
        frac = float((dec[gated] == orc.KEPT).mean())
        assert 0.1 < frac < 0.9, frac


@pytest.mark.parametrize("b_n", [64, 128])
@pytest.mark.parametrize("kind", ["dense", "frontier", "window"])
def test_bm64_static_gates(bsfa, kind, b_n):
    rng = np.random.default_rng(5 + b_n)
    n, d = 576, 128  # 9 query blocks: the last tile holds one real block
    q, k, v = (_inputs(rng, n, d) for _ in range(3))
    tiles = bsfa.TileConfig(64, b_n)
    gate, ref = {
        "dense": (bsfa.dense_gate(), orc.dense_gate),
        "frontier": (bsfa.frontier_only_gate(), orc.frontier_only_gate),
        "window": (bsfa.SlidingWindowGate(192), orc.sliding_window_gate(192, 64, b_n)),
    }[kind]
    out, trace = bsfa.flash_forward(bsfa.HeadInput(q, k, v), tiles, gate)
    _check_forward(out, trace, q, k, v, True, 64, b_n, ref)
    if kind == "dense":
        o64, _ = orc.dense_attention(q, k, v, True)
        assert np.abs(out.o - o64).max() <= ATOL


@pytest.mark.parametrize("lam,b_n", [(0.5, 64), (-0.5, 64), (0.5, 128)])
def test_bm64_running_max_gate(bsfa, lam, b_n):
    """RunningMaxGate (gates.py:101-118) per 64-row block, gate tiles of a step in key order."""
    rng = np.random.default_rng(int(10 * lam) + b_n + 3)
    n, d = 1088, 128
    q, k, v = (_inputs(rng, n, d) for _ in range(3))
    tiles = bsfa.TileConfig(64, b_n)
    out, trace = bsfa.flash_forward(bsfa.HeadInput(q, k, v), tiles, bsfa.RunningMaxGate(lam))
    diffs = {}

    def recording_gate(s, i, j, m):
        with np.errstate(invalid="ignore"):
            dmax = float((s.max(axis=1) - m).max())
        diffs[(i, j)] = dmax
        return dmax >= lam

    _, _, dec_ref = orc.flash_forward(q, k, v, True, 64, b_n, recording_gate)
    bad = [(i, j) for (i, j) in zip(*np.nonzero(trace.decisions != dec_ref))
           if not abs(diffs.get((int(i), int(j)), np.inf) - lam) <= EPS]
    assert not bad, bad[:5]
    dec = trace.decisions
    if lam >= 0:
        assert (dec == orc.SKIPPED).any() and (dec == orc.KEPT).any()
    o_rep, lse_rep, _ = orc.flash_forward(q, k, v, True, 64, b_n, orc.replay_gate(dec))
    assert np.abs(out.o - o_rep).max() <= ATOL and _lse_err(out.logsumexp, lse_rep) <= LSE_ATOL


@pytest.mark.parametrize("B,hq,hkv,n,causal,b_n", [(2, 4, 2, 704, True, 64), (1, 3, 1, 448, True, 64),
                                                   (2, 4, 2, 640, False, 128), (1, 8, 2, 1088, True, 64)])
def test_bm64_batched_gqa_and_counters(bsfa, B, hq, hkv, n, causal, b_n):
    """attention() over (batch, GQA heads) -- head pairs per CTA, or query-block pairs for odd
    groups -- against the oracle per head; counters equal the decision-grid counts."""
    rng = np.random.default_rng(B * 1000 + hq * 10 + n)
    d = 128
    q = _inputs(rng, n, d, (B, hq))
    k = _inputs(rng, n, d, (B, hkv))
    v = _inputs(rng, n, d, (B, hkv))
    tiles = bsfa.TileConfig(64, b_n)
    n_pad = tiles.padded_len(n)
    g = hq // hkv
    thr = np.stack([_median_thresholds(q[0, h], k[0, h // g], 64, b_n, rng, n_pad) for h in range(hq)])
    t = bsfa.ThresholdTensor(values=thr[None, None], k_levels=(3,), n_max=n_pad, b_m=64, b_n=b_n)
    dev = lambda x: torch.from_numpy(x).cuda().to(torch.bfloat16)  # noqa: E731
    res = bsfa.attention(dev(q), dev(k), dev(v), causal=causal, tiles=tiles, thresholds=t, k_level=3,
                         return_trace=True)
    dec = res.decisions.cpu().numpy()
    assert dec.shape == (B, hq, n_pad // 64, n_pad // b_n)
    o = res.o.float().cpu().numpy()
    lse = res.lse.cpu().numpy()
    for b in range(B):
        for h in range(hq):
            rec = {}
            _, _, dec_ref = orc.flash_forward(q[b, h], k[b, h // g], v[b, h // g], causal, 64, b_n,
                                              orc.threshold_gate(thr[h]), record=rec)
            smax = _smax_grid(rec, dec_ref.shape)
            bad = _mask_parity(dec[b, h], dec_ref, smax, lambda i: thr[h][min(i, len(thr[h]) - 1)])
            assert not bad, (b, h, bad[:5])
            o_rep, lse_rep, _ = orc.flash_forward(q[b, h], k[b, h // g], v[b, h // g], causal, 64, b_n,
                                                  orc.replay_gate(dec[b, h]))
            assert np.abs(o[b, h] - o_rep).max() <= ATOL and _row_rel_err(o[b, h], o_rep) <= ROW_RTOL
            assert _lse_err(lse[b, h], lse_rep) <= LSE_ATOL
    cnt = res.counters.cpu().numpy()
    assert int(cnt[0]) == int((dec != orc.UNREACHABLE).sum())
    assert int(cnt[1]) == int((dec >= orc.FRONTIER).sum())


@pytest.mark.parametrize("b_n,lengths", [(64, (448, 512, 300)), (128, (320, 512))])
def test_bm64_calibration_matches_oracle(bsfa, b_n, lengths):
    """calibrate() with 64-row blocks (calibration.py:156-222): thresholds, sentinel positions and
    tie counts against the oracle on samples of mixed lengths (odd block counts included)."""
    rng = np.random.default_rng(41 + b_n)
    L, H, Hkv, d = 2, 2, 1, 64
    samples, ref_samples = [], []
    for sid, n in enumerate(lengths):
        q = _inputs(rng, n, d, (L, H))
        k = _inputs(rng, n, d, (L, Hkv))
        samples.append(bsfa.CalibrationSample(sample_id=sid, q=q, k=np.repeat(k, H // Hkv, axis=1)))
        ref_samples.append((sid, q, k))
    tiles = bsfa.TileConfig(64, b_n)
    levels = [0, 1, 3, 6]
    t = bsfa.calibrate(bsfa.CalibrationDump(L, H, d, samples), levels, tiles)
    ref, n_max, ties = orc.calibrate(ref_samples, levels, 64, b_n)
    assert t.n_max == n_max and t.values.shape == ref.shape
    fin = np.isfinite(ref)
    np.testing.assert_array_equal(np.isfinite(t.values), fin)
    np.testing.assert_array_equal(t.values[~fin], ref[~fin])
    assert np.abs(t.values[fin] - ref[fin]).max() <= 1e-4
    assert {kk: t.diagnostics.tie_counts[kk] for kk in levels} == {kk: int(ties[kk]) for kk in levels}
    prof = bsfa.collect_block_maxima(samples[0], tiles)
    ref_prof = orc.block_maxima(ref_samples[0][1][1, 1], ref_samples[0][2][1, 0], 64, b_n)
    assert prof.num_positions == len(ref_prof)
    for p, vals in enumerate(ref_prof):
        np.testing.assert_allclose(prof.maxima[(1, 1, p)], vals, atol=1e-4)


def test_bm64_topk_round_trip(bsfa):
    """Reference acceptance 3 (test_acceptance.py:94-117) at 64x64: calibrate on a sample, gate the
    same sample -> every query block keeps exactly min(k, A_i) off-frontier tiles."""
    rng = np.random.default_rng(77)
    L, H, n, d = 1, 2, 1088, 128
    q = _inputs(rng, n, d, (L, H))
    k = _inputs(rng, n, d, (L, H))
    v = _inputs(rng, n, d, (L, H))
    tiles = bsfa.TileConfig(64, 64)
    k_levels = [1, 4, 9]
    t = bsfa.calibrate(bsfa.CalibrationDump(L, H, d, [bsfa.CalibrationSample(0, q, k)]), k_levels, tiles)
    assert all(x == 0 for x in t.diagnostics.tie_counts.values())
    dev = lambda x: torch.from_numpy(x).cuda().to(torch.bfloat16)  # noqa: E731
    for kk in k_levels:
        res = bsfa.attention(dev(q[0])[None], dev(k[0])[None], dev(v[0])[None], tiles=tiles, thresholds=t,
                             k_level=kk, return_trace=True)
        dec = res.decisions[0].cpu().numpy()
        for h in range(H):
            for i in range(dec.shape[2]):
                a = orc.off_frontier(i, 64, 64)
                kept = int((dec[h, i, :a] == orc.KEPT).sum())
                assert kept == min(kk, a), (kk, h, i, kept)


def test_block_maxima_buffer_validated(bsfa):
    """A caller's block_maxima buffer must match the kernel grid (kernel_len rows) before the launch."""
    rng = np.random.default_rng(3)
    n, d = 448, 64
    q = _inputs(rng, n, d, (2,))
    k = _inputs(rng, n, d, (1,))
    tiles = bsfa.TileConfig(64, 64)
    cal = bsfa.Calibrator([1], tiles, 1, 2, n, d, device="cuda")
    nk = bsfa.kernel_len(n, tiles)
    with pytest.raises(bsfa.InvalidInputError):
        cal.add_layer(0, 0, q, k, block_maxima=torch.zeros((2, n // 64, n // 64), device="cuda"))
    ok = torch.full((2, nk // 64, nk // 64), float("nan"), device="cuda")
    cal.add_layer(0, 0, q, k, block_maxima=ok)
    ref = orc.block_maxima(q[1], k[0], 64, 64)
    got = ok[1].cpu().numpy()
    for p, vals in enumerate(ref):
        np.testing.assert_allclose(np.sort(got[p, :len(vals)])[::-1], vals, atol=1e-4)


def test_bm64_torch_ops(bsfa):
    """torch.ops.bsfa.fwd / blockmax / calib_select at 64x64 on an odd block count: the op equals
    attention() bit for bit, the block maxima equal the oracle's, the selected cutoffs its calibrate()."""
    rng = np.random.default_rng(9)
    n, d = 704, 128
    q = _inputs(rng, n, d, (1, 2))
    k = _inputs(rng, n, d, (1, 1))
    v = _inputs(rng, n, d, (1, 1))
    dev = lambda x: torch.from_numpy(x).cuda().to(torch.bfloat16)  # noqa: E731
    tiles = bsfa.TileConfig(64, 64)
    thr = np.stack([_median_thresholds(q[0, h], k[0, 0], 64, 64, rng, n) for h in range(2)])
    t = bsfa.ThresholdTensor(values=thr[None, None], k_levels=(2,), n_max=n, b_m=64, b_n=64)
    ref = bsfa.attention(dev(q), dev(k), dev(v), tiles=tiles, thresholds=t, k_level=2, return_trace=True)
    o, lse, cnt, dec = torch.ops.bsfa.fwd(dev(q), dev(k), dev(v), torch.from_numpy(thr).cuda(), True, 64, 64,
                                          bsfa.reference_scale(d), True)
    assert torch.equal(o, ref.o) and torch.equal(lse, ref.lse) and torch.equal(dec, ref.decisions)
    assert torch.equal(cnt[:2], ref.counters[:2])
    bm = torch.ops.bsfa.blockmax(dev(q), dev(np.repeat(k, 2, axis=1)), 64, 64)
    assert tuple(bm.shape) == (1, 2, n // 64, n // 64)
    for h in range(2):
        prof = orc.block_maxima(q[0, h], k[0, 0], 64, 64)
        got = bm[0, h].cpu().numpy()
        for p, vals in enumerate(prof):
            np.testing.assert_allclose(np.sort(got[p, :len(vals)])[::-1], vals, atol=1e-4)
    levels = [1, 3]
    sel, _ = torch.ops.bsfa.calib_select(bm, levels, 64, 64)
    ref_vals, _, _ = orc.calibrate([(0, q, k)], levels, 64, 64)
    got = sel.cpu().numpy()[:, 0]  # [levels, heads, positions]
    want = ref_vals[:, 0]
    fin = np.isfinite(want)
    np.testing.assert_array_equal(np.isfinite(got), fin)
    assert np.abs(got[fin] - want[fin]).max() <= 1e-4
