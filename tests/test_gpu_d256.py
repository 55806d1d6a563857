"""GPU parity for head_dim 129..256 (kernels at d = 256) against the CPU oracle.

The reference accepts any head dimension (core.py:20-56, engine.py:144 scale =
1/sqrt(d)).  The kernels run d = 256 with ONE query tile per CTA whose O spans
both O slots of the d = 128 TMEM layout; narrower heads are zero-padded to 256
and use their own scale.  Same tolerances as tests/test_gpu_parity.py.
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


def _inputs(rng, shape):
    return orc.round_bf16(rng.standard_normal(shape).astype(np.float32))


def _thresholds(q, k, b_m, b_n, rng, n_pad):
    grid = orc.tile_maxima_grid(q, k, b_m, b_n)
    fin = grid[np.isfinite(grid)]
    base = float(np.median(fin)) if fin.size else 0.0
    return (base + 0.05 * rng.standard_normal(n_pad // b_m)).astype(np.float32)


@pytest.mark.parametrize("n,d,causal,b_m,b_n", [(1024, 256, True, 128, 64), (2048, 256, True, 128, 64),
                                                (700, 192, True, 128, 64), (1000, 160, False, 128, 128),
                                                (640, 256, True, 64, 64), (512, 256, False, 64, 128)])
def test_d256_threshold_forward(bsfa, n, d, causal, b_m, b_n):
    rng = np.random.default_rng(n + d + b_m + b_n)
    q, k, v = (_inputs(rng, (n, d)) for _ in range(3))
    tiles = bsfa.TileConfig(b_m, b_n)
    n_pad = tiles.padded_len(n)
    thr = _thresholds(q, k, b_m, b_n, rng, n_pad)
    t = bsfa.ThresholdTensor(values=thr[None, None, None], k_levels=(4,), n_max=n_pad, b_m=b_m, b_n=b_n)
    out, trace = bsfa.flash_forward(bsfa.HeadInput(q, k, v, causal=causal), tiles, bsfa.threshold_gate(t),
                                    bsfa.GateContext(k_level=4))
    rec = {}
    _, _, dec_ref = orc.flash_forward(q, k, v, causal, b_m, b_n, orc.threshold_gate(thr), record=rec)
    bad = _mask_parity(trace.decisions, dec_ref, _smax_grid(rec, dec_ref.shape), lambda i: thr[min(i, len(thr) - 1)])
    assert not bad, bad[:5]
    o_rep, lse_rep, _ = orc.flash_forward(q, k, v, causal, b_m, b_n, orc.replay_gate(trace.decisions))
    assert out.o.shape == (n, d)
    assert np.abs(out.o - o_rep).max() <= ATOL
    assert _row_rel_err(out.o, o_rep) <= ROW_RTOL
    assert _lse_err(out.logsumexp, lse_rep) <= LSE_ATOL


@pytest.mark.parametrize("kind", ["dense", "frontier", "window", "runmax"])
def test_d256_other_gates(bsfa, kind):
    rng = np.random.default_rng(11)
    n, d = 1152, 256
    q, k, v = (_inputs(rng, (n, d)) for _ in range(3))
    tiles = bsfa.TileConfig(128, 64)
    gate, ref = {
        "dense": (bsfa.dense_gate(), orc.dense_gate),
        "frontier": (bsfa.frontier_only_gate(), orc.frontier_only_gate),
        "window": (bsfa.SlidingWindowGate(300), orc.sliding_window_gate(300, 128, 64)),
        "runmax": (bsfa.RunningMaxGate(0.5), None),
    }[kind]
    out, trace = bsfa.flash_forward(bsfa.HeadInput(q, k, v), tiles, gate)
    if ref is not None:
        _, _, dec_ref = orc.flash_forward(q, k, v, True, 128, 64, ref)
        np.testing.assert_array_equal(trace.decisions, dec_ref)
    else:
        diffs = {}

        def recording_gate(s, i, j, m):
            with np.errstate(invalid="ignore"):
                dmax = float((s.max(axis=1) - m).max())
            diffs[(i, j)] = dmax
            return dmax >= 0.5

        _, _, dec_ref = orc.flash_forward(q, k, v, True, 128, 64, recording_gate)
        bad = [(i, j) for (i, j) in zip(*np.nonzero(trace.decisions != dec_ref))
               if not abs(diffs.get((int(i), int(j)), np.inf) - 0.5) <= EPS]
        assert not bad, bad[:5]
    o_rep, lse_rep, _ = orc.flash_forward(q, k, v, True, 128, 64, orc.replay_gate(trace.decisions))
    assert np.abs(out.o - o_rep).max() <= ATOL and _lse_err(out.logsumexp, lse_rep) <= LSE_ATOL
    if kind == "dense":
        o64, _ = orc.dense_attention(q, k, v, True)
        assert np.abs(out.o - o64).max() <= ATOL


def test_d256_batched_gqa_counters_and_plan(bsfa):
    """attention() over (batch, GQA heads) at d = 256 against the oracle per head; counters equal
    the decision-grid counts; a BsfaPlan run is bit-identical to attention()."""
    rng = np.random.default_rng(23)
    B, hq, hkv, n, d = 2, 4, 2, 1536, 256
    q = _inputs(rng, (B, hq, n, d))
    k = _inputs(rng, (B, hkv, n, d))
    v = _inputs(rng, (B, hkv, n, d))
    g = hq // hkv
    thr = np.stack([_thresholds(q[0, h], k[0, h // g], 128, 64, rng, n) for h in range(hq)])
    t = bsfa.ThresholdTensor(values=thr[None, None], k_levels=(2,), n_max=n, b_m=128, b_n=64)
    dev = lambda x: torch.from_numpy(x).cuda().to(torch.bfloat16)  # noqa: E731
    res = bsfa.attention(dev(q), dev(k), dev(v), thresholds=t, k_level=2, return_trace=True)
    dec = res.decisions.cpu().numpy()
    o = res.o.float().cpu().numpy()
    for b in range(B):
        for h in range(hq):
            rec = {}
            _, _, dec_ref = orc.flash_forward(q[b, h], k[b, h // g], v[b, h // g], True, 128, 64,
                                              orc.threshold_gate(thr[h]), record=rec)
            bad = _mask_parity(dec[b, h], dec_ref, _smax_grid(rec, dec_ref.shape), lambda i: thr[h][min(i, 11)])
            assert not bad, (b, h, bad[:5])
            o_rep, _, _ = orc.flash_forward(q[b, h], k[b, h // g], v[b, h // g], True, 128, 64,
                                            orc.replay_gate(dec[b, h]))
            assert np.abs(o[b, h] - o_rep).max() <= ATOL and _row_rel_err(o[b, h], o_rep) <= ROW_RTOL
    cnt = res.counters.cpu().numpy()
    assert int(cnt[0]) == int((dec != orc.UNREACHABLE).sum()) and int(cnt[1]) == int((dec >= orc.FRONTIER).sum())
    plan = bsfa.BsfaPlan(B, hq, hkv, n, d, thresholds=t, k_level=2, return_trace=True)
    po = plan.run(dev(q), dev(k), dev(v))
    torch.cuda.synchronize()
    assert torch.equal(po, res.o) and torch.equal(plan.decisions, res.decisions)


@pytest.mark.parametrize("d,b_m", [(256, 128), (200, 64)])
def test_d256_calibration_matches_oracle(bsfa, d, b_m):
    rng = np.random.default_rng(d + b_m)
    L, H, Hkv = 1, 2, 1
    samples, ref_samples = [], []
    for sid, n in enumerate((1024, 832)):
        q = _inputs(rng, (L, H, n, d))
        k = _inputs(rng, (L, Hkv, n, d))
        samples.append(bsfa.CalibrationSample(sample_id=sid, q=q, k=np.repeat(k, H // Hkv, axis=1)))
        ref_samples.append((sid, q, k))
    tiles = bsfa.TileConfig(b_m, 64)
    levels = [0, 2, 5]
    t = bsfa.calibrate(bsfa.CalibrationDump(L, H, d, samples), levels, tiles)
    ref, n_max, ties = orc.calibrate(ref_samples, levels, b_m, 64)
    assert t.n_max == n_max
    fin = np.isfinite(ref)
    np.testing.assert_array_equal(np.isfinite(t.values), fin)
    np.testing.assert_array_equal(t.values[~fin], ref[~fin])
    assert np.abs(t.values[fin] - ref[fin]).max() <= 1e-4
    assert {kk: t.diagnostics.tie_counts[kk] for kk in levels} == {kk: int(ties[kk]) for kk in levels}


@pytest.mark.parametrize("T", [3.9, 9.0])
def test_d256_at_scale_sampled_heads(bsfa, T):
    """16 q / 8 kv heads x 16K tokens at d = 256 (Gemma-like), ~40 % kept and frontier-only-like
    thresholds: mask parity away from T and output / LSE parity of sampled heads against the oracle
    replaying the GPU's decisions (the regime where K chunks stream while the MMAs run)."""
    n, d, hq, hkv = 16384, 256, 16, 8
    gen = torch.Generator(device="cuda").manual_seed(5 + int(T))
    q = torch.randn((1, hq, n, d), generator=gen, device="cuda").to(torch.bfloat16)
    k = torch.randn((1, hkv, n, d), generator=gen, device="cuda").to(torch.bfloat16)
    v = torch.randn((1, hkv, n, d), generator=gen, device="cuda").to(torch.bfloat16)
    t = bsfa.ThresholdTensor(values=np.full((1, 1, hq, n // 128), T, dtype=np.float32), k_levels=(1,),
                             n_max=n, b_m=128, b_n=64)
    res = bsfa.attention(q, k, v, thresholds=t, k_level=1, return_trace=True)
    for h in (0, 13):
        qh, kh, vh = (x[0, hh].float().cpu().numpy() for x, hh in ((q, h), (k, h // 2), (v, h // 2)))
        dec = res.decisions[0, h].cpu().numpy()
        rec = {}
        o_ref, lse_ref, _ = orc.flash_forward_fast(qh, kh, vh, True, 128, 64,
                                                   lambda i_idx, j, sm: dec[i_idx, j] == orc.KEPT, record=rec)
        for j, (i_idx, smax) in rec.items():
            far = np.abs(smax - T) > EPS
            want = np.where(smax > T, orc.KEPT, orc.SKIPPED)
            assert (dec[i_idx[far], j] == want[far]).all(), (h, j)
        o_gpu = res.o[0, h].float().cpu().numpy()
        assert np.abs(o_gpu - o_ref).max() <= ATOL and _row_rel_err(o_gpu, o_ref) <= ROW_RTOL
        assert _lse_err(res.lse[0, h].cpu().numpy(), lse_ref) <= LSE_ATOL
