"""BASELINE configs[2] and configs[4] as GPU tests.

configs[2]: Llama-3.1-8B shape (32 q / 8 kv heads, d=128) at 64K, thresholds
calibrated on the GPU from synthetic samples for ~30/50/70 % block skip, gated
on held-out samples: measured density tracks the predicted one (reference
acceptance 7, test_acceptance.py:170-195, bound 0.08) and one head is checked
against the CPU oracle (mask exactly outside |s_max - T| <= EPS, output and LSE
with the replayed mask).

configs[4]: the calibration pass over all 32 layers x 32 heads on synthetic
32K model-dump samples (structured and random heads, workloads.py:185-216),
then per layer dense vs BSFA on a held-out sample, with sampled (layer, head)
pairs -- one structured, one random -- checked against the oracle's
calibrate() (calibration.py:156-222) and forward (engine.py:117-193).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import record_metric  # noqa: E402
from oracle import bsfa_oracle as orc  # noqa: E402
from test_gpu_parity import ATOL, EPS, LSE_ATOL, ROW_RTOL, _lse_err, _row_rel_err  # noqa: E402

pytestmark = pytest.mark.gpu

HQ, HKV, D = 32, 8, 128


@pytest.fixture(scope="module")
def bsfa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_07011_b200 as m
    return m


def _mask_mismatches(dec, grid, T_row):
    """Gated tiles whose GPU decision disagrees with s_max > T away from the EPS band."""
    gated = np.isfinite(grid)
    T = T_row[np.minimum(np.arange(grid.shape[0]), len(T_row) - 1)][:, None]
    far = gated & (np.abs(grid - T) > EPS)
    want = np.where(grid > T, orc.KEPT, orc.SKIPPED)
    return int(np.count_nonzero(dec[far] != want[far])), int(np.count_nonzero(gated & ~far))


def test_config2_64k_calibrated_sweep(bsfa):
    from paper_2512_07011_b200 import costs
    from paper_2512_07011_b200.workloads import model_dump_layer

    n = 65536
    tiles = bsfa.TileConfig(128, 64)
    levels = sorted(costs.k_for_density(n, tiles, x) for x in (0.7, 0.5, 0.3))
    assert levels == [166, 299, 462]
    cal = bsfa.Calibrator(levels, tiles, 1, HQ, n, D)
    for s in range(4):
        q, k = model_dump_layer(s, 0, HQ, HKV, n, D, with_v=False)
        cal.add_layer(s, 0, q, k)
    thr = cal.finish()
    kept, reach = {kk: 0 for kk in levels}, {kk: 0 for kk in levels}
    held = [16, 17]
    for s in held:
        q, k, v = (x[None] for x in model_dump_layer(s, 0, HQ, HKV, n, D))
        for kk in levels:
            c = bsfa.attention(q, k, v, thresholds=thr, k_level=kk, tiles=tiles).counters.cpu().numpy()
            kept[kk] += int(c[1])
            reach[kk] += int(c[0])
    for kk in levels:
        measured, pred = kept[kk] / reach[kk], costs.predicted_density(n, tiles, kk)
        record_metric(f"config2_k{kk}_density_abs_diff", abs(measured - pred))
        assert abs(measured - pred) <= 0.08, (kk, measured, pred)

    # oracle: one structured head (kv group 0 of layer 0) of the first held-out sample, every level
    q, k, v = model_dump_layer(held[0], 0, HQ, HKV, n, D)
    h = 1
    qh, kh, vh = (x[c].float().cpu().numpy() for x, c in ((q, h), (k, 0), (v, 0)))
    grid = orc.tile_maxima_grid(qh, kh, 128, 64)
    for kk in levels:
        res = bsfa.attention(q[None], k[None], v[None], thresholds=thr, k_level=kk, tiles=tiles,
                             return_trace=True)
        dec = res.decisions[0, h].cpu().numpy()
        bad, band = _mask_mismatches(dec, grid, thr.values[levels.index(kk), 0, h])
        assert bad == 0, (kk, bad, band)
        if kk == 299:
            o_ref, lse_ref, _ = orc.flash_forward_fast(qh, kh, vh, True, 128, 64,
                                                       lambda i_idx, j, sm: dec[i_idx, j] == orc.KEPT)
            o_gpu = res.o[0, h].float().cpu().numpy()
            rel = _row_rel_err(o_gpu, o_ref)
            lerr = _lse_err(res.lse[0, h].cpu().numpy(), lse_ref)
            record_metric("config2_row_rel", rel)
            record_metric("config2_lse_abs", lerr)
            assert np.abs(o_gpu - o_ref).max() <= ATOL
            assert rel <= ROW_RTOL and lerr <= LSE_ATOL, (rel, lerr)


def test_config4_calibration_pass_and_parity_sweep(bsfa):
    from paper_2512_07011_b200 import costs
    from paper_2512_07011_b200.workloads import model_dump_layer

    n, L, samples = 32768, 32, 2
    tiles = bsfa.TileConfig(128, 64)
    levels = sorted(costs.k_for_density(n, tiles, x) for x in (0.7, 0.5, 0.3))
    k50 = costs.k_for_density(n, tiles, 0.5)
    cal = bsfa.Calibrator(levels, tiles, L, HQ, n, D)
    for s in range(samples):
        for layer in range(L):
            q, k = model_dump_layer(s, layer, HQ, HKV, n, D, with_v=False)
            cal.add_layer(s, layer, q, k)
    thr = cal.finish()
    assert thr.values.shape == (3, L, HQ, n // 128)

    # held-out sweep over every layer: dense and BSFA, density tracking per layer
    eval_sample = 1000
    dens = []
    for layer in range(L):
        q, k, v = (x[None] for x in model_dump_layer(eval_sample, layer, HQ, HKV, n, D))
        rb = bsfa.attention(q, k, v, thresholds=thr, layer=layer, k_level=k50, tiles=tiles)
        rd = bsfa.attention(q, k, v, tiles=tiles)
        c = rb.counters.cpu().numpy()
        dens.append(c[1] / c[0])
        assert int(rd.counters[1]) == int(rd.counters[0])  # dense keeps every reachable tile
        assert int(rb.status[0]) == 0 and int(rd.status[0]) == 0
    pred = costs.predicted_density(n, tiles, k50)
    record_metric("config4_density_abs_diff_mean", abs(float(np.mean(dens)) - pred))
    record_metric("config4_density_abs_diff_worst_layer", float(np.max(np.abs(np.array(dens) - pred))))
    assert abs(float(np.mean(dens)) - pred) <= 0.08
    assert float(np.max(np.abs(np.array(dens) - pred))) <= 0.08

    # oracle spot checks: (layer, head) with a structured kv group (layer*Hkv + g even) and a random one
    for layer, h in ((6, 9), (6, 13)):
        g = h // (HQ // HKV)
        structured = (layer * HKV + g) % 2 == 0
        cal_samples = []
        for s in range(samples):
            q, k = model_dump_layer(s, layer, HQ, HKV, n, D, with_v=False)
            cal_samples.append((s, q[h].float().cpu().numpy()[None, None], k[g].float().cpu().numpy()[None, None]))
        ref_vals, _, ref_ties = orc.calibrate(cal_samples, levels, 128, 64)
        gpu_vals = thr.values[:, layer, h]
        fin = np.isfinite(ref_vals[:, 0, 0])
        np.testing.assert_array_equal(np.isfinite(gpu_vals), fin)
        np.testing.assert_array_equal(gpu_vals[~fin], ref_vals[:, 0, 0][~fin])
        terr = float(np.abs(gpu_vals[fin] - ref_vals[:, 0, 0][fin]).max())
        record_metric(f"config4_threshold_abs_{'structured' if structured else 'random'}", terr)
        assert terr <= 1e-4

        q, k, v = model_dump_layer(eval_sample, layer, HQ, HKV, n, D)
        qh, kh, vh = (x[c].float().cpu().numpy() for x, c in ((q, h), (k, g), (v, g)))
        rb = bsfa.attention(q[None], k[None], v[None], thresholds=thr, layer=layer, k_level=k50, tiles=tiles,
                            return_trace=True)
        rd = bsfa.attention(q[None], k[None], v[None], tiles=tiles)
        dec = rb.decisions[0, h].cpu().numpy()
        bad, band = _mask_mismatches(dec, orc.tile_maxima_grid(qh, kh, 128, 64), thr.values[levels.index(k50), layer, h])
        assert bad == 0, (layer, h, bad, band)
        for name, r, keep in (("bsfa", rb, lambda i_idx, j, sm: dec[i_idx, j] == orc.KEPT),
                              ("dense", rd, lambda i_idx, j, sm: np.ones(len(i_idx), bool))):
            o_ref, lse_ref, _ = orc.flash_forward_fast(qh, kh, vh, True, 128, 64, keep)
            o_gpu = r.o[0, h].float().cpu().numpy()
            rel = _row_rel_err(o_gpu, o_ref)
            lerr = _lse_err(r.lse[0, h].cpu().numpy(), lse_ref)
            kind = "structured" if structured else "random"
            record_metric(f"config4_{name}_{kind}_row_rel", rel)
            record_metric(f"config4_{name}_{kind}_lse_abs", lerr)
            assert np.abs(o_gpu - o_ref).max() <= ATOL, (name, layer, h)
            assert rel <= ROW_RTOL and lerr <= LSE_ATOL, (name, layer, h, rel, lerr)
