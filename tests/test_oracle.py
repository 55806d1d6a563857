"""Pins the CPU oracle to the reference: golden vectors + reference KATs (CPU only)."""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from oracle import bsfa_oracle as orc

ENGINE_CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "engine_*.npz")))


def _gate_for(case):
    kind = str(case["kind"])
    if kind == "dense":
        return orc.dense_gate
    if kind == "frontier":
        return orc.frontier_only_gate
    return orc.threshold_gate(case["thr"])


@pytest.mark.parametrize("name", ENGINE_CASES)
def test_engine_matches_reference_golden(name):
    c = load_golden(name)
    b_m, b_n, causal = int(c["b_m"]), int(c["b_n"]), bool(c["causal"])
    rec = {}
    o, lse, dec = orc.flash_forward(c["q"], c["k"], c["v"], causal, b_m, b_n, _gate_for(c), record=rec)
    np.testing.assert_array_equal(dec, c["decisions"])
    assert orc.max_rel_err(o, c["o"]) <= 1e-5
    assert orc.max_rel_err(lse, c["lse"]) <= 1e-5
    for (i, j), v in rec.items():
        want = c["smax"][i, j]
        if np.isnan(want):
            continue
        if np.isinf(want):
            assert v == want
        else:
            assert abs(v - want) <= 1e-5 * (1 + abs(v))


@pytest.mark.parametrize("name", ENGINE_CASES)
def test_fast_engine_matches_tile_engine(name):
    c = load_golden(name)
    b_m, b_n, causal = int(c["b_m"]), int(c["b_n"]), bool(c["causal"])
    kind = str(c["kind"])
    thr = c["thr"]

    def keep_fn(i_idx, j, smax):
        if kind == "dense":
            return np.ones(len(i_idx), dtype=bool)
        if kind == "frontier":
            return np.zeros(len(i_idx), dtype=bool)
        return smax > thr[np.minimum(i_idx, len(thr) - 1)]

    o, lse, dec = orc.flash_forward_fast(c["q"], c["k"], c["v"], causal, b_m, b_n, keep_fn)
    np.testing.assert_array_equal(dec, c["decisions"])
    assert orc.max_rel_err(o, c["o"]) <= 1e-5
    assert orc.max_rel_err(lse, c["lse"]) <= 1e-5


def test_toy_config_golden():
    c = load_golden("toy")
    q, k, v = orc.gen_random(1024, 64, seed=0)
    np.testing.assert_array_equal(q[:4], c["raw_q_head"])  # same seeded stream as workloads.py:58-77
    for key, gate in (("dense", orc.dense_gate), ("frontier", orc.frontier_only_gate),
                      ("thr", orc.threshold_gate(np.full(8, c["T"], dtype=np.float32)))):
        o, lse, dec = orc.flash_forward(c["q"], c["k"], c["v"], True, 128, 64, gate)
        np.testing.assert_array_equal(dec, c[f"dec_{key}"])
        assert orc.max_rel_err(o, c[f"o_{key}"]) <= 1e-5
    # the fixed threshold skips about half of the 56 gated tiles
    dec = c["dec_thr"]
    gated = np.count_nonzero(dec == orc.KEPT) + np.count_nonzero(dec == orc.SKIPPED)
    assert gated == 56
    assert 0.3 < np.count_nonzero(dec == orc.SKIPPED) / gated < 0.7


def test_dense_oracle_kats():
    # reference tests/test_core.py:10-31
    o, lse = orc.dense_attention(np.array([[1.0], [1.0]]), np.zeros((2, 1)), np.array([[1.0], [4.2]]))
    np.testing.assert_allclose(o, [[1.0], [2.6]])
    np.testing.assert_allclose(lse, [0.0, np.log(2.0)])
    o, lse = orc.dense_attention(np.array([[1.0, 2.0]]), np.array([[3.0, 4.0]]), np.array([[3.0, 7.0]]))
    np.testing.assert_allclose(o, [[3.0, 7.0]])
    np.testing.assert_allclose(lse, [11.0 / np.sqrt(2.0)])
    rng = np.random.default_rng(0)
    v = rng.standard_normal((4, 3)).astype(np.float32)
    o, _ = orc.dense_attention(np.zeros((4, 3)), rng.standard_normal((4, 3)), v)
    np.testing.assert_allclose(o, np.cumsum(v.astype(np.float64), axis=0) / np.arange(1, 5)[:, None], rtol=1e-6)


def test_engine_dense_vs_fp64_oracle():
    rng = np.random.default_rng(5)
    for n, causal in ((64, True), (257, False), (512, True)):
        q, k, v = (rng.standard_normal((n, 32)).astype(np.float32) for _ in range(3))
        o, lse, _ = orc.flash_forward(q, k, v, causal, 128, 64, orc.dense_gate)
        o64, lse64 = orc.dense_attention(q, k, v, causal)
        assert orc.max_rel_err(o, o64) <= 1e-4
        assert orc.max_rel_err(lse, lse64) <= 1e-4


def test_gated_engine_vs_masked_oracle():
    rng = np.random.default_rng(6)
    q, k, v = (rng.standard_normal((640, 32)).astype(np.float32) for _ in range(3))
    for gate in (orc.frontier_only_gate, orc.sliding_window_gate(200, 128, 64), orc.running_max_gate(0.3),
                 orc.threshold_gate(np.linspace(0.2, 1.0, 5))):
        o, _, dec = orc.flash_forward(q, k, v, True, 128, 64, gate)
        o64, _ = orc.masked_dense_attention(q, k, v, dec, 128, 64)
        assert orc.max_rel_err(o, o64) <= 1e-4


def test_calibration_matches_reference_golden():
    c = load_golden("calib")
    samples = [(i, c[f"q{i}"], c[f"k{i}"]) for i in (2, 0, 1)]  # order must not matter
    vals, n_max, ties = orc.calibrate(samples, c["k_levels"], 128, 64)
    assert n_max == int(c["n_max"])
    np.testing.assert_array_equal(vals, c["values"])
    assert [ties[int(k)] for k in c["k_levels"]] == list(c["ties"])
    prof = orc.block_maxima(c["q1"][0, 1], c["k1"][0, 1], 128, 64)
    for p, vals_p in enumerate(prof):
        np.testing.assert_allclose(vals_p, c["maxima_sample1"][0, 1, p, :len(vals_p)], rtol=1e-6)


def test_cutoff_kats():
    # reference tests/test_calibration.py:32-47
    vals = np.array([5.0, 4.0, 3.0, 2.0, 1.0], dtype=np.float32)
    assert orc.cutoff(vals, 2) == 3.0 and orc.cutoff(vals, 4) == 1.0
    assert orc.cutoff(vals, 0) == np.inf and orc.cutoff(vals, 5) == -np.inf
    tied = np.array([5.0, 5.0, 3.0], dtype=np.float32)
    assert orc.cutoff(tied, 1) == 5.0 and orc.is_tie(tied, 1) and not orc.is_tie(tied, 2)


def test_workload_stream_matches_reference():
    c = load_golden("workload")
    q, k, v = orc.gen_random(64, 8, seed=3, sample=1, layer=2, head=5)
    np.testing.assert_array_equal(q, c["q"])
    np.testing.assert_array_equal(k, c["k"])
    np.testing.assert_array_equal(v, c["v"])


def test_round_bf16():
    x = np.array([1.0, 1.00390625, 1.005859375, -3.14159, 1e-40, np.inf], dtype=np.float32)
    r = orc.round_bf16(x)
    assert r[0] == 1.0 and r[1] == 1.0  # tie to even
    assert r[2] == np.float32(1.0078125)
    assert np.isinf(r[5])
    np.testing.assert_array_equal(orc.round_bf16(r), r)


def test_tile_maxima_grid_matches_block_maxima():
    q, k, _ = orc.gen_random(1024, 64, seed=3)
    grid = orc.tile_maxima_grid(q, k, 128, 64)
    bm = orc.block_maxima(q, k, 128, 64)
    for p, vals in enumerate(bm):
        row = grid[p][np.isfinite(grid[p])]
        np.testing.assert_array_equal(np.sort(row)[::-1], vals)


def test_fast_oracle_query_block_subset():
    q, k, v = orc.gen_random(1024, 64, seed=4)
    full_o, full_l, full_d = orc.flash_forward_fast(q, k, v, True, 128, 64, lambda i, j, s: s > 3.9)
    sub_o, sub_l, sub_d = orc.flash_forward_fast(q, k, v, True, 128, 64, lambda i, j, s: s > 3.9, q_blocks=[5, 7])
    for i in (5, 7):
        rows = slice(i * 128, (i + 1) * 128)
        np.testing.assert_array_equal(sub_o[rows], full_o[rows])
        np.testing.assert_array_equal(sub_l[rows], full_l[rows])
        np.testing.assert_array_equal(sub_d[i], full_d[i])
    assert np.isnan(sub_o[:128]).all()
