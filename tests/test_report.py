"""Trace npz and report schema 1 in the reference formats (cli.py:36-101, costs.py:78-95)."""
import importlib
import json
import os
import sys

import numpy as np
import pytest

from paper_2512_07011_b200 import FormatError, TileConfig
from paper_2512_07011_b200.report import (load_report, load_traces, measured_density, save_traces,
                                          traces_from_decisions, write_report)

REF_SRC = "/root/reference/pkg/src"


def _decisions(rng, h=3, m_q=4, m_kv=8):
    dec = np.zeros((1, h, m_q, m_kv), dtype=np.int8)
    for i in range(m_q):
        dec[0, :, i, :2 * i] = rng.choice([1, 3], size=(h, 2 * i))
        dec[0, :, i, 2 * i:2 * i + 2] = 2
    return dec


def test_trace_round_trip_and_density(tmp_path):
    rng = np.random.default_rng(0)
    tiles = TileConfig(128, 64)
    s0 = traces_from_decisions(_decisions(rng), tiles, layer=2, head_offset=4)
    s1 = traces_from_decisions(_decisions(rng), tiles, layer=2, head_offset=4)
    path = tmp_path / "t.npz"
    save_traces(path, [s0, s1], tiles, causal=True)
    with np.load(path) as z:
        meta = json.loads(bytes(z["meta"]))
        assert meta == {"bm": 128, "bn": 64, "causal": True, "samples": 2}
        assert sorted(n for n in z.files if n != "meta") == sorted(
            f"s{s}_l2_h{h}" for s in range(2) for h in (4, 5, 6))
    back = load_traces(path)
    assert [[(t.layer, t.head) for t in s] for s in back] == [[(2, 4), (2, 5), (2, 6)]] * 2
    for a, b in zip(s0, back[0]):
        assert np.array_equal(a.decisions, b.decisions)
    mean, std = measured_density([s0, s1])
    fr = [sum(t.kept_blocks() for t in s) / sum(t.reachable_blocks() for t in s) for s in (s0, s1)]
    assert mean == pytest.approx(np.mean(fr)) and std == pytest.approx(np.std(fr))


def test_report_schema(tmp_path):
    cfg = {"n": 1024, "d": 64, "layers": 1, "heads": 1, "bm": 128, "bn": 64, "gate": "threshold",
           "params": {"k": 4}}
    path = tmp_path / "r.json"
    write_report(path, cfg, {"mean_ms": 1.0, "std_ms": 0.1, "repeats": 3},
                 {"qk_flops": 1, "pv_flops": 1, "softmax_ops": 1, "v_traffic": 1, "k_traffic": 1,
                  "gate_overhead_ops": 1}, {"predicted": 0.5, "measured_mean": 0.5, "measured_std": 0.0}, None)
    r = load_report(path)
    assert r["schema"] == 1 and r["config"]["gate"] == "threshold"
    bad = json.loads(path.read_text())
    bad["timing"]["gpu_ms"] = 1.0
    path.write_text(json.dumps(bad))
    with pytest.raises(FormatError):
        load_report(path)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not mounted (GPU box)")
def test_reference_tooling_reads_gpu_traces(tmp_path):
    """The reference's own load_traces / measured_density consume our files."""
    sys.path.insert(0, REF_SRC)
    try:
        cli = importlib.import_module("bsfa.cli")
        costs = importlib.import_module("bsfa.costs")
    finally:
        sys.path.remove(REF_SRC)
    rng = np.random.default_rng(1)
    tiles = TileConfig(128, 64)
    ours = [traces_from_decisions(_decisions(rng), tiles), traces_from_decisions(_decisions(rng), tiles)]
    path = tmp_path / "t.npz"
    save_traces(path, ours, tiles, causal=True)
    theirs = cli.load_traces(path)
    assert costs.measured_density(theirs) == pytest.approx(measured_density(ours))
