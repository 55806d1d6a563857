"""Trace files and run reports in the reference formats, from GPU runs.

* ``save_traces`` / ``load_traces``: the reference's npz trace container
  (pkg/src/bsfa/cli.py:76-101) -- a ``meta`` JSON blob (bm, bn, causal,
  samples) plus one int8 decision grid per ``s{sample}_l{layer}_h{head}`` --
  so the reference ``density --trace`` tooling reads GPU traces unchanged.
* ``traces_from_decisions``: the kernel's ``decisions`` output
  ([B, Hq, M_q, M_kv] int8, codes 0..3) as per-head :class:`GateTrace` objects.
* ``measured_density``: per-sample pooled retained fraction, mean and
  population std (costs.py:78-95).
* ``write_report`` / ``load_report``: run report schema 1 (cli.py:36-73) with
  the same key sets and the same unknown-field rejection.
"""

from __future__ import annotations

import json
from datetime import datetime, timezone

import numpy as np

from .errors import FormatError, InvalidInputError
from .tiling import TileConfig
from .trace import GateTrace

REPORT_KEYS = {
    None: {"schema", "config", "timing", "cost", "density", "verify"},
    "config": {"n", "d", "layers", "heads", "bm", "bn", "gate", "params"},
    "timing": {"mean_ms", "std_ms", "repeats"},
    "cost": {"qk_flops", "pv_flops", "softmax_ops", "v_traffic", "k_traffic", "gate_overhead_ops"},
    "density": {"predicted", "measured_mean", "measured_std"},
    "verify": {"max_rel_err", "rtol", "pass"},
}


def traces_from_decisions(decisions, tiles: TileConfig, causal: bool = True, layer: int = 0,
                          head_offset: int = 0, batch_index: int = 0) -> list[GateTrace]:
    """One GateTrace per q head of a kernel decision tensor ([B, Hq, M_q, M_kv] or [Hq, M_q, M_kv])."""
    if hasattr(decisions, "detach"):
        decisions = decisions.detach().cpu().numpy()
    dec = np.asarray(decisions)
    if dec.ndim == 4:
        dec = dec[batch_index]
    if dec.ndim != 3:
        raise InvalidInputError(f"decisions must be [B, H, M_q, M_kv] or [H, M_q, M_kv], got {dec.shape}")
    return [GateTrace(decisions=np.ascontiguousarray(dec[h], dtype=np.int8), tiles=tiles, causal=causal,
                      layer=layer, head=head_offset + h) for h in range(dec.shape[0])]


def save_traces(path, traces_by_sample, tiles: TileConfig, causal: bool) -> None:
    arrays = {"meta": np.frombuffer(json.dumps(
        {"bm": tiles.b_m, "bn": tiles.b_n, "causal": causal, "samples": len(traces_by_sample)}).encode(),
        dtype=np.uint8)}
    for si, traces in enumerate(traces_by_sample):
        for t in traces:
            arrays[f"s{si}_l{t.layer}_h{t.head}"] = t.decisions
    np.savez(path, **arrays)


def load_traces(path):
    with np.load(path) as data:
        meta = json.loads(bytes(data["meta"]))
        tiles = TileConfig(meta["bm"], meta["bn"])
        by_sample = [[] for _ in range(meta["samples"])]
        for name in data.files:
            if name == "meta":
                continue
            si, layer, head = (int(part[1:]) for part in name.split("_"))
            by_sample[si].append(GateTrace(decisions=data[name], tiles=tiles, causal=meta["causal"],
                                           layer=layer, head=head))
    return by_sample


def measured_density(traces_by_sample) -> tuple[float, float]:
    fractions = []
    for traces in traces_by_sample:
        traces = list(traces)
        if not traces:
            continue
        kept = sum(t.kept_blocks() for t in traces)
        reachable = sum(t.reachable_blocks() for t in traces)
        fractions.append(kept / reachable)
    if not fractions:
        raise InvalidInputError("no traces to measure density from")
    arr = np.asarray(fractions)
    return float(arr.mean()), float(arr.std())


def write_report(path, config: dict, timing: dict, cost: dict, density: dict, verify: dict | None) -> dict:
    report = {"schema": 1, "timestamp": datetime.now(timezone.utc).isoformat(), "config": config,
              "timing": timing, "cost": cost, "density": density, "verify": verify}
    _check_keys(report, path)
    with open(path, "w", encoding="utf-8") as f:
        json.dump(report, f, indent=2)
        f.write("\n")
    return report


def load_report(path) -> dict:
    with open(path, "r", encoding="utf-8") as f:
        report = json.load(f)
    if report.get("schema") != 1:
        raise FormatError(f"{path}: unsupported report schema {report.get('schema')!r}")
    _check_keys(report, path)
    return report


def _check_keys(report: dict, path) -> None:
    for section, keys in REPORT_KEYS.items():
        obj = report if section is None else report.get(section)
        if obj is None:
            continue
        extra = set(obj) - keys - ({"timestamp"} if section is None else set())
        if extra:
            raise FormatError(f"{path}: unknown report fields {sorted(extra)}")
