"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference ``bsfa`` package from /root/reference/pkg/src,
feeds it seeded inputs (rounded to bf16-representable float32 so the same
fixtures also drive GPU parity) and stores inputs + reference outputs as
small .npz files next to this script.  The fixtures are committed; nothing
at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(HERE, "..", ".."))

import bsfa  # noqa: E402  (the reference)
from bsfa import (CalibrationDump, CalibrationSample, GateContext, HeadInput,  # noqa: E402
                  ThresholdTensor, TileConfig, WorkloadSpec, calibrate, collect_block_maxima,
                  flash_forward, save_thresholds)
from bsfa.gates import dense_gate, frontier_only_gate, threshold_gate  # noqa: E402
from bsfa.workloads import gen_random  # noqa: E402

from oracle.bsfa_oracle import round_bf16  # noqa: E402


class RecordingThreshold:
    """Reference-protocol gate: ThresholdGate that also records tile maxima."""

    def __init__(self, tensor):
        self.inner = threshold_gate(tensor)
        self.smax = {}

    def validate(self, tiles, ctx):
        self.inner.validate(tiles, ctx)

    def decide(self, tile, i, j, stats, ctx, tiles):
        self.smax[(i, j)] = tile.s_max
        return self.inner.decide(tile, i, j, stats, ctx, tiles)


def _bf16_head(rng, n, d, causal=True):
    return HeadInput(q=round_bf16(rng.standard_normal((n, d)).astype(np.float32)),
                     k=round_bf16(rng.standard_normal((n, d)).astype(np.float32)),
                     v=round_bf16(rng.standard_normal((n, d)).astype(np.float32)), causal=causal)


def engine_cases():
    cases = []
    rng = np.random.default_rng(20260101)
    # (n, d, causal, b_m, b_n, gate kind)
    specs = [
        (256, 64, True, 128, 64, "dense"), (256, 64, True, 128, 64, "frontier"),
        (512, 64, True, 128, 64, "threshold"), (130, 64, True, 128, 64, "threshold"),
        (257, 128, True, 128, 64, "threshold"), (384, 128, True, 128, 128, "threshold"),
        (300, 64, False, 128, 64, "threshold"), (200, 64, False, 128, 128, "dense"),
        (512, 32, True, 128, 64, "threshold"), (192, 16, True, 64, 64, "threshold"),
        (640, 64, True, 128, 64, "frontier"), (512, 64, False, 128, 64, "frontier"),
    ]
    for idx, (n, d, causal, b_m, b_n, kind) in enumerate(specs):
        inp = _bf16_head(rng, n, d, causal)
        tiles = TileConfig(b_m, b_n)
        p = tiles.padded_len(n) // b_m
        thr = rng.uniform(0.0, 1.2, size=(1, 1, 1, p)).astype(np.float32)
        tensor = ThresholdTensor(values=thr, k_levels=(4,), n_max=tiles.padded_len(n), b_m=b_m, b_n=b_n)
        if kind == "dense":
            gate, ctx = dense_gate(), GateContext()
        elif kind == "frontier":
            gate, ctx = frontier_only_gate(), GateContext()
        else:
            gate, ctx = RecordingThreshold(tensor), GateContext(k_level=4)
        out, trace = flash_forward(inp, tiles, gate, ctx)
        smax = np.full(trace.decisions.shape, np.nan, dtype=np.float64)
        if kind == "threshold":
            for (i, j), v in gate.smax.items():
                smax[i, j] = v
        cases.append(dict(name=f"engine_{idx:02d}", q=inp.q, k=inp.k, v=inp.v, causal=causal, b_m=b_m,
                          b_n=b_n, kind=kind, thr=thr[0, 0, 0], o=out.o, lse=out.logsumexp,
                          decisions=trace.decisions, smax=smax))
    return cases


def toy_case():
    """BASELINE configs[0]: B=1 H=1 N=1024 d=64 gen_random seed 0, causal, 128x64, fixed T."""
    inp = gen_random(WorkloadSpec(n=1024, d=64, seed=0))
    raw_q = inp.q.copy()
    inp = HeadInput(round_bf16(inp.q), round_bf16(inp.k), round_bf16(inp.v), causal=True)
    tiles = TileConfig(128, 64)
    out = {}
    for T in (3.94,):
        tensor = ThresholdTensor(values=np.full((1, 1, 1, 8), T, dtype=np.float32), k_levels=(1,),
                                 n_max=1024, b_m=128, b_n=64)
        g = RecordingThreshold(tensor)
        o, tr = flash_forward(inp, tiles, g, GateContext(k_level=1))
        smax = np.full(tr.decisions.shape, np.nan)
        for (i, j), v in g.smax.items():
            smax[i, j] = v
        out.update(o_thr=o.o, lse_thr=o.logsumexp, dec_thr=tr.decisions, smax=smax)
    od, trd = flash_forward(inp, tiles, dense_gate())
    of, trf = flash_forward(inp, tiles, frontier_only_gate())
    return dict(name="toy", q=inp.q, k=inp.k, v=inp.v, raw_q_head=raw_q[:4], T=np.float32(3.94),
                o_dense=od.o, lse_dense=od.logsumexp, dec_dense=trd.decisions,
                o_frontier=of.o, lse_frontier=of.logsumexp, dec_frontier=trf.decisions, **out)


def calibration_case():
    rng = np.random.default_rng(77)
    tiles = TileConfig(128, 64)
    samples = []
    for sid, n in ((0, 512), (1, 1024), (2, 768)):
        q = round_bf16(rng.standard_normal((1, 2, n, 64)).astype(np.float32))
        k = round_bf16(rng.standard_normal((1, 2, n, 64)).astype(np.float32))
        samples.append(CalibrationSample(sample_id=sid, q=q, k=k))
    dump = CalibrationDump(1, 2, 64, samples)
    k_levels = [0, 1, 3, 6, 99]
    t = calibrate(dump, k_levels, tiles)
    prof = collect_block_maxima(samples[1], tiles)
    flat = np.full((1, 2, 8, 16), np.nan, dtype=np.float32)
    for (l, h, p), vals in prof.maxima.items():
        flat[l, h, p, :len(vals)] = vals
    path = os.path.join(HERE, "_tmp_thr.bin")
    save_thresholds(t, path)
    blob = np.frombuffer(open(path, "rb").read(), dtype=np.uint8).copy()
    os.remove(path)
    out = dict(name="calib", k_levels=np.array(k_levels), values=t.values, n_max=t.n_max,
               ties=np.array([t.diagnostics.tie_counts[k] for k in k_levels]), maxima_sample1=flat,
               file_bytes=blob)
    for s in samples:
        out[f"q{s.sample_id}"] = s.q
        out[f"k{s.sample_id}"] = s.k
    return out


def workload_case():
    inp = gen_random(WorkloadSpec(n=64, d=8, seed=3), sample=1, layer=2, head=5)
    return dict(name="workload", q=inp.q, k=inp.k, v=inp.v)


def main():
    for case in engine_cases() + [toy_case(), calibration_case(), workload_case()]:
        name = case.pop("name")
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **case)
        print("wrote", name)
    print("reference version", bsfa.__version__)


if __name__ == "__main__":
    main()
