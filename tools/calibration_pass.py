"""BASELINE configs[4]: threshold calibration over all 32 layers x 32 heads on
synthetic 32K sequences, then a dense (threshold = -inf) vs BSFA parity sweep.

    python tools/calibration_pass.py [--layers 32] [--seq 32768] [--samples 2] [--oracle-heads 2]

1. Calibration: model-dump-style synthetic layers generated on the GPU
   (paper_2512_07011_b200.workloads), streamed layer by layer through the
   calibration kernel (one launch per (sample, layer)) for k levels at
   predicted densities 0.3 / 0.5 / 0.7.  Timed with CUDA events.
2. Evaluation on a held-out sample: per layer, the DenseGate and the
   ThresholdGate at density 0.5 -- measured vs predicted density, time, and
   the (informational) max |O_bsfa - O_dense|.
3. Oracle spot checks (CPU, numpy port of the reference): for sampled
   (layer, head) pairs, the calibrated thresholds vs the oracle calibrate()
   on the same bf16 tensors, the dense output vs the fp32 oracle, and the
   BSFA decisions (exact outside |s_max - T| <= 1e-3) and output (replayed
   decisions, max-abs <= 2e-2).
Prints one JSON object per phase.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2512_07011_b200 as bsfa  # noqa: E402
from paper_2512_07011_b200 import costs  # noqa: E402
from paper_2512_07011_b200.report import measured_density, save_traces, traces_from_decisions, write_report  # noqa: E402
from paper_2512_07011_b200.workloads import model_dump_layer  # noqa: E402
from oracle import bsfa_oracle as orc  # noqa: E402

HQ, HKV, D = 32, 8, 128
EPS = 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--seq", type=int, default=32768)
    ap.add_argument("--samples", type=int, default=2)
    ap.add_argument("--oracle-heads", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3, help="interleaved (dense, BSFA) timing rounds per layer")
    ap.add_argument("--traces", default=None, help="write the evaluation decisions (reference npz trace format)")
    ap.add_argument("--report", default=None, help="write a reference schema-1 run report (JSON)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    n, L = args.seq, args.layers
    tiles = bsfa.TileConfig(128, 64)
    levels = sorted(costs.k_for_density(n, tiles, x) for x in (0.7, 0.5, 0.3))
    k50 = costs.k_for_density(n, tiles, 0.5)

    # ---- 1. calibration
    cal = bsfa.Calibrator(levels, tiles, L, HQ, n, D, device=dev)
    gen_ms = cal_ms = 0.0
    for s in range(args.samples):
        for layer in range(L):
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
            q, k = model_dump_layer(s, layer, HQ, HKV, n, D, device=dev, with_v=False)
            e1.record()
            cal.add_layer(s, layer, q, k)
            e2.record()
            torch.cuda.synchronize()
            gen_ms += e0.elapsed_time(e1)
            cal_ms += e1.elapsed_time(e2)
    thr = cal.finish()
    qk_flops = 0
    for p_ in range(n // 128):
        qk_flops += 2 * 128 * 64 * D * orc.off_frontier(p_, 128, 64)
    qk_flops *= HQ * L * args.samples
    print(json.dumps({"phase": "calibration", "layers": L, "heads_q": HQ, "heads_kv": HKV, "seq_len": n,
                      "samples": args.samples, "k_levels": levels, "calib_kernel_ms": cal_ms,
                      "generator_ms": gen_ms, "qk_tflop": qk_flops / 1e12,
                      "calib_tflops": qk_flops / cal_ms / 1e9,
                      "tie_counts": {str(k): int(v) for k, v in thr.diagnostics.tie_counts.items()}}),
          flush=True)

    # ---- 2. held-out evaluation, dense vs BSFA per layer.  Timing: device-only
    # launches through BsfaPlan (same kernels attention() runs), --reps rounds
    # of (dense, BSFA) interleaved after one warm-up pair, medians per layer.
    rows = []
    eval_sample = 1000
    traces = []
    plan_d = bsfa.BsfaPlan(1, HQ, HKV, n, D, tiles=tiles, device=dev)
    for layer in range(L):
        q, k, v = model_dump_layer(eval_sample, layer, HQ, HKV, n, D, device=dev)
        q, k, v = q[None], k[None], v[None]
        rd = bsfa.attention(q, k, v, tiles=tiles)
        rb = bsfa.attention(q, k, v, thresholds=thr, layer=layer, k_level=k50, tiles=tiles,
                            return_trace=args.traces is not None or args.report is not None)
        plan_b = bsfa.BsfaPlan(1, HQ, HKV, n, D, tiles=tiles, device=dev, thresholds=thr, layer=layer,
                               k_level=k50)
        td, tb = [], []
        for r in range(args.reps + 1):
            for plan, acc in ((plan_d, td), (plan_b, tb)):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                plan.run(q, k, v)
                e1.record()
                torch.cuda.synchronize()
                if r:
                    acc.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        c = rb.counters.cpu().numpy()
        dev_max = float((rb.o.float() - rd.o.float()).abs().max())
        if rb.decisions is not None:
            traces.extend(traces_from_decisions(rb.decisions, tiles, causal=True, layer=layer))
        rows.append({"layer": layer, "density": float(c[1] / c[0]), "v_fetch_frac": float(c[2] / c[3]),
                     "dense_ms": float(np.median(td)), "bsfa_ms": float(np.median(tb)),
                     "max_abs_bsfa_vs_dense": dev_max})
    dens = np.array([r["density"] for r in rows])
    print(json.dumps({"phase": "evaluation", "k_level": k50,
                      "predicted_density": costs.predicted_density(n, tiles, k50),
                      "measured_density_mean": float(dens.mean()), "measured_density_std": float(dens.std()),
                      "v_fetch_frac_mean": float(np.mean([r["v_fetch_frac"] for r in rows])),
                      "dense_ms_total": sum(r["dense_ms"] for r in rows),
                      "bsfa_ms_total": sum(r["bsfa_ms"] for r in rows),
                      "speedup": sum(r["dense_ms"] for r in rows) / sum(r["bsfa_ms"] for r in rows),
                      "per_layer": rows}), flush=True)

    if args.traces:
        save_traces(args.traces, [traces], tiles, causal=True)
    if args.report:
        mean, std = measured_density([traces])
        bsfa_ms = np.array([r["bsfa_ms"] for r in rows])
        cc = costs.tile_counts(n, tiles)
        per_tile = 2 * 128 * 64 * D
        write_report(args.report,
                     {"n": n, "d": D, "layers": L, "heads": HQ, "bm": 128, "bn": 64, "gate": "threshold",
                      "params": {"k": k50, "device": "B200 sm_100a", "heads_kv": HKV}},
                     {"mean_ms": float(bsfa_ms.mean()), "std_ms": float(bsfa_ms.std()), "repeats": L},
                     {"qk_flops": per_tile * cc[0] * HQ, "pv_flops": per_tile * cc[0] * mean * HQ,
                      "softmax_ops": 128 * 64 * cc[0] * mean * HQ, "v_traffic": 64 * D * cc[0] * mean * HQ,
                      "k_traffic": 64 * D * cc[0] * HQ, "gate_overhead_ops": (128 * 64 + 1) * (cc[0] - cc[1]) * HQ},
                     {"predicted": costs.predicted_density(n, tiles, k50), "measured_mean": mean,
                      "measured_std": std}, None)

    # ---- 3. oracle spot checks on sampled (layer, head)
    rng = np.random.default_rng(7)
    picks = [(int(rng.integers(L)), int(rng.integers(HQ))) for _ in range(args.oracle_heads)]
    checks = []
    for layer, h in picks:
        g = h // (HQ // HKV)
        # thresholds: oracle calibrate over the same bf16 calibration tensors of this head
        samples = []
        for s in range(args.samples):
            q, k = model_dump_layer(s, layer, HQ, HKV, n, D, device=dev, with_v=False)
            samples.append((s, q[h].float().cpu().numpy()[None, None], k[g].float().cpu().numpy()[None, None]))
        t0 = time.perf_counter()
        vals, _, _ = orc.calibrate(samples, [k50], 128, 64)
        t_cal = time.perf_counter() - t0
        gpu = thr.values[levels.index(k50), layer, h]
        ref = vals[0, 0, 0]
        both = np.isfinite(gpu) & np.isfinite(ref)
        thr_err = float(np.abs(gpu[both] - ref[both]).max()) if both.any() else 0.0
        sentinel_ok = bool(np.array_equal(np.isfinite(gpu), np.isfinite(ref)))
        # dense and BSFA on the held-out sample
        q, k, v = model_dump_layer(eval_sample, layer, HQ, HKV, n, D, device=dev)
        qh, kh, vh = (x.float().cpu().numpy() for x in (q[h], k[g], v[g]))
        rd = bsfa.attention(q[None], k[None], v[None], tiles=tiles)
        rb = bsfa.attention(q[None], k[None], v[None], thresholds=thr, layer=layer, k_level=k50, tiles=tiles,
                            return_trace=True)
        t0 = time.perf_counter()
        o_dense, _, _ = orc.flash_forward_fast(qh, kh, vh, True, 128, 64, lambda i, j, sm: True)
        dec = rb.decisions[0, h].cpu().numpy()
        rec = {}
        o_bsfa, _, _ = orc.flash_forward_fast(qh, kh, vh, True, 128, 64,
                                              lambda i, j, sm: dec[i, j] == orc.KEPT, record=rec)
        t_orc = time.perf_counter() - t0
        T = thr.values[levels.index(k50), layer, h]
        mism = 0
        band = 0
        gated = 0
        for j, (idx, smax) in rec.items():
            tb = T[np.minimum(idx, len(T) - 1)]
            want = smax > tb
            got = dec[idx, j] == orc.KEPT
            near = np.abs(smax - tb) <= EPS
            band += int(near.sum())
            mism += int(((want != got) & ~near).sum())
            gated += idx.size
        checks.append({"layer": layer, "head": h, "threshold_max_abs_err": thr_err, "sentinels_match": sentinel_ok,
                       "dense_max_abs": float(np.abs(rd.o[0, h].float().cpu().numpy() - o_dense).max()),
                       "bsfa_max_abs": float(np.abs(rb.o[0, h].float().cpu().numpy() - o_bsfa).max()),
                       "decision_mismatches_outside_eps": mism, "decisions_in_eps_band": band,
                       "gated_tiles": gated, "oracle_calibrate_s": t_cal, "oracle_forward_s": t_orc})
    ok = all(c["decision_mismatches_outside_eps"] == 0 and c["dense_max_abs"] <= 2e-2 and c["bsfa_max_abs"] <= 2e-2
             and c["sentinels_match"] for c in checks)
    print(json.dumps({"phase": "oracle_checks", "ok": ok, "checks": checks}), flush=True)


if __name__ == "__main__":
    main()
