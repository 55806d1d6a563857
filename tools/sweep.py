"""Sparsity / sequence-length sweep of the BSFA forward on one B200 (BASELINE configs 2-4).

    python tools/sweep.py [--seqs 32768 65536 131072] [--densities 0.3 0.5 0.7] [--steps 5]

For each sequence length: thresholds calibrated on a separate synthetic sample
(seed 1000) for each target predicted density (reference costs.predicted_density
inverted to a k level), then BSFA and the same kernel with the DenseGate timed
with CUDA events (inputs resident, 32 q / 8 kv heads, d=128, causal, 128x64
tiles).  One JSON line per (seq, density) plus one dense line per seq; each
speedup divides by a dense run timed right after the BSFA run (a first, cold
dense run is up to 10 % faster than later ones).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2512_07011_b200 as bsfa  # noqa: E402
from paper_2512_07011_b200 import costs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", type=int, nargs="+", default=[32768, 65536, 131072])
    ap.add_argument("--densities", type=float, nargs="+", default=[0.3, 0.5, 0.7])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    tiles = bsfa.TileConfig(128, 64)
    stream = torch.cuda.current_stream(dev)
    peak, _, src = bench.measured_peaks()
    for n in args.seqs:
        cfg = dict(heads_q=32, heads_kv=8, seq_len=n, head_dim=128)
        q, k, v = bench.make_inputs(cfg, 0, dev)
        dplan = bsfa.BsfaPlan(1, 32, 8, n, 128, tiles=tiles, device=dev)
        _, dtot = bench.time_steps(lambda: dplan.run(q, k, v), args.steps, args.warmup, stream)
        dms = dtot / args.steps
        cnt = dplan.counters.cpu().numpy()
        f_dense = costs.dense_flops(int(cnt[0]), tiles, 128)
        print(json.dumps({"seq_len": n, "gate": "dense", "ms": dms, "tflops": f_dense / dms / 1e9,
                          "frac_of_peak": f_dense / dms / 1e9 / peak, "peak_source": src}), flush=True)
        for dens in args.densities:
            kl = costs.k_for_density(n, tiles, dens)
            thr = bench.calibrated_thresholds(cfg, tiles, kl, dev)
            plan = bsfa.BsfaPlan(1, 32, 8, n, 128, tiles=tiles, thresholds=thr, k_level=kl, device=dev)
            _, tot = bench.time_steps(lambda: plan.run(q, k, v), args.steps, args.warmup, stream)
            ms = tot / args.steps
            # dense again right after, so the speedup pairs runs at the same thermal state
            _, dtot2 = bench.time_steps(lambda: dplan.run(q, k, v), args.steps, 1, stream)
            dms_pair = dtot2 / args.steps
            c = plan.counters.cpu().numpy()
            reach, kept, vl, vu = (int(x) for x in c)
            f_exec = costs.executed_flops(reach, kept, tiles, 128)
            print(json.dumps({"seq_len": n, "gate": "threshold", "k_level": kl, "predicted_density": dens,
                              "measured_density": kept / reach, "skip_frac": 1 - kept / reach,
                              "v_fetch_skip_frac": 1 - vl / vu, "ms": ms, "exec_tflops": f_exec / ms / 1e9,
                              "effective_dense_tflops": costs.dense_flops(reach, tiles, 128) / ms / 1e9,
                              "frac_of_peak": f_exec / ms / 1e9 / peak, "dense_ms_adjacent": dms_pair,
                              "speedup_vs_dense": dms_pair / ms}), flush=True)
            del plan, thr
        del dplan
        del q, k, v
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
