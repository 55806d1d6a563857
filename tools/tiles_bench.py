"""Forward time per reference tiling at one attention shape (1 GPU).

    python tools/tiles_bench.py [--seq 32768] [--density 0.5] [--rounds 4]
                                [--heads-q 32 --heads-kv 8 --head-dim 128]

For each tiling b_m x b_n in {128, 64} x {64, 128}: thresholds calibrated on
the GPU on a separate sample for the predicted density, then BSFA and the same
kernel with the DenseGate timed interleaved (rounds x 3 launches each, medians).
Prints one JSON line per tiling: ms, executed TFLOP/s from the kernel's own
counters (F_exec = 2 b_m b_n d (R + K), costs.py), measured density, speedup.
"""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2512_07011_b200 as bsfa  # noqa: E402
from paper_2512_07011_b200 import costs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=32768)
ap.add_argument("--density", type=float, default=0.5)
ap.add_argument("--rounds", type=int, default=4)
ap.add_argument("--tiles", nargs="+", default=["128x64", "128x128", "64x64", "64x128"])
ap.add_argument("--heads-q", type=int, default=32)
ap.add_argument("--heads-kv", type=int, default=8)
ap.add_argument("--head-dim", type=int, default=128)
ap.add_argument("--non-causal", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
cfg = dict(heads_q=a.heads_q, heads_kv=a.heads_kv, seq_len=a.seq, head_dim=a.head_dim)
q, k, v = bench.make_inputs(cfg, 0, dev)
stream = torch.cuda.current_stream(dev)
for spec in a.tiles:
    bm, bn = (int(x) for x in spec.split("x"))
    tiles = bsfa.TileConfig(bm, bn)
    kl = costs.k_for_density(a.seq, tiles, a.density)
    thr = bench.calibrated_thresholds(cfg, tiles, kl, dev)
    hq, hkv, d = a.heads_q, a.heads_kv, a.head_dim
    causal = not a.non_causal
    pb = bsfa.BsfaPlan(1, hq, hkv, a.seq, d, tiles=tiles, thresholds=thr, k_level=kl, device=dev, causal=causal)
    pd = bsfa.BsfaPlan(1, hq, hkv, a.seq, d, tiles=tiles, device=dev, causal=causal)
    for p in (pb, pd):
        p.run(q, k, v)
    torch.cuda.synchronize()
    cnt = pb.counters.cpu().tolist()
    res = {"bsfa": [], "dense": []}
    for _ in range(a.rounds):
        for arm, plan in (("bsfa", pb), ("dense", pd)):
            _, t = bench.time_steps(lambda: plan.run(q, k, v), 3, 0, stream)
            res[arm].append(t / 3)
    mb, md = statistics.median(res["bsfa"]), statistics.median(res["dense"])
    f_exec = costs.executed_flops(cnt[0], cnt[1], tiles, d)
    print(json.dumps({"tiles": spec, "seq": a.seq, "causal": causal, "heads": [hq, hkv], "head_dim": d,
                      "k_level": kl,
                      "predicted_density": round(costs.predicted_density(a.seq, tiles, kl), 4),
                      "measured_density": round(cnt[1] / cnt[0], 4),
                      "v_units_skipped_frac": round(1 - cnt[2] / cnt[3], 4),
                      "bsfa_ms": round(mb, 4), "dense_ms": round(md, 4), "speedup": round(md / mb, 4),
                      "executed_tflops": round(f_exec / mb / 1e9, 1)}), flush=True)
