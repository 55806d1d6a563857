"""A/B timing of the forward library in $BSFA_LIB_PATH: BSFA and dense interleaved.

    python tools/ab.py [--seq 32768] [--density 0.5] [--rounds 5] [--tag name]

Thresholds are calibrated once per (seq, density) on the seed-1000 sample and
cached under /tmp, so every library variant gates with identical thresholds.
Prints one JSON line: per-arm median ms over `rounds` ABAB rounds of 3 launches each.
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
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--tag", default=os.path.basename(os.environ.get("BSFA_LIB_PATH", "default")))
a = ap.parse_args()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
tiles = bsfa.TileConfig(128, 64)
cfg = dict(heads_q=32, heads_kv=8, seq_len=a.seq, head_dim=128)
kl = costs.k_for_density(a.seq, tiles, a.density)
path = f"/tmp/thr_{a.seq}_{kl}.bsfa"
if os.path.exists(path):
    thr = bsfa.load_thresholds(path)
else:
    thr = bench.calibrated_thresholds(cfg, tiles, kl, dev)
    bsfa.save_thresholds(thr, path)
q, k, v = bench.make_inputs(cfg, 0, dev)
plan = bsfa.BsfaPlan(1, 32, 8, a.seq, 128, tiles=tiles, thresholds=thr, k_level=kl, device=dev)
dplan = bsfa.BsfaPlan(1, 32, 8, a.seq, 128, tiles=tiles, device=dev)
stream = torch.cuda.current_stream(dev)
for _ in range(3):
    plan.run(q, k, v)
    dplan.run(q, k, v)
bs, ds = [], []
clk = {"bsfa": [], "dense": []}
pwr = {"bsfa": [], "dense": []}


def sample(arm, fn):
    with bench.ClockSampler(0) as cs:
        _, t = bench.time_steps(fn, 3, 0, stream)
    clk[arm] += [x for x, _, _ in cs.samples]
    pwr[arm] += [w for _, _, w in cs.samples if w]
    return t / 3


for _ in range(a.rounds):
    bs.append(sample("bsfa", lambda: plan.run(q, k, v)))
    ds.append(sample("dense", lambda: dplan.run(q, k, v)))
c = plan.counters.cpu().numpy()
reach, kept = int(c[0]), int(c[1])
fe = costs.executed_flops(reach, kept, tiles, 128)
mb, md = statistics.median(bs), statistics.median(ds)
print(json.dumps({"tag": a.tag, "seq": a.seq, "density": round(kept / reach, 4), "bsfa_ms": round(mb, 4),
                  "dense_ms": round(md, 4), "speedup": round(md / mb, 4), "bsfa_tflops": round(fe / mb / 1e9, 1),
                  "dense_tflops": round(costs.dense_flops(reach, tiles, 128) / md / 1e9, 1),
                  "bsfa_mhz": statistics.median(clk["bsfa"]) if clk["bsfa"] else None,
                  "dense_mhz": statistics.median(clk["dense"]) if clk["dense"] else None,
                  "bsfa_w": statistics.median(pwr["bsfa"]) if pwr["bsfa"] else None,
                  "dense_w": statistics.median(pwr["dense"]) if pwr["dense"] else None,
                  "bsfa_all": [round(x, 3) for x in bs], "dense_all": [round(x, 3) for x in ds]}), flush=True)
