"""Throughput of the forward for other GQA group sizes at 32K (d = 128, 32 q heads, ~50 % skip)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2512_07011_b200 as bsfa  # noqa: E402
from paper_2512_07011_b200 import costs  # noqa: E402

dev = torch.device("cuda", 0)
tiles = bsfa.TileConfig(128, 64)
stream = torch.cuda.current_stream(dev)
n, d, hq = 32768, 128, 32
for hkv in (8, 32, 16):
    cfg = dict(heads_q=hq, heads_kv=hkv, seq_len=n, head_dim=d)
    q, k, v = bench.make_inputs(cfg, 0, dev)
    kl = costs.k_for_density(n, tiles, 0.5)
    thr = bench.calibrated_thresholds(cfg, tiles, kl, dev)
    plan = bsfa.BsfaPlan(1, hq, hkv, n, d, tiles=tiles, thresholds=thr, k_level=kl, device=dev)
    _, tot = bench.time_steps(lambda: plan.run(q, k, v), 10, 3, stream)
    c = plan.counters.cpu().tolist()
    ms = tot / 10
    dplan = bsfa.BsfaPlan(1, hq, hkv, n, d, tiles=tiles, device=dev)
    _, dtot = bench.time_steps(lambda: dplan.run(q, k, v), 10, 3, stream)
    print(json.dumps({"heads_kv": hkv, "group": hq // hkv, "ms": ms, "dense_ms": dtot / 10,
                      "exec_tflops": costs.executed_flops(c[0], c[1], tiles, d) / ms / 1e9,
                      "skip": 1 - c[1] / c[0]}))
    del q, k, v, plan, dplan
