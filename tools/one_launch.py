"""Two forward launches at one Llama-shaped config, for ncu captures (-s 1 -c 1).

    python tools/one_launch.py [--seq 32768] [--gate dense|threshold] [--T 3.84]

Fixed threshold (no calibration launch), so the only kernels are the forward.
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2512_07011_b200 as bsfa  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=32768)
ap.add_argument("--gate", default="threshold")
ap.add_argument("--T", type=float, default=3.84)
ap.add_argument("--launches", type=int, default=2)
ap.add_argument("--heads-q", type=int, default=32)
ap.add_argument("--heads-kv", type=int, default=8)
ap.add_argument("--head-dim", type=int, default=128)
a = ap.parse_args()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
cfg = dict(heads_q=a.heads_q, heads_kv=a.heads_kv, seq_len=a.seq, head_dim=a.head_dim)
q, k, v = bench.make_inputs(cfg, 0, dev)
tiles = bsfa.TileConfig(128, 64)
thr = None
if a.gate == "threshold":
    P = a.seq // 128
    thr = bsfa.ThresholdTensor(values=np.full((1, 1, a.heads_q, P), a.T, dtype=np.float32), k_levels=(1,),
                               n_max=a.seq, b_m=128, b_n=64)
plan = bsfa.BsfaPlan(1, a.heads_q, a.heads_kv, a.seq, a.head_dim, tiles=tiles, thresholds=thr,
                     k_level=1 if thr else None, device=dev)
for _ in range(a.launches):
    plan.run(q, k, v)
torch.cuda.synchronize()
c = plan.counters.cpu().numpy()
print("counters", c.tolist(), "density", c[1] / c[0])
