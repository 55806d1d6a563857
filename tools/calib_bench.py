"""Time the calibration kernel (K2) on one Llama-shaped layer: 32 q / 8 kv heads, d = 128, N = 32K.

    python tools/calib_bench.py [--n 32768] [--reps 10]
Prints ms per layer and QK TFLOP/s over the off-frontier tiles it scores.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_07011_b200 as bsfa  # noqa: E402
from paper_2512_07011_b200.workloads import model_dump_layer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--hkv", type=int, default=8, help="kv heads (32 q heads): 8 = Llama GQA, 32 = MHA")
    a = ap.parse_args()
    n, hq, hkv, d = a.n, 32, a.hkv, 128
    tiles = bsfa.TileConfig(128, 64)
    q, k = model_dump_layer(0, 0, hq, hkv, n, d, device="cuda", with_v=False)
    cal = bsfa.Calibrator([82, 149, 231], tiles, 1, hq, n, d)
    for _ in range(3):
        cal.add_layer(0, 0, q, k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        cal.add_layer(0, 0, q, k)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    m_q = n // 128
    tiles_scored = hq * sum(2 * i for i in range(m_q))  # off-frontier gate tiles j < 2i per query block
    flops = 2.0 * 128 * 64 * d * tiles_scored
    print(json.dumps({"n": n, "heads_kv": hkv, "ms_per_layer": ms, "qk_tflops": flops / (ms * 1e-3) / 1e12}))


if __name__ == "__main__":
    main()
