"""Same-process A/B of several builds of the library: BSFA and dense launches of
every variant interleaved round-robin, so all variants see the same thermal /
power state (cross-process A/B runs drift by +-3 %).

    python tools/ab_multi.py --libs v3 vp [--seq 32768] [--rounds 8]

Each variant is paper_2512_07011_b200/_lib/libbsfa_b200_<name>.so, loaded with
ctypes under its own handle; the plans are the package's BsfaPlan with the
library handle swapped.  Prints one JSON line per variant (median ms).
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2512_07011_b200 as bsfa  # noqa: E402
from paper_2512_07011_b200 import _lib, costs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--libs", nargs="+", required=True)
ap.add_argument("--seq", type=int, default=32768)
ap.add_argument("--density", type=float, default=0.5)
ap.add_argument("--rounds", type=int, default=8)
ap.add_argument("--launches", type=int, default=2)
ap.add_argument("--tiles", default="128x64", help="b_m x b_n")
a = ap.parse_args()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
tiles = bsfa.TileConfig(*(int(x) for x in a.tiles.split("x")))
cfg = dict(heads_q=32, heads_kv=8, seq_len=a.seq, head_dim=128)
kl = costs.k_for_density(a.seq, tiles, a.density)
thr = bench.calibrated_thresholds(cfg, tiles, kl, dev)
q, k, v = bench.make_inputs(cfg, 0, dev)
stream = torch.cuda.current_stream(dev)
variants = {}
for name in a.libs:
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2512_07011_b200", "_lib", f"libbsfa_b200_{name}.so"))
    lib.bsfa_fwd.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    lib.bsfa_fwd.restype = ctypes.c_int
    lib.bsfa_last_error.restype = ctypes.c_char_p
    pb = bsfa.BsfaPlan(1, 32, 8, a.seq, 128, tiles=tiles, thresholds=thr, k_level=kl, device=dev)
    pd = bsfa.BsfaPlan(1, 32, 8, a.seq, 128, tiles=tiles, device=dev)
    pb.lib = lib
    pd.lib = lib
    variants[name] = (pb, pd, {"bsfa": [], "dense": []})
for _ in range(2):
    for pb, pd, _r in variants.values():
        pb.run(q, k, v)
        pd.run(q, k, v)
torch.cuda.synchronize()
ref = None
for name, (pb, pd, _r) in variants.items():  # every build must compute the same thing
    o = pb.run(q, k, v).clone()
    c = pb.counters.clone()
    torch.cuda.synchronize()
    if ref is None:
        ref = (o, c)
    else:
        assert torch.equal(c, ref[1]), f"{name}: counters differ"
        err = (o.float() - ref[0].float()).abs().max().item()
        assert err < 2e-2, f"{name}: output differs by {err}"
for _ in range(a.rounds):
    for arm in ("bsfa", "dense"):
        for name, (pb, pd, res) in variants.items():
            plan = pb if arm == "bsfa" else pd
            _, t = bench.time_steps(lambda: plan.run(q, k, v), a.launches, 0, stream)
            res[arm].append(t / a.launches)
for name, (pb, pd, res) in variants.items():
    mb, md = statistics.median(res["bsfa"]), statistics.median(res["dense"])
    print(json.dumps({"lib": name, "seq": a.seq, "bsfa_ms": round(mb, 4), "dense_ms": round(md, 4),
                      "speedup": round(md / mb, 4), "bsfa_all": [round(x, 3) for x in res["bsfa"]],
                      "dense_all": [round(x, 3) for x in res["dense"]]}), flush=True)
