"""Per-tile timeline of one CTA (debug trace hook) for the L32K workload.

Runs the BSFA and dense forward with bsfa_debug_trace enabled on CTA 0
(query block 255, the longest) and prints median intervals (SM cycles).
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_07011_b200 as bsfa  # noqa: E402
from paper_2512_07011_b200 import _lib, costs  # noqa: E402

EV = ["SReady", "Voted", "PDone", "PSeen", "Issued"]


def run(mode, seq=32768, cta=0):
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    q = torch.randn((1, 32, seq, 128), generator=g, device=dev).to(torch.bfloat16)
    k = torch.randn((1, 8, seq, 128), generator=g, device=dev).to(torch.bfloat16)
    v = torch.randn((1, 8, seq, 128), generator=g, device=dev).to(torch.bfloat16)
    tiles = bsfa.TileConfig(128, 64)
    if mode == "bsfa":
        kl = costs.k_for_density(seq, tiles, 0.5)
        cal = bsfa.Calibrator([kl], tiles, 1, 32, seq, 128)
        cal.add_layer(0, 0, q[0], k[0])
        thr = cal.finish()
        plan = bsfa.BsfaPlan(1, 32, 8, seq, 128, thresholds=thr, k_level=kl)
    else:
        plan = bsfa.BsfaPlan(1, 32, 8, seq, 128)
    buf = torch.zeros((8, 4096), dtype=torch.int64, device=dev)
    lib = _lib.load_library()
    plan.run(q, k, v)
    lib.bsfa_debug_trace(ctypes.c_void_p(buf.data_ptr()), cta)
    plan.run(q, k, v)
    torch.cuda.synchronize()
    lib.bsfa_debug_trace(None, -1)
    t = buf.cpu().numpy().astype(np.int64)
    per_bg = (seq // 128) * 4
    qi = seq // 128 - 1 - (cta % per_bg) // 4
    n = (qi + 1) * 2
    sr, vo, pd, ps, iss, vr, kr = (t[i, :n] for i in range(7))
    out = {}
    out["softmax_C"] = np.median(pd - sr)
    out["vote_part"] = np.median(vo - sr)
    out["mma_lag_after_pdone"] = np.median(ps - pd)
    out["mma_issue"] = np.median(iss - ps)
    kept = vr > 0
    out["v_wait_after_pseen"] = float(np.median((vr - ps)[kept])) if kept.any() else -1
    out["v_ready_minus_voted"] = float(np.median((vr - vo)[kept])) if kept.any() else -1
    out["k_ready(j+NS)_minus_pseen(j)"] = float(np.median(kr[4:] - ps[:-4]))
    out["kept_frac"] = float(kept.mean())
    out["chain_issue_to_sready_j+2"] = np.median(sr[2:] - iss[:-2])
    out["per_tile_pdone_step"] = np.median(np.diff(pd))
    out["per_tile_pseen_step"] = np.median(np.diff(ps))
    out["total_cycles"] = int(pd[n - 1] - sr[0])
    out["cycles_per_tile"] = out["total_cycles"] / n
    print(mode, "cta", cta, "tiles", n, json.dumps({k: round(float(v), 1) for k, v in out.items()}))
    # first 12 tiles raw (relative)
    base = sr[0]
    for j in range(0, 12):
        print(f"  j={j:3d} S={sr[j]-base:8d} V={vo[j]-base:8d} P={pd[j]-base:8d} seen={ps[j]-base:8d} "
              f"vrdy={(vr[j]-base) if vr[j] else -1:8d} krdy={kr[j]-base:8d} iss={iss[j]-base:8d}")


for cta in (0, 2560):
    for m in ("bsfa", "dense"):
        run(m, cta=cta)
