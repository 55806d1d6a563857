"""Per-step timeline of one CTA (debug trace hook) for the L32K workload.

Needs the trace build:  nvcc ... -DBSFA_TRACE=1 -o paper_2512_07011_b200/_lib/variants/libbsfa_b200_trace.so
and BSFA_LIB_PATH pointing at it.  Runs the BSFA and dense forward with
bsfa_debug_trace on one CTA and prints median intervals (SM cycles) per
query tile s of the CTA.
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

EV = ["SReady", "Voted", "PDone", "PSeen", "VReady", "Issued", "MaxDone", "Half0"]
STEPS = 2048


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
    buf = torch.zeros((16, STEPS), dtype=torch.int64, device=dev)
    lib = _lib.load_library()
    plan.run(q, k, v)
    lib.bsfa_debug_trace(ctypes.c_void_p(buf.data_ptr()), cta)
    plan.run(q, k, v)
    torch.cuda.synchronize()
    lib.bsfa_debug_trace(None, -1)
    t = buf.cpu().numpy().astype(np.int64)
    m_q = seq // 128
    per_bg = m_q * 2
    qi = m_q - 1 - (cta % per_bg) // 2
    n = qi + 1
    ev = {name: [t[e * 2 + s, :n] for s in range(2)] for e, name in enumerate(EV)}
    base = ev["SReady"][0][0]
    out = {"steps": n}
    for s in range(2):
        sr, vo, pd, ps, vr, iss, ld, ex = (ev[x][s] for x in EV)
        out[f"s{s}_ldmax(S->MaxDone)"] = float(np.median(ld - sr))
        out[f"s{s}_vote(MaxDone->Voted)"] = float(np.median(vo - ld))
        kept0 = ex > 0
        out[f"s{s}_half0(Voted->Half0 arrive)"] = float(np.median((ex - vo)[kept0])) if kept0.any() else -1
        out[f"s{s}_half1(Half0->PDone)"] = float(np.median((pd - ex)[kept0])) if kept0.any() else -1
        out[f"s{s}_softmax(S->Pdone)"] = float(np.median(pd - sr))
        out[f"s{s}_vote(S->Voted)"] = float(np.median(vo - sr))
        out[f"s{s}_mma_lag(Pdone->Pseen)"] = float(np.median(ps - pd))
        out[f"s{s}_mma_issue(Pseen->Issued)"] = float(np.median(iss - ps))
        out[f"s{s}_S_wait(Issued_j->SReady_j+1)"] = float(np.median(sr[1:] - iss[:-1]))
        out[f"s{s}_step"] = float(np.median(np.diff(pd)))
    out["cycles_per_step"] = float((ev["PDone"][1][n - 1] - base) / n)
    print(mode, "cta", cta, "qblock", qi, json.dumps({k: round(v, 1) for k, v in out.items()}))
    for j in list(range(0, 6)) + list(range(n // 2, n // 2 + 4)):
        row = " ".join(f"{x}{s}={int(ev[x][s][j] - base) if ev[x][s][j] else -1:8d}" for s in range(2) for x in EV)
        print(f"  j={j:4d} {row}")


if __name__ == "__main__":
    for cta in (0, 1280):
        for m in ("bsfa", "dense"):
            run(m, cta=cta)
