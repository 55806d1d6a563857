"""Per-step timeline of one CTA of the v3 forward (debug trace build).

    nvcc ... -DBSFA_TRACE=1 -o paper_2512_07011_b200/_lib/libbsfa_b200_v3trace.so   (tools/build_variants.sh)
    BSFA_LIB_PATH=paper_2512_07011_b200/_lib/libbsfa_b200_v3trace.so python tools/trace_v3.py [--cta 0] [--mode bsfa]

Events (SM clock64): softmax of tile s -- 0 S landed, 1 S copied + released,
2 voted, 3 P half 0 released, 4 step done; MMA warp -- 5 QK_s(j) issued,
6 PV_s(j) picked up (p0 seen), 7 PV_s(j) issued.  Prints medians of the
intervals over the CTA's steps and a few raw rows.
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2512_07011_b200 as bsfa  # noqa: E402
from paper_2512_07011_b200 import _lib, costs  # noqa: E402

STEPS = 2048
EV = ["S", "Ld", "Vote", "P0", "Done", "QKi", "PVseen", "PVi", "Max", "Bar", "QKw", "PVv", "CTA", "Vvote", "Vtma"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=32768)
    ap.add_argument("--cta", type=int, nargs="+", default=[0, 1000])
    ap.add_argument("--mode", nargs="+", default=["bsfa", "dense"])
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = dict(heads_q=32, heads_kv=8, seq_len=a.seq, head_dim=128)
    q, k, v = bench.make_inputs(cfg, 0, dev)
    tiles = bsfa.TileConfig(128, 64)
    kl = costs.k_for_density(a.seq, tiles, 0.5)
    thr = bench.calibrated_thresholds(cfg, tiles, kl, dev)
    lib = _lib.load_library()
    for mode in a.mode:
        plan = (bsfa.BsfaPlan(1, 32, 8, a.seq, 128, tiles=tiles, thresholds=thr, k_level=kl, device=dev)
                if mode == "bsfa" else bsfa.BsfaPlan(1, 32, 8, a.seq, 128, tiles=tiles, device=dev))
        for cta in a.cta:
            buf = torch.zeros((30, STEPS), dtype=torch.int64, device=dev)
            plan.run(q, k, v)
            lib.bsfa_debug_trace(ctypes.c_void_p(buf.data_ptr()), cta)
            plan.run(q, k, v)
            torch.cuda.synchronize()
            lib.bsfa_debug_trace(None, -1)
            t = buf.cpu().numpy().astype(np.int64)
            m_q = a.seq // 128
            qi = m_q - 1 - (cta % (m_q * 2)) // 2
            n = qi + 1
            ev = {name: [t[e * 2 + s, :n] for s in range(2)] for e, name in enumerate(EV)}
            base = min(ev["QKi"][0][0], ev["S"][0][0])
            out = {"mode": mode, "cta": cta, "steps": n,
                   "cycles_per_step": float((ev["Done"][1][n - 1] - ev["Done"][1][0]) / max(1, n - 1))}
            for s in range(2):
                S, Ld, Vo, P0, Dn, QKi, PVs, PVi, Mx, Br, QKw, PVv, _, Vv, Vt = (ev[x][s] for x in EV)
                o = s ^ 1
                out[f"s{s}"] = {
                    "wait_S(Done_j-1->S_j)": float(np.median(S[1:] - Dn[:-1])),
                    "ld(S->Ld)": float(np.median(Ld - S)),
                    "vote(Ld->Vote)": float(np.median(Vo - Ld)),
                    "  max(Ld->Max)": float(np.median(Mx - Ld)),
                    "  bar(Max->Bar)": float(np.median(Br - Mx)),
                    "  post(Bar->Vote)": float(np.median(Vo - Br)),
                    "half0(Vote->P0)": float(np.median(P0 - Vo)),
                    "rest(P0->Done)": float(np.median(Dn - P0)),
                    "softmax_busy(S->Done)": float(np.median(Dn - S)),
                    "qk_land(QKi->S)": float(np.median(S - QKi)),
                    "pv_pickup(P0->PVseen)": float(np.median(PVs - P0)),
                    "pv_issue(PVseen->PVi)": float(np.median(PVi - PVs)),
                    "  qk_mma_issue(QKw->QKi)": float(np.median(QKi - QKw)),
                    "  pv_vwait(PVseen->PVv, kept)": float(np.median((PVv - PVs)[PVv > PVs])) if (PVv > PVs).any() else -1,
                    "  pv_mma_issue(PVv->PVi, kept)": float(np.median((PVi - PVv)[PVv > PVs])) if (PVv > PVs).any() else -1,
                    "vprod_vote_seen(Vote->Vvote)": float(np.median(Vv - Vo)),
                    "vprod_tma(Vvote->Vtma, issued)": float(np.median((Vt - Vv)[Vt > Vv])) if (Vt > Vv).any() else -1,
                    "v_latency(Vtma->PVv, kept)": float(np.median((PVv - Vt)[(PVv > PVs) & (Vt > Vv)])) if ((PVv > PVs) & (Vt > Vv)).any() else -1,
                }
            # QK issue lag behind the previous S owner's release
            QK0, QK1 = ev["QKi"][0], ev["QKi"][1]
            Ld0, Ld1 = ev["Ld"][0], ev["Ld"][1]
            out["qk1_issue_after_ld0"] = float(np.median(QK1[:n] - Ld0[:n]))
            out["qk0_issue_after_ld1(prev)"] = float(np.median(QK0[1:n] - Ld1[:n - 1]))
            t0, e0, e1 = t[24, 0], t[25, 0], t[25, 1]
            out["cta_prologue(start->S0(0))"] = int(ev["S"][0][0] - t0)
            out["cta_epilogue(Done0(last)->end0)"] = int(e0 - ev["Done"][0][n - 1])
            out["cta_total"] = int(max(e0, e1) - t0)
            out["cta_steps_share"] = round(float(ev["Done"][0][n - 1] - ev["S"][0][0]) / max(1, int(max(e0, e1) - t0)), 3)
            print(json.dumps(out), flush=True)
            for j in (1, 2, 3, n // 2, n // 2 + 1, n // 2 + 2):
                if j < n:
                    print("   j=%4d " % j + " ".join(f"{x}{s}={int(ev[x][s][j] - base):8d}" for s in range(2) for x in EV))


if __name__ == "__main__":
    main()
