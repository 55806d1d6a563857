"""Per-step timeline of one CTA pair of the v7 (cta_group::2) forward, debug trace build.

    tools/build_variants.sh v7trace "-DBSFA_TRACE=1"
    BSFA_LIB_PATH=paper_2512_07011_b200/_lib/libbsfa_b200_v7trace.so python tools/trace_v7.py [--unit 0 500]

Events (SM clock64; rank r = CTA of the pair, both SMs' clocks): softmax warp 0
-- 0 S landed, 1 S copied + s_free, 2 voted, 3 exps done, 4 step done
(p_full); MMA warp (rank 0) -- 10 QK(j) K ready, 5 QK(j) issued, 6 p_full(j)
seen, 11 V of PV(j) ready, 7 PV(j) issued; V producer -- 13 decision read,
14 V TMA issued.  Prints medians of the intervals over the unit's steps.
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


def med(x):
    x = x[np.isfinite(x)]
    return float(np.median(x)) if x.size else -1.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=32768)
    ap.add_argument("--unit", type=int, nargs="+", default=[0, 1000])
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
    m_q = a.seq // 128
    for mode in a.mode:
        plan = (bsfa.BsfaPlan(1, 32, 8, a.seq, 128, tiles=tiles, thresholds=thr, k_level=kl, device=dev)
                if mode == "bsfa" else bsfa.BsfaPlan(1, 32, 8, a.seq, 128, tiles=tiles, device=dev))
        for unit in a.unit:
            buf = torch.zeros((32, STEPS), dtype=torch.int64, device=dev)
            plan.run(q, k, v)
            lib.bsfa_debug_trace(ctypes.c_void_p(buf.data_ptr()), unit)
            plan.run(q, k, v)
            torch.cuda.synchronize()
            lib.bsfa_debug_trace(None, -1)
            t = buf.cpu().numpy().astype(np.float64)
            qi = m_q - 1 - (unit % (m_q * 2)) // 2
            n = qi + 1
            ev = lambda e, r: t[e * 2 + r, :n]  # noqa: E731
            out = {"mode": mode, "unit": unit, "steps": n}
            for r in range(2):
                S, Ld, Vo, Ex, Dn = (ev(e, r) for e in range(5))
                out[f"r{r}_cycles_per_step"] = float((Dn[n - 1] - Dn[0]) / max(1, n - 1))
                out[f"r{r}"] = {
                    "wait_S(Done_j-1->S_j)": med(S[1:] - Dn[:-1]),
                    "ld(S->Ld)": med(Ld - S),
                    "vote(Ld->Vote)": med(Vo - Ld),
                    "exps(Vote->Exps)": med(Ex - Vo),
                    "tail(Exps->Done)": med(Dn - Ex),
                    "busy(S->Done)": med(Dn - S),
                }
            QKw, QKi, Pseen, Vr, PVi = (ev(e, 0) for e in (10, 5, 6, 11, 7))
            S0, Ld0, Dn0 = ev(0, 0), ev(1, 0), ev(4, 0)
            Vd, Vt = ev(13, 0), ev(14, 0)
            kept = Vr > 0
            out["mma"] = {
                "qk_issue(QKw->QKi)": med(QKi - QKw),
                "qk_land(QKi(j)->S(j))": med(S0 - QKi),
                "qk_lead(S(j) ready before softmax wants it: Done(j-1)-S(j))": med(Dn0[:-1] - S0[1:]),
                "pfull_seen(Done(j)->Pseen(j))": med(Pseen - Dn0),
                "v_wait(Pseen->Vready, kept)": med((Vr - Pseen)[kept]),
                "pv_issue(Pseen->PVi)": med(PVi - Pseen),
                "qk(j+2)_after_ld(j)": med(QKw[2:] - Ld0[:-2]),
                "vdec_after_vote": med(Vd - ev(2, 0)),
                "vtma_after_dec": med((Vt - Vd)[Vt > 0]),
                "v_latency(Vtma->Vready)": med((Vr - Vt)[(Vr > 0) & (Vt > 0)]),
            }
            print(json.dumps(out), flush=True)
            for j in (1, 2, 3, n // 2, n // 2 + 1):
                if j < n:
                    print("   j=%4d " % j + " ".join(f"e{e}r{r}={int(t[e * 2 + r, j] - t[0, 0]):8d}"
                                                     for r in range(2) for e in (0, 1, 2, 3, 4, 13, 14)
                                                     ) + " | " + " ".join(f"e{e}={int(t[e * 2, j] - t[0, 0]):8d}"
                                                                          for e in (10, 5, 6, 11, 7)))


if __name__ == "__main__":
    main()
