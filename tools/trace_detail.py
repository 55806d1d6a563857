"""Per-step softmax phase durations of one CTA, split by which gate halves were kept.

Needs the BSFA_TRACE=1 build via BSFA_LIB_PATH.  Prints, per query tile of the
traced CTA, the median duration of each phase for steps with 0, 1 or 2 kept
64-key halves.
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_07011_b200 as bsfa  # noqa: E402
from paper_2512_07011_b200 import _lib, costs  # noqa: E402

EV = ["SReady", "Voted", "PDone", "PSeen", "VReady", "Issued", "MaxDone", "Half0"]
seq, cta = 32768, int(sys.argv[1]) if len(sys.argv) > 1 else 1280
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
q = torch.randn((1, 32, seq, 128), generator=g, device=dev).to(torch.bfloat16)
k = torch.randn((1, 8, seq, 128), generator=g, device=dev).to(torch.bfloat16)
v = torch.randn((1, 8, seq, 128), generator=g, device=dev).to(torch.bfloat16)
tiles = bsfa.TileConfig(128, 64)
kl = costs.k_for_density(seq, tiles, 0.5)
cal = bsfa.Calibrator([kl], tiles, 1, 32, seq, 128)
cal.add_layer(0, 0, q[0], k[0])
thr = cal.finish()
plan = bsfa.BsfaPlan(1, 32, 8, seq, 128, thresholds=thr, k_level=kl, return_trace=True)
buf = torch.zeros((16, 2048), dtype=torch.int64, device=dev)
lib = _lib.load_library()
plan.run(q, k, v)
lib.bsfa_debug_trace(ctypes.c_void_p(buf.data_ptr()), cta)
plan.run(q, k, v)
torch.cuda.synchronize()
lib.bsfa_debug_trace(None, -1)
t = buf.cpu().numpy().astype(np.int64)
m_q = seq // 128
per_bg = m_q * 2
bg, rem = divmod(cta, per_bg)
qi = m_q - 1 - rem // 2
pr = rem % 2
heads = [bg * 4 + pr * 2 + s for s in range(2)]
dec = plan.decisions[0].cpu().numpy()
n = qi + 1
for s in range(2):
    e = {name: t[i * 2 + s, :n] for i, name in enumerate(EV)}
    d = dec[heads[s], qi, : 2 * n].reshape(n, 2)
    nk = (d >= 2).sum(1)
    print(f"tile {s} (head {heads[s]}, qblock {qi}): kept halves per step: 0:{(nk == 0).sum()} 1:{(nk == 1).sum()} 2:{(nk == 2).sum()}")
    for c in (0, 1, 2):
        sel = nk == c
        sel[-1] = False  # frontier step
        if not sel.any():
            continue
        ph = {
            "post(Voted->PostDone)": e["MaxDone"] - e["Voted"],
            "S->Voted": e["Voted"] - e["SReady"],
            "PostDone->Half0": e["Half0"] - e["MaxDone"],
            "half1": e["PDone"] - e["Half0"],
            "S->PDone": e["PDone"] - e["SReady"],
        }
        nxt = np.append(e["SReady"][1:], 0) - e["PDone"]
        ph["PDone->S(j+1)"] = nxt
        print(f"  kept={c}: " + " ".join(f"{kk} {int(np.median(vv[sel]))}" for kk, vv in ph.items()))
