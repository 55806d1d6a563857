"""Per-step timeline of one CTA of the gate-step kernel (64-key steps), BSFA_TRACE build."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_07011_b200 as bsfa  # noqa: E402
from paper_2512_07011_b200 import _lib, costs  # noqa: E402

EV = ["SReady", "Voted", "PDone", "PSeen", "VReady", "Issued"]
seq = 32768
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
q = torch.randn((1, 32, seq, 128), generator=g, device=dev).to(torch.bfloat16)
k = torch.randn((1, 8, seq, 128), generator=g, device=dev).to(torch.bfloat16)
v = torch.randn((1, 8, seq, 128), generator=g, device=dev).to(torch.bfloat16)
tiles = bsfa.TileConfig(128, 64)
for mode in ("bsfa", "dense"):
    for cta in (0, 1280):
        if mode == "bsfa":
            kl = costs.k_for_density(seq, tiles, 0.5)
            cal = bsfa.Calibrator([kl], tiles, 1, 32, seq, 128)
            cal.add_layer(0, 0, q[0], k[0])
            plan = bsfa.BsfaPlan(1, 32, 8, seq, 128, thresholds=cal.finish(), k_level=kl, return_trace=True)
        else:
            plan = bsfa.BsfaPlan(1, 32, 8, seq, 128, return_trace=True)
        buf = torch.zeros((16, 2048), dtype=torch.int64, device=dev)
        lib = _lib.load_library()
        plan.run(q, k, v)
        lib.bsfa_debug_trace(ctypes.c_void_p(buf.data_ptr()), cta)
        plan.run(q, k, v)
        torch.cuda.synchronize()
        lib.bsfa_debug_trace(None, -1)
        t = buf.cpu().numpy().astype(np.int64)
        m_q = seq // 128
        bg, rem = divmod(cta, m_q * 2)
        qi = m_q - 1 - rem // 2
        n = min(2 * qi + 2, 2048)
        heads = [bg * 4 + (rem % 2) * 2 + s for s in range(2)]
        dec = plan.decisions[0].cpu().numpy()
        for s in range(2):
            e = {name: t[i * 2 + s, :n] for i, name in enumerate(EV)}
            kept = dec[heads[s], qi, :n] >= 2
            per = np.diff(e["SReady"])
            out = {"step(S->S)": np.median(per), "S->Voted": np.median(e["Voted"] - e["SReady"]),
                   "Voted->PDone kept": np.median((e["PDone"] - e["Voted"])[kept]),
                   "Voted->PDone skip": np.median((e["PDone"] - e["Voted"])[~kept]) if (~kept).any() else -1,
                   "PDone->PSeen": np.median(e["PSeen"] - e["PDone"]),
                   "PSeen->Issued": np.median(e["Issued"] - e["PSeen"]),
                   "PDone(j)->SReady(j+2)": np.median(e["SReady"][2:] - e["PDone"][:-2]),
                   "SReady(j+1)-PDone(j) (negative = S ready early)": np.median(e["SReady"][1:] - e["PDone"][:-1]),
                   "cycles/64 keys": (e["PDone"][n - 1] - e["SReady"][0]) / n, "kept frac": kept.mean()}
            print(mode, "cta", cta, "tile", s, " ".join(f"{kk}={vv:.0f}" if kk != "kept frac" else f"{kk}={vv:.2f}"
                                                        for kk, vv in out.items()))
