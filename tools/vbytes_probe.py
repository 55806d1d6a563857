"""One BSFA launch and one dense launch of the l32k workload (for an ncu metric
capture of L2->SM bytes: the difference is the V traffic the gate skipped).

    ncu --metrics lts__t_sectors_srcunit_tex_op_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum \
        -k regex:bsfa_kernel python tools/vbytes_probe.py
Prints the kernel counters of both launches (V tiles loaded / loadable).
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2512_07011_b200 as bsfa  # noqa: E402
from paper_2512_07011_b200 import costs  # noqa: E402

cfg = bench.CONFIGS["l32k"]
dev = torch.device("cuda", 0)
tiles = bsfa.TileConfig(128, 64)
n, d, hq, hkv = cfg["seq_len"], cfg["head_dim"], cfg["heads_q"], cfg["heads_kv"]
k_level = costs.k_for_density(n, tiles, 0.5)
thr = bench.calibrated_thresholds(cfg, tiles, k_level, dev)
q, k, v = bench.make_inputs(cfg, 0, dev)
out = {}
for name, kw in (("bsfa", dict(thresholds=thr, k_level=k_level)), ("dense", {})):
    plan = bsfa.BsfaPlan(1, hq, hkv, n, d, tiles=tiles, device=dev, **kw)
    plan.run(q, k, v)
    torch.cuda.synchronize()
    c = plan.counters.cpu().tolist()
    out[name] = {"reachable": c[0], "kept": c[1], "v_loaded": c[2], "v_loadable": c[3],
                 "v_bytes": c[2] * 64 * d * 2}
print(json.dumps(out))
