"""Synthetic model-dump generator (paper_2512_07011_b200.workloads) -- CPU checks.

The distribution restated from reference workloads.py:139-216: structured kv
groups (layer * Hkv + g even) bias every q row of the group and the elevated
k rows (sink, trailing window, heavy hitters) along one unit direction with
norm sqrt(6 * sqrt(d)); random groups are plain N(0, 1).
"""
import math

import torch

from paper_2512_07011_b200.workloads import ELEVATION, model_dump_layer


def test_shapes_and_determinism():
    a = model_dump_layer(0, 3, 8, 2, 512, 64, device="cpu", dtype=torch.float32)
    b = model_dump_layer(0, 3, 8, 2, 512, 64, device="cpu", dtype=torch.float32)
    c = model_dump_layer(1, 3, 8, 2, 512, 64, device="cpu", dtype=torch.float32)
    assert [tuple(x.shape) for x in a] == [(8, 512, 64), (2, 512, 64), (2, 512, 64)]
    assert all(torch.equal(x, y) for x, y in zip(a, b))
    assert not torch.equal(a[0], c[0])
    q, k = model_dump_layer(0, 3, 8, 2, 512, 64, device="cpu", with_v=False)
    assert q.dtype == torch.bfloat16 and k.shape == (2, 512, 64)


def test_structured_groups_carry_the_bias():
    n, d, hq, hkv = 1024, 128, 8, 4
    q, k, _ = model_dump_layer(0, 0, hq, hkv, n, d, device="cpu", dtype=torch.float32)
    amp = math.sqrt(ELEVATION * math.sqrt(d))
    g = hq // hkv
    for gk in range(hkv):
        qmean = q[gk * g:(gk + 1) * g].mean(dim=(0, 1))  # the shared bias survives the row mean
        if gk % 2 == 0:  # layer 0: even kv groups are structured
            assert abs(float(qmean.norm()) - amp) < 0.3 * amp
            direction = qmean / qmean.norm()
            proj = k[gk] @ direction
            # sink rows and the trailing window are elevated, the middle is not
            assert float(proj[:64].mean()) > 0.7 * amp
            assert float(proj[n - 128:].mean()) > 0.7 * amp
            assert abs(float(proj[256:512].median())) < 0.5
        else:
            assert float(qmean.norm()) < 0.3 * amp


def test_structure_is_stable_across_samples():
    # the bias direction is a property of (layer, kv head), not of the sample
    q0, _, _ = model_dump_layer(0, 2, 4, 2, 2048, 64, device="cpu", dtype=torch.float32)
    q1, _, _ = model_dump_layer(5, 2, 4, 2, 2048, 64, device="cpu", dtype=torch.float32)
    layer2_structured = 0  # (2 * 2 + 0) % 2 == 0
    m0 = q0[layer2_structured * 2:(layer2_structured + 1) * 2].mean(dim=(0, 1))
    m1 = q1[layer2_structured * 2:(layer2_structured + 1) * 2].mean(dim=(0, 1))
    cos = float(torch.dot(m0, m1) / (m0.norm() * m1.norm()))
    assert cos > 0.95
