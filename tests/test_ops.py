"""torch.ops.bsfa.* registration and fake (meta) shapes -- CPU; numerics are in test_gpu_parity.py."""
import torch
from torch._subclasses.fake_tensor import FakeTensorMode

import paper_2512_07011_b200  # noqa: F401  (registers the ops)


def test_ops_registered_with_fake_shapes():
    with FakeTensorMode():
        q = torch.empty(2, 4, 1000, 64, dtype=torch.bfloat16, device="cuda")
        k = torch.empty(2, 2, 1000, 64, dtype=torch.bfloat16, device="cuda")
        thr = torch.empty(4, 8, device="cuda")
        o, lse, cnt, dec = torch.ops.bsfa.fwd(q, k, k, thr, True, 128, 64, 0.125, True)
        assert o.shape == q.shape and o.dtype == torch.bfloat16 and o.device.type == "cuda"
        assert lse.shape == (2, 4, 1000) and cnt.shape == (4,) and dec.shape == (2, 4, 8, 16)
        _, _, _, nodec = torch.ops.bsfa.fwd(q, k, k, thr[:0], True, 128, 128, 0.125, False)
        assert nodec.numel() == 0
        bm = torch.ops.bsfa.blockmax(q, k, 128, 64)
        assert bm.shape == (2, 4, 8, 16) and bm.dtype == torch.float32
        t, ties = torch.ops.bsfa.calib_select(bm, [0, 3, 7], 128, 64)
        assert t.shape == (3, 2, 4, 8) and ties.shape == (3,)


def test_ops_fake_shapes_bm64():
    """b_m = 64: the reference grid of n = 1000 is 1024 rows (lcm 64 / 128), 16 query blocks."""
    with FakeTensorMode():
        q = torch.empty(1, 2, 1000, 128, dtype=torch.bfloat16, device="cuda")
        thr = torch.empty(2, 16, device="cuda")
        _, _, _, dec = torch.ops.bsfa.fwd(q, q, q, thr, True, 64, 64, 0.088, True)
        assert dec.shape == (1, 2, 16, 16)
        assert torch.ops.bsfa.blockmax(q, q, 64, 128).shape == (1, 2, 16, 8)
