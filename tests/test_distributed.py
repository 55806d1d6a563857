"""Head sharding + output all-gather, exercised with world_size 2 on gloo (CPU).

The per-rank compute is the CPU oracle (tests may use it); what is tested is
the partition (which q/kv heads and threshold rows a rank owns) and the
gather layout, i.e. the multi-GPU logic of ``distributed.py`` minus the
kernel itself.
"""

import os
import socket
from dataclasses import dataclass

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_07011_b200.distributed import HeadShard, gather_heads, shard_heads, sharded_attention
from paper_2512_07011_b200.errors import ConfigurationError


def test_shard_heads_partition():
    assert shard_heads(32, 8, 8, 3) == HeadShard(3, 8, 12, 16, 3, 4)
    assert shard_heads(32, 8, 2, 1) == HeadShard(1, 2, 16, 32, 4, 8)
    cover = sorted(h for r in range(4) for h in range(*(lambda s: (s.q_lo, s.q_hi))(shard_heads(32, 8, 4, r))))
    assert cover == list(range(32))
    with pytest.raises(ConfigurationError):
        shard_heads(32, 8, 3, 0)


@dataclass
class _Res:
    o: torch.Tensor


def _oracle_compute(q, k, v, thresholds=None, layer=0, k_level=None, head_offset=0, **kw):
    from oracle import bsfa_oracle as orc
    b, hq, n, d = q.shape
    g = hq // k.shape[1]
    lvl = thresholds.level_index(k_level)
    out = torch.empty_like(q)
    for bi in range(b):
        for h in range(hq):
            thr = thresholds.values[lvl, layer, head_offset + h]
            o, _, _ = orc.flash_forward(q[bi, h].numpy(), k[bi, h // g].numpy(), v[bi, h // g].numpy(), True,
                                        128, 64, orc.threshold_gate(thr))
            out[bi, h] = torch.from_numpy(o)
    return _Res(out)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, k, v, thr, expected, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, full = sharded_attention(q, k, v, rank=rank, world=world, thresholds=thr, layer=1, k_level=4,
                                    gather=True, compute=_oracle_compute)
        err = float((full - expected).abs().max())
        result_q.put((rank, tuple(full.shape), err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [1, 2])
def test_two_rank_gather_matches_single_process(batch):
    import paper_2512_07011_b200 as bsfa
    rng = np.random.default_rng(batch)
    hq, hkv, n, d = 4, 2, 256, 16
    q = torch.from_numpy(rng.standard_normal((batch, hq, n, d)).astype(np.float32))
    k = torch.from_numpy(rng.standard_normal((batch, hkv, n, d)).astype(np.float32))
    v = torch.from_numpy(rng.standard_normal((batch, hkv, n, d)).astype(np.float32))
    vals = rng.uniform(0.5, 1.0, size=(1, 2, hq, 2)).astype(np.float32)
    thr = bsfa.ThresholdTensor(values=vals, k_levels=(4,), n_max=256, b_m=128, b_n=64)
    expected = _oracle_compute(q, k, v, thresholds=thr, layer=1, k_level=4).o
    ctx = mp.get_context("spawn")
    result_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, k, v, thr, expected, result_q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    results = sorted(result_q.get(timeout=10) for _ in range(2))
    for rank, shape, err in results:
        assert shape == (batch, hq, n, d)
        assert err == 0.0, (rank, err)


def test_gather_single_rank_is_identity():
    x = torch.randn(1, 2, 8, 4)
    assert gather_heads(x, 1) is x


def _peer_compute(q, k, v, out=None, o_peers=(), **kw):
    """The epilogue's contract on CPU: O into `out` and byte-identical copies at every peer address."""
    import ctypes
    res = _oracle_compute(q, k, v, **kw)
    out.copy_(res.o)
    for ptr in o_peers:
        ctypes.memmove(ptr, out.data_ptr(), out.numel() * out.element_size())
    return res


def _peer_worker(rank, world, port, bufs, q, k, v, thr, expected, result_q):
    from paper_2512_07011_b200.distributed import PeerGatherBuffer
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pb = PeerGatherBuffer(bufs[rank], [b.data_ptr() for b in bufs], rank, dist.barrier)
        assert pb.peers == [bufs[p].data_ptr() + rank * pb.out.numel() * 4 for p in range(world) if p != rank]
        _, full = sharded_attention(q, k, v, rank=rank, world=world, thresholds=thr, layer=1, k_level=4,
                                    gather="peer", peer_buffer=pb, compute=_peer_compute)
        result_q.put((rank, tuple(full.shape), float((full - expected).abs().max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [1, 2])
def test_two_rank_peer_gather(batch):
    """gather="peer": each rank's rows land in its slot of BOTH ranks' buffers (rank-major layout)."""
    import paper_2512_07011_b200 as bsfa
    rng = np.random.default_rng(10 + batch)
    hq, hkv, n, d = 4, 2, 256, 16
    q = torch.from_numpy(rng.standard_normal((batch, hq, n, d)).astype(np.float32))
    k = torch.from_numpy(rng.standard_normal((batch, hkv, n, d)).astype(np.float32))
    v = torch.from_numpy(rng.standard_normal((batch, hkv, n, d)).astype(np.float32))
    vals = rng.uniform(0.5, 1.0, size=(1, 2, hq, 2)).astype(np.float32)
    thr = bsfa.ThresholdTensor(values=vals, k_levels=(4,), n_max=256, b_m=128, b_n=64)
    expected = _oracle_compute(q, k, v, thresholds=thr, layer=1, k_level=4).o
    bufs = [torch.zeros((2, batch, hq // 2, n, d)).share_memory_() for _ in range(2)]
    ctx = mp.get_context("fork")
    result_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port, bufs, q, k, v, thr, expected, result_q))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    results = sorted(result_q.get(timeout=10) for _ in range(2))
    for rank, shape, err in results:
        assert shape == (batch, hq, n, d)
        assert err == 0.0, (rank, err)


def _oracle_calibrate(dump, k_levels, tiles):
    """CPU stand-in for the GPU calibrate(): the oracle restatement (calibration.py:156-222)."""
    import paper_2512_07011_b200 as bsfa
    from oracle import bsfa_oracle as orc
    samples = [(s.sample_id, np.asarray(s.q), np.asarray(s.k)) for s in dump.samples]
    values, n_max, _ = orc.calibrate(samples, k_levels, tiles.b_m, tiles.b_n)
    return bsfa.ThresholdTensor(values=values, k_levels=tuple(k_levels), n_max=n_max, b_m=tiles.b_m, b_n=tiles.b_n)


def _calib_worker(rank, world, port, dump, result_q):
    import paper_2512_07011_b200 as bsfa
    from paper_2512_07011_b200.distributed import sharded_calibrate
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = sharded_calibrate(dump, [1, 3], bsfa.TileConfig(128, 64), rank=rank, world=world,
                              calibrate_fn=_oracle_calibrate)
        result_q.put((rank, t.values))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_calibration_matches_single_process():
    import paper_2512_07011_b200 as bsfa
    from oracle import bsfa_oracle as orc
    rng = np.random.default_rng(3)
    L, hq, hkv, n, d = 2, 4, 2, 512, 16
    samples = [bsfa.CalibrationSample(sid, orc.round_bf16(rng.standard_normal((L, hq, n, d)).astype(np.float32)),
                                      orc.round_bf16(rng.standard_normal((L, hkv, n, d)).astype(np.float32)))
               for sid in (0, 1)]
    dump = bsfa.CalibrationDump(L, hq, d, samples)
    want = _oracle_calibrate(dump, [1, 3], bsfa.TileConfig(128, 64)).values
    ctx = mp.get_context("spawn")
    result_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_calib_worker, args=(r, 2, port, dump, result_q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    results = sorted((result_q.get(timeout=10) for _ in range(2)), key=lambda x: x[0])
    for rank, values in results:
        np.testing.assert_array_equal(values, want)


def test_sharded_attention_local_shard_needs_full_head_counts():
    """A rank passing only its shard gets its own heads and threshold rows: with the full
    counts given, the shard is used as is; an ambiguous head count raises instead of re-slicing."""
    seen = {}

    def capture(q, k, v, head_offset=0, **kw):
        seen.update(hq=q.shape[1], hkv=k.shape[1], off=head_offset)
        return _Res(q)

    full_q, full_k = torch.zeros(1, 32, 8, 4), torch.zeros(1, 8, 8, 4)
    sharded_attention(full_q[:, 16:], full_k[:, 4:], full_k[:, 4:], rank=1, world=2, compute=capture,
                      heads_q=32, heads_kv=8)
    assert seen == dict(hq=16, hkv=4, off=16)
    sharded_attention(full_q, full_k, full_k, rank=1, world=2, compute=capture)
    assert seen == dict(hq=16, hkv=4, off=16)
    with pytest.raises(ConfigurationError):
        sharded_attention(full_q[:, :8], full_k[:, :2], full_k[:, :2], rank=1, world=2, compute=capture,
                          heads_q=32, heads_kv=8)
    with pytest.raises(ConfigurationError):
        sharded_attention(full_q, full_k, full_k, rank=0, world=2, compute=capture, heads_q=32)
