"""Calibration-dump directories (reference calibration.py:225-299) -- CPU checks.

Byte-identical files both ways against the reference's own save_dump /
load_dump when the reference package is mounted; format errors; lazy
(memory-mapped) samples; the GPU-generator writer on the CPU device.
"""
import importlib
import json
import os
import sys

import numpy as np
import pytest
import torch

from paper_2512_07011_b200 import (CalibrationDump, CalibrationSample, FormatError, ConfigurationError,
                                   load_dump, save_dump, write_model_dump)
from paper_2512_07011_b200.workloads import model_dump_layer

REF_SRC = "/root/reference/pkg/src"


def _dump(with_v=(True, False), L=2, H=3, n=40, d=8):
    rng = np.random.default_rng(0)
    samples = []
    for sid, hv in zip((3, 1), with_v):
        q, k = (rng.standard_normal((L, H, n + sid, d)).astype(np.float32) for _ in range(2))
        v = rng.standard_normal((L, H, n + sid, d)).astype(np.float32) if hv else None
        samples.append(CalibrationSample(sample_id=sid, q=q, k=k, v=v))
    return CalibrationDump(num_layers=L, num_heads=H, head_dim=d, samples=samples)


def _files(directory):
    return {name: open(os.path.join(directory, name), "rb").read() for name in sorted(os.listdir(directory))}


def test_round_trip_and_lazy_views(tmp_path):
    dump = _dump()
    save_dump(dump, tmp_path)
    man = json.loads((tmp_path / "manifest.json").read_text())
    assert [e["path"] for e in man["samples"]] == ["sample_0001.bin", "sample_0003.bin"]
    back = load_dump(tmp_path)
    by_id = {s.sample_id: s for s in dump.samples}
    for s in back.samples:
        ref = by_id[s.sample_id]
        assert isinstance(s.q.base, np.memmap) or isinstance(s.q, np.memmap)  # no host copy
        assert np.array_equal(s.q, ref.q) and np.array_equal(s.k, ref.k)
        assert (s.v is None) == (ref.v is None)
        if s.v is not None:
            assert np.array_equal(s.v, ref.v)
    assert load_dump(tmp_path / "manifest.json").num_heads == 3


def test_format_errors(tmp_path):
    save_dump(_dump(), tmp_path)
    blob = tmp_path / "sample_0001.bin"
    blob.write_bytes(blob.read_bytes()[:-4])
    with pytest.raises(FormatError, match="expected"):
        load_dump(tmp_path)
    (tmp_path / "manifest.json").write_text("{not json")
    with pytest.raises(FormatError, match="invalid manifest"):
        load_dump(tmp_path)
    (tmp_path / "manifest.json").write_text(json.dumps({"num_layers": 1, "samples": []}))
    with pytest.raises(FormatError, match="missing field"):
        load_dump(tmp_path)
    gqa = CalibrationDump(num_layers=1, num_heads=4, head_dim=8, samples=[CalibrationSample(
        sample_id=0, q=np.zeros((1, 4, 16, 8), np.float32), k=np.zeros((1, 2, 16, 8), np.float32))])
    with pytest.raises(ConfigurationError, match="GQA"):
        save_dump(gqa, tmp_path / "g")


def test_model_dump_writer_matches_generator(tmp_path):
    write_model_dump(tmp_path, 2, 2, 2, 256, 16, seed=5, sample_offset=7, device="cpu")
    back = load_dump(tmp_path)
    assert [s.sample_id for s in back.samples] == [7, 8]
    for s in back.samples:
        for layer in range(2):
            q, k, v = model_dump_layer(s.sample_id, layer, 2, 2, 256, 16, seed=5, device="cpu", dtype=torch.float32)
            assert np.array_equal(s.q[layer], q.numpy()) and np.array_equal(s.k[layer], k.numpy())
            assert np.array_equal(s.v[layer], v.numpy())


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not mounted (GPU box)")
def test_byte_identical_with_reference(tmp_path):
    sys.path.insert(0, REF_SRC)
    try:
        rcal = importlib.import_module("bsfa.calibration")
    finally:
        sys.path.remove(REF_SRC)
    dump = _dump()
    ref_dump = rcal.CalibrationDump(num_layers=2, num_heads=3, head_dim=8, samples=[
        rcal.CalibrationSample(sample_id=s.sample_id, q=s.q, k=s.k, v=s.v) for s in dump.samples])
    save_dump(dump, tmp_path / "ours")
    rcal.save_dump(ref_dump, tmp_path / "ref")
    assert _files(tmp_path / "ours") == _files(tmp_path / "ref")
    # each side reads the other's files
    theirs = rcal.load_dump(str(tmp_path / "ours"))
    mine = load_dump(tmp_path / "ref")
    for a, b in zip(sorted(theirs.samples, key=lambda s: s.sample_id), sorted(mine.samples, key=lambda s: s.sample_id)):
        assert a.sample_id == b.sample_id and np.array_equal(a.q, b.q) and np.array_equal(a.k, b.k)
