"""Host-side logic of the drop-in API and the C-ABI boundary (CPU only, no GPU calls)."""

import ctypes
import os
import re
import struct

import numpy as np
import pytest

from conftest import ROOT, load_golden

import paper_2512_07011_b200 as bsfa
from paper_2512_07011_b200 import _lib
from paper_2512_07011_b200.errors import ConfigurationError, FormatError, InvalidInputError


# ------------------------------------------------------------------ C ABI
def _header_symbols():
    text = open(os.path.join(ROOT, "include", "bsfa_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(bsfa_\w+)\s*\(", text, re.M)))


def test_header_declares_binding_symbols():
    assert _header_symbols() == sorted(_lib.EXPORTED_SYMBOLS)


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.load_library()
    for name in _header_symbols():
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value
    assert lib.bsfa_abi_version() == _lib.ABI_VERSION


def test_struct_layout_matches_header():
    # field order in the ctypes mirrors must follow the C declarations
    text = open(os.path.join(ROOT, "include", "bsfa_b200.h")).read()
    for cname, cls in (("bsfa_fwd_args", _lib.FwdArgs), ("bsfa_calib_args", _lib.CalibArgs)):
        body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (cname, cname), text, re.S).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        names = []
        for decl in body.split(";"):
            decl = re.sub(r"\[.*?\]", "", decl).strip()
            if not decl:
                continue
            for part in decl.split(","):
                names.append(re.findall(r"\w+", part)[-1])
        assert names == [f[0] for f in cls._fields_], cname


def test_invalid_arguments_are_rejected_without_touching_the_gpu():
    lib = _lib.load_library()
    a = _lib.FwdArgs()
    a.b_m, a.b_n, a.head_dim = 64, 32, 64
    assert lib.bsfa_fwd(ctypes.byref(a), None) == _lib.BSFA_ERR_INVALID
    assert b"unsupported tiles" in lib.bsfa_last_error()
    a.b_m, a.b_n, a.head_dim = 128, 64, 96
    assert lib.bsfa_fwd(ctypes.byref(a), None) == _lib.BSFA_ERR_INVALID
    c = _lib.CalibArgs()
    c.b_m, c.b_n, c.head_dim, c.heads_q, c.heads_kv, c.seq_len = 128, 64, 64, 2, 1, 200
    assert lib.bsfa_calib_blockmax(ctypes.byref(c), None) == _lib.BSFA_ERR_INVALID
    assert lib.bsfa_calib_finalize(None, None, None, None, None, -1, None) == _lib.BSFA_ERR_INVALID


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(_lib.NativeLibraryError):
        _lib.load_library(str(tmp_path / "nope.so"))


# ------------------------------------------------------------------ geometry
def test_tiling_matches_reference_kats():
    # reference tests/test_tiling.py
    assert list(bsfa.frontier_blocks(3, bsfa.TileConfig(64, 64))) == [3]
    t = bsfa.TileConfig(128, 64)
    assert list(bsfa.frontier_blocks(0, t)) == [0, 1] and list(bsfa.frontier_blocks(5, t)) == [10, 11]
    assert list(bsfa.frontier_blocks(3, bsfa.TileConfig(64, 128))) == [1]
    assert bsfa.off_frontier_count(3, bsfa.TileConfig(64, 128)) == 1
    assert list(bsfa.frontier_blocks(1, t, n=130)) == [2]
    assert bsfa.off_frontier_count(0, t) == 0 and bsfa.off_frontier_count(2, t) == 4
    assert bsfa.frontier_count(2, t) == 2
    assert t.padded_len(130) == 256 and t.padded_len(256) == 256
    assert bsfa.TileConfig(64, 128).padded_len(70) == 128
    for bad in ((96, 64), (0, 64)):
        with pytest.raises(ConfigurationError):
            bsfa.TileConfig(*bad)
    assert bsfa.kernel_supports(t) and bsfa.kernel_supports(bsfa.TileConfig(128, 128))
    assert bsfa.kernel_supports(bsfa.TileConfig(64, 64)) and bsfa.kernel_supports(bsfa.TileConfig(64, 128))
    assert not bsfa.kernel_supports(bsfa.TileConfig(64, 32)) and not bsfa.kernel_supports(bsfa.TileConfig(256, 128))
    assert bsfa.kernel_len(192, bsfa.TileConfig(64, 64)) == 256 and bsfa.kernel_len(200, bsfa.TileConfig(64, 128)) == 256


# ------------------------------------------------------------------ thresholds
def _tensor():
    rng = np.random.default_rng(0)
    values = rng.standard_normal((2, 3, 4, 8)).astype(np.float32)
    values[0, 0, 0, 0] = np.inf
    values[1, 2, 3, 7] = -np.inf
    return bsfa.ThresholdTensor(values=values, k_levels=(4, 16), n_max=1024, b_m=128, b_n=64)


def test_threshold_file_round_trip(tmp_path):
    t = _tensor()
    bsfa.save_thresholds(t, tmp_path / "a.bin")
    u = bsfa.load_thresholds(tmp_path / "a.bin")
    np.testing.assert_array_equal(u.values, t.values)
    assert (u.k_levels, u.n_max, u.b_m, u.b_n) == (t.k_levels, t.n_max, t.b_m, t.b_n)
    bsfa.save_thresholds(u, tmp_path / "b.bin")
    assert (tmp_path / "a.bin").read_bytes() == (tmp_path / "b.bin").read_bytes()


def test_reference_threshold_file_is_read_and_rewritten_byte_identically(tmp_path):
    c = load_golden("calib")
    blob = c["file_bytes"].tobytes()
    (tmp_path / "ref.bin").write_bytes(blob)
    t = bsfa.load_thresholds(tmp_path / "ref.bin")
    np.testing.assert_array_equal(t.values, c["values"])
    assert list(t.k_levels) == [int(x) for x in c["k_levels"]]
    bsfa.save_thresholds(t, tmp_path / "again.bin")
    assert (tmp_path / "again.bin").read_bytes() == blob


def test_threshold_lookup_and_validation():
    t = _tensor()
    ctx = bsfa.GateContext(layer=1, head=2, k_level=16, query_block=100)
    assert bsfa.threshold_lookup(t, ctx) == float(t.values[1, 1, 2, 7])
    assert bsfa.threshold_lookup(t, bsfa.GateContext(k_level=4)) == np.inf
    with pytest.raises(ConfigurationError):
        bsfa.threshold_lookup(t, bsfa.GateContext(layer=5, k_level=4))
    with pytest.raises(ConfigurationError):
        t.level_index(99)
    values = np.zeros((2, 1, 1, 8), dtype=np.float32)
    for kw in (dict(k_levels=(4,), n_max=1024), dict(k_levels=(16, 4), n_max=1024),
               dict(k_levels=(4, 16), n_max=2048)):
        with pytest.raises(ConfigurationError):
            bsfa.ThresholdTensor(values=values, b_m=128, b_n=64, **kw)
    np.testing.assert_array_equal(t.layer_slice(16, 2), t.values[1, 2])


def test_threshold_format_errors(tmp_path):
    t = _tensor()
    bsfa.save_thresholds(t, tmp_path / "t.bin")
    raw = (tmp_path / "t.bin").read_bytes()
    cases = {"magic": b"XXXX" + raw[4:], "version": raw[:4] + struct.pack("<I", 99) + raw[8:],
             "trunc": raw[:-8], "empty": b""}
    for name, blob in cases.items():
        (tmp_path / name).write_bytes(blob)
        with pytest.raises(FormatError):
            bsfa.load_thresholds(tmp_path / name)


# ------------------------------------------------------------------ gates
def test_gate_validation_matches_reference():
    t = bsfa.ThresholdTensor(values=np.zeros((1, 1, 1, 1), dtype=np.float32), k_levels=(4,), n_max=128,
                             b_m=128, b_n=64)
    g = bsfa.threshold_gate(t)
    tiles = bsfa.TileConfig(128, 64)
    with pytest.raises(ConfigurationError):
        g.validate(tiles, bsfa.GateContext())
    with pytest.raises(ConfigurationError):
        g.validate(tiles, bsfa.GateContext(k_level=8))
    with pytest.raises(ConfigurationError):
        g.validate(bsfa.TileConfig(64, 64), bsfa.GateContext(k_level=4))
    g.validate(tiles, bsfa.GateContext(k_level=4))


def test_gate_decide_semantics_are_strict():
    class Tile:
        def __init__(self, m):
            self.s_max = m

    t = bsfa.ThresholdTensor(values=np.full((1, 1, 1, 1), 0.5, dtype=np.float32), k_levels=(1,), n_max=128,
                             b_m=128, b_n=64)
    g = bsfa.threshold_gate(t)
    ctx = bsfa.GateContext(k_level=1)
    assert not g.decide(Tile(0.5), 1, 0, None, ctx, None)
    assert g.decide(Tile(float(np.nextafter(np.float32(0.5), 1))), 1, 0, None, ctx, None)
    assert bsfa.dense_gate().decide(Tile(-100.0), 1, 0, None, ctx, None)
    assert not bsfa.frontier_only_gate().decide(Tile(100.0), 1, 0, None, ctx, None)


def test_unknown_gate_refused_before_any_device_work():
    from paper_2512_07011_b200.gates import kernel_gate_mode

    class RunningMax:
        pass

    with pytest.raises(ConfigurationError):
        kernel_gate_mode(RunningMax())


# ------------------------------------------------------------------ inputs
def test_head_input_validation():
    with pytest.raises(InvalidInputError):
        bsfa.HeadInput(q=np.zeros((2, 2)), k=np.zeros((2, 2)), v=np.zeros((3, 2)))
    with pytest.raises(InvalidInputError):
        bsfa.HeadInput(q=np.zeros(4), k=np.zeros(4), v=np.zeros(4))
    bad = np.zeros((2, 2))
    bad[0, 0] = np.nan
    with pytest.raises(InvalidInputError):
        bsfa.HeadInput(q=bad, k=np.zeros((2, 2)), v=np.zeros((2, 2)))


def test_attention_refuses_cpu_tensors():
    import torch
    x = torch.zeros((1, 1, 128, 64), dtype=torch.bfloat16)
    with pytest.raises(InvalidInputError):
        bsfa.attention(x, x, x)


def test_calibration_argument_validation():
    rng = np.random.default_rng(5)
    s = bsfa.CalibrationSample(0, rng.standard_normal((1, 1, 256, 16)), rng.standard_normal((1, 1, 256, 16)))
    dump = bsfa.CalibrationDump(1, 1, 16, [s])
    tiles = bsfa.TileConfig(128, 64)
    with pytest.raises(ConfigurationError):
        bsfa.calibrate(bsfa.CalibrationDump(1, 1, 16, []), [1], tiles)
    with pytest.raises(ConfigurationError):
        bsfa.calibrate(dump, [], tiles)
    with pytest.raises(ConfigurationError):
        bsfa.calibrate(dump, [4, 2], tiles)
    with pytest.raises(ConfigurationError):
        bsfa.CalibrationDump(2, 1, 16, [s])
    with pytest.raises(InvalidInputError):
        bsfa.CalibrationSample(0, np.zeros((1, 3, 8, 4)), np.zeros((1, 2, 8, 4)))


def test_struct_offsets_match_the_c_compiler(tmp_path):
    """Byte layout of the ctypes mirrors == what a C compiler makes of include/bsfa_b200.h."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    lines = ['#include <stddef.h>', '#include <stdio.h>', '#include "bsfa_b200.h"', "int main(void) {"]
    for cname, cls in (("bsfa_fwd_args", _lib.FwdArgs), ("bsfa_calib_args", _lib.CalibArgs)):
        lines.append(f'  printf("{cname} %zu\\n", sizeof({cname}));')
        for f in cls._fields_:
            lines.append(f'  printf("{cname}.{f[0]} %zu\\n", offsetof({cname}, {f[0]}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    got = dict(line.rsplit(" ", 1) for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                              check=True).stdout.splitlines())
    for cname, cls in (("bsfa_fwd_args", _lib.FwdArgs), ("bsfa_calib_args", _lib.CalibArgs)):
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for f in cls._fields_:
            assert int(got[f"{cname}.{f[0]}"]) == getattr(cls, f[0]).offset, (cname, f[0])


def test_bench_reads_measured_peaks_in_any_layout(tmp_path):
    import json
    import sys
    sys.path.insert(0, ROOT)
    import bench
    for doc in ({"bf16_tflops": 1616.9, "bf16_tflops_sustained": 1390.4},
                {"bf16_dense_tflops": {"burst": 1616.9, "sustained_4s": 1390.4}, "hbm_gbps": 6549.8}):
        f = tmp_path / "peaks.json"
        f.write_text(json.dumps(doc))
        assert bench.measured_peaks(str(f)) == (1616.9, 1390.4, "measured")
    assert bench.measured_peaks(str(tmp_path / "absent.json"))[2] == "fallback"
