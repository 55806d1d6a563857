"""Calibration-dump directories in the reference's disk format, streamed to the GPU.

Format (reference pkg/src/bsfa/calibration.py:225-299): a directory with
``manifest.json``::

    {"head_dim": d, "num_heads": H, "num_layers": L,
     "samples": [{"has_v": true, "id": 0, "path": "sample_0000.bin", "seq_len": N}, ...]}

(``json.dump(indent=2, sort_keys=True)`` plus a trailing newline) and one raw
little-endian float32 blob per sample in layout [layer][head][tensor: Q=0,
K=1, V=2 if present][row][col].

Differences from the reference are only in residency: ``load_dump`` maps the
blobs (``np.memmap``) instead of reading them, so :func:`calibrate` streams one
(sample, layer) slice at a time to the device -- a Llama-scale sample (16 GiB
per tensor at 32K) never has to fit in host memory; ``write_model_dump`` fills
a dump from the GPU generator (``workloads.model_dump_layer``) layer by layer.
Files written here are byte-identical to the reference's ``save_dump`` output
for the same arrays.
"""

from __future__ import annotations

import json
import os

import numpy as np

from .calibration import CalibrationDump, CalibrationSample
from .errors import ConfigurationError, FormatError

MANIFEST_NAME = "manifest.json"


def _blob_name(sample_id: int) -> str:
    return f"sample_{sample_id:04d}.bin"


def _write_manifest(directory, num_layers: int, num_heads: int, head_dim: int, entries) -> str:
    manifest = {"num_layers": num_layers, "num_heads": num_heads, "head_dim": head_dim, "samples": entries}
    path = os.path.join(directory, MANIFEST_NAME)
    with open(path, "w", encoding="utf-8") as f:
        json.dump(manifest, f, indent=2, sort_keys=True)
        f.write("\n")
    return path


def _host(x) -> np.ndarray:
    if hasattr(x, "detach"):
        x = x.detach().float().cpu().numpy()
    return np.asarray(x)


def save_dump(dump: CalibrationDump, directory) -> str:
    """Write ``dump`` (calibration.py:235-257); returns the manifest path.

    Each layer is written in place, so a sample is never stacked into a second
    host copy.
    """
    os.makedirs(directory, exist_ok=True)
    entries = []
    for s in sorted(dump.samples, key=lambda s: s.sample_id):
        if tuple(s.k.shape) != tuple(s.q.shape):
            raise ConfigurationError(
                f"sample {s.sample_id}: the dump format stores one head count; GQA-shaped k "
                f"{tuple(s.k.shape)} vs q {tuple(s.q.shape)} is not representable")
        name = _blob_name(s.sample_id)
        has_v = s.v is not None
        parts = [s.q, s.k] + ([s.v] if has_v else [])
        L, H, n, d = s.q.shape
        out = np.memmap(os.path.join(directory, name), dtype="<f4", mode="w+", shape=(L, H, len(parts), n, d))
        for layer in range(L):
            for t, part in enumerate(parts):
                out[layer, :, t] = _host(part[layer])
        out.flush()
        del out
        entries.append({"id": s.sample_id, "seq_len": s.seq_len, "path": name, "has_v": has_v})
    return _write_manifest(directory, dump.num_layers, dump.num_heads, dump.head_dim, entries)


def load_dump(directory) -> CalibrationDump:
    """Map a dump directory (or its manifest path) (calibration.py:260-299).

    The returned samples hold read-only ``np.memmap`` views; :func:`calibrate`
    uploads them one (sample, layer) at a time.
    """
    path = directory
    if os.path.isdir(path):
        path = os.path.join(path, MANIFEST_NAME)
    with open(path, "r", encoding="utf-8") as f:
        try:
            manifest = json.load(f)
        except json.JSONDecodeError as e:
            raise FormatError(f"{path}: invalid manifest JSON: {e}") from e
    try:
        num_layers = int(manifest["num_layers"])
        num_heads = int(manifest["num_heads"])
        head_dim = int(manifest["head_dim"])
        entries = manifest["samples"]
    except (KeyError, TypeError) as e:
        raise FormatError(f"{path}: manifest missing field: {e}") from e
    base = os.path.dirname(path)
    samples = []
    for e in entries:
        n = int(e["seq_len"])
        t = 3 if e["has_v"] else 2
        blob_path = os.path.join(base, e["path"])
        count = num_layers * num_heads * t * n * head_dim
        size = os.path.getsize(blob_path)
        if size != 4 * count:
            raise FormatError(f"{blob_path}: expected {count} float32 values, found {size // 4}")
        blob = np.memmap(blob_path, dtype="<f4", mode="r", shape=(num_layers, num_heads, t, n, head_dim))
        samples.append(CalibrationSample(sample_id=int(e["id"]), q=blob[:, :, 0], k=blob[:, :, 1],
                                         v=blob[:, :, 2] if t == 3 else None))
    return CalibrationDump(num_layers=num_layers, num_heads=num_heads, head_dim=head_dim, samples=samples)


def write_model_dump(directory, num_samples: int, layers: int, heads: int, n: int, d: int, *, seed: int = 0,
                     sample_offset: int = 0, include_v: bool = True, device=None) -> str:
    """A model-dump-style calibration set (structured / random heads, reference
    workloads.py:193-216 distribution) generated on ``device`` and written one
    layer at a time in the reference dump format.  Returns the manifest path.
    """
    from .workloads import model_dump_layer
    import torch

    os.makedirs(directory, exist_ok=True)
    t = 3 if include_v else 2
    entries = []
    for s in range(sample_offset, sample_offset + num_samples):
        name = _blob_name(s)
        out = np.memmap(os.path.join(directory, name), dtype="<f4", mode="w+", shape=(layers, heads, t, n, d))
        for layer in range(layers):
            parts = model_dump_layer(s, layer, heads, heads, n, d, seed=seed, device=device, dtype=torch.float32,
                                     with_v=include_v)
            for ti, part in enumerate(parts[:t]):
                out[layer, :, ti] = part.cpu().numpy()
        out.flush()
        del out
        entries.append({"id": s, "seq_len": n, "path": name, "has_v": include_v})
    return _write_manifest(directory, layers, heads, d, entries)
