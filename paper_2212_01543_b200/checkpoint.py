"""HRTCKPT1 weight files (the reference's checkpoint format, checkpoint.py:1-69).

Layout: 8-byte magic "HRTCKPT1", uint32 little-endian JSON-header length,
UTF-8 JSON header {"config": ModelConfig fields, "params": [{"name", "shape"}]},
then every parameter's float64 little-endian values in manifest order (the
reference writes sorted-name order). Loading gives an HRTModel the engine
accepts directly, so models trained with the reference run on the B200 path.
"""

from __future__ import annotations

import json
import struct

import numpy as np

from .model import HRTModel, ModelConfig, ModelError, param_layout

MAGIC = b"HRTCKPT1"


class CheckpointError(RuntimeError):
    """Malformed or incompatible checkpoint (reference checkpoint.py:20)."""


def read_checkpoint(path):
    """(ModelConfig, {name: float64 array}) from an HRTCKPT1 file."""
    with open(path, "rb") as f:
        blob = f.read()
    if blob[:8] != MAGIC:
        raise CheckpointError(f"bad checkpoint magic {blob[:8]!r}")
    (hlen,) = struct.unpack_from("<I", blob, 8)
    try:
        header = json.loads(blob[12: 12 + hlen].decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as ex:
        raise CheckpointError(f"unreadable checkpoint header: {ex}") from None
    cfg = ModelConfig.from_any(header["config"])
    pos = 12 + hlen
    values = {}
    for entry in header["params"]:
        shape = tuple(int(s) for s in entry["shape"])
        count = int(np.prod(shape)) if shape else 1
        end = pos + 8 * count
        if end > len(blob):
            raise CheckpointError(f"truncated checkpoint at {entry['name']}")
        values[entry["name"]] = np.frombuffer(blob, dtype="<f8", count=count, offset=pos).reshape(shape).copy()
        pos = end
    return cfg, values


def load_model(path):
    """HRTModel from an HRTCKPT1 file, validated against the parameter layout."""
    cfg, values = read_checkpoint(path)
    params = {}
    for name, shape in param_layout(cfg):
        if name not in values:
            raise CheckpointError(f"checkpoint missing parameter {name}")
        if tuple(values[name].shape) != tuple(shape):
            raise CheckpointError(f"shape mismatch for {name}: {values[name].shape} vs {shape}")
        params[name] = values[name]
    return HRTModel(cfg, params)


def save_checkpoint(model, path):
    """Write `model` (HRTModel or reference TransformerModel) as HRTCKPT1."""
    cfg = ModelConfig.from_any(model.config)
    arrays = {n: np.asarray(getattr(p, "data", p), dtype=np.float64) for n, p in model.params.items()}
    names = sorted(arrays)
    header = json.dumps({
        "config": {"d_model": cfg.d_model, "d_ff": cfg.d_ff, "n_heads": cfg.n_heads,
                   "enc_layers": cfg.enc_layers, "dec_layers": cfg.dec_layers, "vocab_size": cfg.vocab_size,
                   "max_len": cfg.max_len, "chunk_sizes": list(cfg.chunk_sizes)},
        "params": [{"name": n, "shape": list(arrays[n].shape)} for n in names],
    }).encode()
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<I", len(header)))
        f.write(header)
        for n in names:
            f.write(np.ascontiguousarray(arrays[n], dtype="<f8").tobytes())


__all__ = ["CheckpointError", "read_checkpoint", "load_model", "save_checkpoint", "ModelError"]
