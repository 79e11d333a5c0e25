"""Model description the engine consumes: config, parameter layout, seeded init.

Mirrors the reference's `ModelConfig` fields (model.py:25-62) and parameter
names/shapes/insertion order (model.py:146-181), so a reference
`TransformerModel` (or its HRTCKPT1 checkpoint) can be handed to the engine
as-is. The special ids are the reference's (data.py:14-17).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

PAD, BOS, EOS, MASK = 0, 1, 2, 3
SUPPORTED_K = (2, 3, 4)
BOS_K = {2: 4, 3: 5, 4: 6}
EXCLUDED_OUTPUT_IDS = (PAD, BOS, MASK) + tuple(BOS_K.values())  # decoding.py:36


class ModelError(ValueError):
    """Invalid model description (reference model.py:21)."""


@dataclass(frozen=True)
class ModelConfig:
    d_model: int = 64
    d_ff: int = 256
    n_heads: int = 4
    enc_layers: int = 4
    dec_layers: int = 1
    vocab_size: int = 71
    max_len: int = 200
    chunk_sizes: tuple = SUPPORTED_K

    def __post_init__(self):
        if self.d_model % self.n_heads != 0:
            raise ModelError("d_model must be divisible by n_heads")
        if self.dec_layers < 1:
            raise ModelError("dec_layers must be >= 1")

    @property
    def d_head(self):
        return self.d_model // self.n_heads

    @classmethod
    def from_any(cls, c):
        """Accept this class, the reference ModelConfig, a dict or a ModelShape."""
        if isinstance(c, cls):
            return c
        if isinstance(c, dict):
            d = dict(c)
        else:
            d = {k: getattr(c, k) for k in ("d_model", "d_ff", "n_heads", "enc_layers", "dec_layers",
                                            "vocab_size", "max_len") if hasattr(c, k)}
            if hasattr(c, "chunk_sizes"):
                d["chunk_sizes"] = c.chunk_sizes
        d["chunk_sizes"] = tuple(d.get("chunk_sizes", SUPPORTED_K))
        return cls(**d)


def param_layout(cfg: ModelConfig):
    """[(name, shape)] in the reference insertion order (model.py:146-181)."""
    d, f = cfg.d_model, cfg.d_ff
    out = [("embed", (cfg.vocab_size, d))]

    def ln(p):
        out.extend([(f"{p}.g", (d,)), (f"{p}.b", (d,))])

    def attn(p):
        out.extend((f"{p}.{w}", (d, d)) for w in ("wq", "wk", "wv", "wo"))
        out.extend((f"{p}.{b}", (d,)) for b in ("bq", "bk", "bv", "bo"))

    def ffn(p):
        out.extend([(f"{p}.w1", (d, f)), (f"{p}.b1", (f,)), (f"{p}.w2", (f, d)), (f"{p}.b2", (d,))])

    for i in range(cfg.enc_layers):
        ln(f"enc.{i}.ln1"); attn(f"enc.{i}.attn"); ln(f"enc.{i}.ln2"); ffn(f"enc.{i}.ffn")
    ln("enc.final_ln")
    for i in range(cfg.dec_layers):
        ln(f"dec.{i}.ln1"); attn(f"dec.{i}.attn"); ln(f"dec.{i}.ln2")
        attn(f"dec.{i}.cross"); ln(f"dec.{i}.ln3"); ffn(f"dec.{i}.ffn")
    ln("dec.final_ln")
    return out


def init_params(cfg: ModelConfig, seed: int, std: float = 0.02):
    """BASELINE random init: one default_rng(seed) stream in
    layout order; matrices N(0, std) in float64, biases 0, LN gains 1."""
    rng = np.random.default_rng(seed)
    params = {}
    for name, shape in param_layout(cfg):
        if len(shape) == 2:
            params[name] = rng.normal(0.0, std, size=shape)
        elif name.endswith(".g"):
            params[name] = np.ones(shape)
        else:
            params[name] = np.zeros(shape)
    return params


@dataclass
class HRTModel:
    """Config + float64 parameters (the reference TransformerModel's data)."""

    config: ModelConfig
    params: dict = field(default_factory=dict)

    @classmethod
    def random(cls, cfg, seed, std=0.02):
        cfg = ModelConfig.from_any(cfg)
        return cls(cfg, init_params(cfg, seed, std))


def flat_params(model, dtype=np.float32):
    """Concatenate parameters in layout order (the hrt_create blob)."""
    cfg = ModelConfig.from_any(model.config)
    params = model.params
    parts = []
    for name, shape in param_layout(cfg):
        if name not in params:
            raise ModelError(f"missing parameter {name}")
        p = params[name]
        a = np.asarray(getattr(p, "data", p))
        if tuple(a.shape) != tuple(shape):
            raise ModelError(f"parameter {name} has shape {a.shape}, expected {shape}")
        parts.append(np.ascontiguousarray(a, dtype=dtype).reshape(-1))
    return np.concatenate(parts)
