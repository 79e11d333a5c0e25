"""Seeded synthetic workloads for the BASELINE configs.

The reference publishes no dataset for this path; these generators stand in
for the paper's WMT test sets with the BASELINE's shapes and distributions:

* source ids: truncated Zipf(s=1.1) over ranks 1..31996 mapped to ids
  4..31999 (rank r -> id 3 + r), then EOS=2 appended;
* lengths: uniform (C1, C4) or log-normal with mean 28 (sigma 0.5), clipped
  to [4, 200] (C2, C3, C5);
* per-sentence Stage-I cap: max_steps = ceil(floor(1.2 n + 10) / k), n the
  source length without EOS.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

EOS = 2
ZIPF_S = 1.1
ZIPF_RANKS = 31996  # ids 4..31999


@dataclass(frozen=True)
class ModelShape:
    """HRT model shape (mirrors the reference ModelConfig fields, model.py:25-62)."""

    d_model: int
    d_ff: int
    n_heads: int
    enc_layers: int
    dec_layers: int
    vocab_size: int = 32000
    max_len: int = 256
    chunk_sizes: tuple = (2, 3, 4)


# BASELINE.json configs (weights seeds 0..3; C5 reuses the C2 architecture + seed).
C1 = ModelShape(512, 2048, 8, 6, 1)
C2 = ModelShape(512, 2048, 8, 12, 1)
C3 = ModelShape(512, 2048, 8, 20, 1)
C4 = ModelShape(1024, 4096, 16, 12, 2)
CONFIGS = {
    "c1": dict(shape=C1, seed=0, k=2, beam=1, dtype="f32", lengths=("uniform", 8, 64)),
    "c2": dict(shape=C2, seed=1, k=2, beam=1, dtype="bf16", lengths=("lognormal", 28.0, 0.5)),
    "c3": dict(shape=C3, seed=2, k=3, beam=1, dtype="bf16", lengths=("lognormal", 28.0, 0.5)),
    "c4": dict(shape=C4, seed=3, k=2, beam=4, dtype="bf16", lengths=("uniform", 16, 128)),
    "c5": dict(shape=C2, seed=1, k=2, beam=1, dtype="bf16", lengths=("lognormal", 28.0, 0.5)),
}


def zipf_probs(n_ranks=ZIPF_RANKS, s=ZIPF_S):
    p = np.arange(1, n_ranks + 1, dtype=np.float64) ** (-s)
    return p / p.sum()


_ZIPF = None


def sample_lengths(rng, n, spec):
    kind = spec[0]
    if kind == "uniform":
        return rng.integers(spec[1], spec[2] + 1, size=n)
    if kind == "lognormal":
        mean, sigma = spec[1], spec[2]
        mu = math.log(mean) - sigma * sigma / 2
        x = rng.lognormal(mu, sigma, size=n)
        return np.clip(np.round(x), 4, 200).astype(np.int64)
    raise ValueError(f"unknown length spec {spec!r}")


def make_sources(n_sentences, seed, lengths=("lognormal", 28.0, 0.5), vocab_size=32000):
    """List of source id lists (each ending in EOS)."""
    global _ZIPF
    rng = np.random.default_rng(seed)
    lens = sample_lengths(rng, n_sentences, lengths)
    n_ranks = min(ZIPF_RANKS, vocab_size - 4)
    if _ZIPF is None or len(_ZIPF) != n_ranks:
        _ZIPF = zipf_probs(n_ranks)
    total = int(lens.sum())
    flat = rng.choice(n_ranks, size=total, p=_ZIPF) + 4
    out, o = [], 0
    for n in lens:
        out.append(flat[o : o + n].tolist() + [EOS])
        o += n
    return out


def tmax_for(n_words):
    return int(math.floor(1.2 * n_words + 10))


def max_steps_for(n_words, k):
    return int(math.ceil(tmax_for(n_words) / k))


def stage1_caps(sources, k):
    """Per-sentence Stage-I step caps (source length excludes the trailing EOS)."""
    return [max_steps_for(len(s) - 1, k) for s in sources]
