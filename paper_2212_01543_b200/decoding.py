"""Drop-in decoding API (reference decoding.py:31-302) over the CUDA engine.

`hrt_translate(session, source, k, ...)` keeps the reference signature. With a
`CudaSession` it runs the fused device path (`hrt_translate_batch`: encoder,
Stage-I skip-AT greedy or beam loop, Stage-II fill and Eq.(2) selection all on
the GPU). With any other object implementing the session protocol (e.g. the
reference's own session, or a test double) it runs the protocol-level search
below, one decoder call at a time.

Selection semantics (every rule here is the reference's):
* Stage-I scores: full-vocabulary log-softmax, excluded ids only barred from
  selection (decoding.py:84-87); lowest id wins ties (:112-113);
* forced EOS at the step cap (:108, :128); candidates sorted by
  (-score, token), stable (:120); EOS acceptance / greedy reservation /
  loop break (:134-150); reorder padded with row 0 (:151);
* Stage II: (k-1) MASKs per anchor (:208-217), renormalised fill log-probs
  (infer.py:409-418), score (s_at + s_cmlm) / (k m)^alpha (:289), output
  truncate(truncate_at_eos(filled), max_len) (:293).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from .engine import CudaSession, DecodingError
from .model import BOS, BOS_K, EOS, EXCLUDED_OUTPUT_IDS, MASK, PAD

__all__ = [
    "DecodingError", "EXCLUDED_OUTPUT_IDS", "Hypothesis", "Translation", "truncate_at_eos",
    "build_stage2_input", "combined_score", "skip_at_stage", "skip_cmlm_fill", "hrt_translate",
    "hrt_translate_batch", "at_translate", "at_translate_batch", "PositionedSequence",
]


@dataclass
class PositionedSequence:
    ids: list
    positions: list

    def __len__(self):
        return len(self.ids)


@dataclass
class Hypothesis:
    tokens: list = field(default_factory=list)
    positions: list = field(default_factory=list)
    score: float = 0.0
    finished: bool = False
    forced: bool = False
    is_greedy: bool = False
    row: int = 0

    def __post_init__(self):
        if self.finished and (not self.tokens or self.tokens[-1] != EOS):
            raise DecodingError("finished hypothesis must end with [EOS]")


@dataclass
class Translation:
    tokens: list
    skip_at_score: float
    skip_cmlm_score: float
    score: float
    decoder_calls: int
    wall_time: float = 0.0
    forced: bool = False

    def __post_init__(self):
        if any(t in (MASK, PAD, EOS) for t in self.tokens):
            raise DecodingError("translation must not contain special markers")


def truncate_at_eos(tokens):
    tokens = list(tokens)
    return tokens[: tokens.index(EOS)] if EOS in tokens else tokens


_EXCL = np.array(EXCLUDED_OUTPUT_IDS)


def _search(session, bos, interval, beam, max_steps):
    """Protocol-level causal beam search (decoding.py:90-155 semantics)."""
    cache = session.start_cache(beam, max_steps + 1)
    live = [Hypothesis(is_greedy=True, row=0)]
    done = []
    feed = np.full(beam, bos, dtype=np.int64)
    steps = 0
    for t in range(max_steps):
        for h in live:
            feed[h.row] = h.tokens[-1] if t else bos
        logp = session.step(cache, feed, t * interval)
        steps += 1
        at = (t + 1) * interval
        final = t == max_steps - 1
        rows = np.asarray(logp, dtype=np.float64)[[h.row for h in live]]
        rows[:, _EXCL] = -np.inf
        pool = []
        for h, row in zip(live, rows):
            top = int(np.argmax(row))
            picks = [EOS] if final else np.argsort(-row, kind="stable")[: beam + 1].tolist()
            pool.extend((h.score + float(row[p]), int(p), h, h.is_greedy and (final or p == top)) for p in picks)
        pool.sort(key=lambda c: (-c[0], c[1]))

        def grow(c):
            sc, tok, par, g = c
            return Hypothesis(par.tokens + [tok], par.positions + [at], sc, tok == EOS, final and tok == EOS, g)

        nxt, parents = [], []
        for rank, c in enumerate(pool):
            if c[1] == EOS:
                if rank < beam or c[3]:
                    done.append(grow(c))
            elif len(nxt) < beam:
                nxt.append(grow(c))
                parents.append(c[2].row)
        greedy_done = any(h.is_greedy for h in done)
        if not greedy_done and not any(h.is_greedy for h in nxt):
            keep = next((c for c in pool if c[3] and c[1] != EOS), None)
            if keep is not None and nxt:
                nxt[-1] = grow(keep)
                parents[-1] = keep[2].row
        if not nxt or (len(done) >= beam and greedy_done):
            break
        session.reorder(cache, parents + [0] * (beam - len(parents)))
        for j, h in enumerate(nxt):
            h.row = j
        live = nxt
    return done, steps


def skip_at_stage(session, k, b_at, max_steps=None, ws=None):
    if k not in session.config.chunk_sizes:
        raise DecodingError(f"chunk size k={k} not supported by the model")
    if max_steps is None:
        max_steps = math.ceil(session.config.max_len / k)
    return _search(session, BOS_K[k], k, b_at, max_steps)


def build_stage2_input(anchors, k):
    anchors = list(anchors)
    if not anchors or anchors[-1] != EOS:
        raise DecodingError("stage-II input requires anchors ending with [EOS]")
    ids = [tok for z in anchors for tok in ([MASK] * (k - 1) + [z])]
    return PositionedSequence(ids, list(range(1, len(ids) + 1)))


def skip_cmlm_fill(session, stage2_input, ws=None):
    ids = np.asarray(stage2_input.ids, dtype=np.int64)[None, :]
    pos = np.asarray(stage2_input.positions, dtype=np.int64)[None, :]
    logits = session.parallel_logits(ids, pos, "full", ws)
    amax, lp = session.argmax_logprobs(logits, exclude=EXCLUDED_OUTPUT_IDS)
    filled, lps = [], []
    for j, tok in enumerate(stage2_input.ids):
        if tok == MASK:
            filled.append(int(amax[0, j]))
            lps.append(float(lp[0, j]))
        else:
            filled.append(tok)
    return filled, lps


def combined_score(hypothesis, fill_log_probs, k, length_penalty=0.6):
    m = len(hypothesis.tokens)
    return (hypothesis.score + float(sum(fill_log_probs))) / (k * m) ** length_penalty


def _protocol_translate(session, source, k, b_at, b_nat, length_penalty, max_steps):
    c = session.config
    session.encode(list(source)[: c.max_len])
    done, steps = skip_at_stage(session, k, b_at, max_steps=max_steps)
    done.sort(key=lambda h: -h.score)
    cands = done[:b_nat]
    greedy = next((h for h in done if h.is_greedy), None)
    if greedy is not None and all(h is not greedy for h in cands):
        cands[-1] = greedy
    stage2 = [build_stage2_input(h.tokens, k) for h in cands]
    width = max(len(s) for s in stage2)
    ids = np.full((len(cands), width), PAD, dtype=np.int64)
    real = np.zeros((len(cands), width), dtype=bool)
    for i, s in enumerate(stage2):
        ids[i, : len(s)] = s.ids
        real[i, : len(s)] = True
    pos = np.tile(np.arange(1, width + 1, dtype=np.int64), (len(cands), 1))
    logits = session.parallel_logits(ids, pos, "full", pad_mask=real)
    amax, lp = session.argmax_logprobs(logits, exclude=EXCLUDED_OUTPUT_IDS)
    best = None
    for i, (h, s) in enumerate(zip(cands, stage2)):
        is_mask = np.asarray(s.ids) == MASK
        filled = np.where(is_mask, amax[i, : len(s)], np.asarray(s.ids)).tolist()
        cmlm = 0.0
        for j in np.nonzero(is_mask)[0]:
            cmlm += float(lp[i, j])
        score = (h.score + cmlm) / len(s) ** length_penalty
        if best is None or score > best[0]:
            best = (score, h, filled, cmlm)
    score, h, filled, cmlm = best
    return Translation(tokens=truncate_at_eos(filled)[: c.max_len], skip_at_score=h.score, skip_cmlm_score=cmlm,
                       score=score, decoder_calls=steps + 1, forced=h.forced)


def hrt_translate(session, source, k, b_at=1, b_nat=1, length_penalty=0.6, ws=None, max_steps=None):
    """Two-stage decode of one sentence (decoding.py:249-302).

    `max_steps` caps Stage I (the reference's skip_at_stage parameter); None
    keeps the reference default ceil(max_len / k).
    """
    if b_nat < 1 or b_at < b_nat:
        raise DecodingError("need b_at >= b_nat >= 1")
    if k not in session.config.chunk_sizes:
        raise DecodingError(f"chunk size k={k} not supported by the model")
    t0 = time.perf_counter()
    if isinstance(session, CudaSession):
        ms = None if max_steps is None else [int(max_steps)]
        tr = session.translate_batch([list(source)], k, b_at, b_nat, length_penalty, ms)[0]
    else:
        tr = _protocol_translate(session, source, k, b_at, b_nat, length_penalty, max_steps)
    tr.wall_time = time.perf_counter() - t0
    return tr


def hrt_translate_batch(session, sources, k, b_at=1, b_nat=1, length_penalty=0.6, max_steps=None):
    """Batched hrt_translate: one fused device call for the whole batch."""
    if b_nat < 1 or b_at < b_nat:
        raise DecodingError("need b_at >= b_nat >= 1")
    if isinstance(session, CudaSession):
        return session.translate_batch(list(map(list, sources)), k, b_at, b_nat, length_penalty, max_steps)
    caps = [None] * len(sources) if max_steps is None else list(max_steps)
    return [hrt_translate(session, s, k, b_at, b_nat, length_penalty, max_steps=m) for s, m in zip(sources, caps)]


def at_translate_batch(session, sources, length_penalty=0.6, max_len=None):
    """Batched greedy AT baseline: one fused device call with a CudaSession.
    `max_len` is one cap for all sentences or a per-sentence list."""
    caps = None
    if max_len is not None:
        caps = list(max_len) if hasattr(max_len, "__len__") else [int(max_len)] * len(sources)
    if isinstance(session, CudaSession):
        return session.at_translate_batch(list(map(list, sources)), length_penalty, caps)
    caps = caps or [None] * len(sources)
    return [at_translate(session, s, 1, length_penalty, m) for s, m in zip(sources, caps)]


def at_translate(session, source, beam=1, length_penalty=0.6, max_len=None, ws=None):
    """Autoregressive baseline from BOS over the same kernels (decoding.py:163-185).
    Greedy (beam 1) on a CudaSession runs the fused device path; beam search
    runs the protocol-level search below."""
    if beam < 1:
        raise DecodingError("beam must be >= 1")
    t0 = time.perf_counter()
    max_len = max_len or session.config.max_len
    if isinstance(session, CudaSession) and beam == 1:  # fused greedy AT on the captured loop
        tr = session.at_translate_batch([list(source)], length_penalty, [int(max_len)])[0]
        tr.wall_time = time.perf_counter() - t0
        return tr
    session.encode(list(source)[: session.config.max_len])
    done, steps = _search(session, BOS, 1, beam, max_len)
    best = max(done, key=lambda h: h.score / len(h.tokens) ** length_penalty)
    return Translation(tokens=truncate_at_eos(best.tokens), skip_at_score=best.score, skip_cmlm_score=0.0,
                       score=best.score / len(best.tokens) ** length_penalty, decoder_calls=steps,
                       wall_time=time.perf_counter() - t0, forced=best.forced)
