"""CPU oracle for the HRT inference path.  TEST INFRASTRUCTURE ONLY.

This module is the *checker*: `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s reference / cpu_baseline leg may import it; the product path
(`paper_2212_01543_b200`) never does, and it is never the thing measured for
the GPU arm.

It restates, in plain numpy, the reference's hot path
(`/root/reference/pkg/src/hrt/…`, cited per function below):

* parameter layout and sinusoidal positions       model.py:104-112, :146-181
* the graph-free session (encode / step /
  reorder / parallel_logits / argmax_logprobs)    infer.py:143-418
* LayerNorm / softmax numerics                    kernels.py:22, :30-57
* Stage-I beam search, Stage-II fill, selection   decoding.py:36-302

with one deliberate extension the BASELINE needs (SURVEY.md Fact 1):
`hrt_translate(..., max_steps=...)` forwards a per-sentence Stage-I cap to the
beam search (decoding.py:193 accepts it, decoding.py:261 does not pass it).
With `max_steps=None` the behaviour is exactly the reference's.

Parity pin: `tests/test_oracle_golden.py` checks this module against golden
vectors produced by running the real reference package in the build container
(`tools/make_golden.py`, fixtures under `tests/golden/`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# special ids (data.py:14-17)
PAD, BOS, EOS, MASK = 0, 1, 2, 3
BOS_K = {2: 4, 3: 5, 4: 6}
# ids the decoder may never emit (decoding.py:36)
EXCLUDED_OUTPUT_IDS = (PAD, BOS, MASK) + tuple(BOS_K.values())
LN_EPS = 1e-5  # kernels.py:22
NEG_BIG = -1e9  # additive mask value (infer.py:352, :357)


class OracleError(RuntimeError):
    pass


@dataclass(frozen=True)
class Config:
    """Mirror of ModelConfig (model.py:25-62)."""

    d_model: int = 64
    d_ff: int = 256
    n_heads: int = 4
    enc_layers: int = 4
    dec_layers: int = 1
    vocab_size: int = 71
    max_len: int = 200
    chunk_sizes: tuple = (2, 3, 4)

    @property
    def d_head(self):
        return self.d_model // self.n_heads

    @property
    def pe_rows(self):
        # model.py:124-126 / infer.py:151-153
        return self.max_len + max(self.chunk_sizes) + 1


# ---------------------------------------------------------------------------
# parameters
# ---------------------------------------------------------------------------


def param_layout(cfg: Config):
    """(name, shape, kind) in the reference's insertion order (model.py:146-181).

    kind: "matrix" (2-D weight incl. the tied embedding), "zeros" (bias / LN
    shift), "ones" (LN gain).
    """
    d, f = cfg.d_model, cfg.d_ff
    out = [("embed", (cfg.vocab_size, d), "matrix")]

    def attn(p):
        out.extend((f"{p}.{w}", (d, d), "matrix") for w in ("wq", "wk", "wv", "wo"))
        out.extend((f"{p}.{b}", (d,), "zeros") for b in ("bq", "bk", "bv", "bo"))

    def ln(p):
        out.extend([(f"{p}.g", (d,), "ones"), (f"{p}.b", (d,), "zeros")])

    def ffn(p):
        out.extend([(f"{p}.w1", (d, f), "matrix"), (f"{p}.b1", (f,), "zeros"),
                    (f"{p}.w2", (f, d), "matrix"), (f"{p}.b2", (d,), "zeros")])

    for i in range(cfg.enc_layers):
        ln(f"enc.{i}.ln1"); attn(f"enc.{i}.attn"); ln(f"enc.{i}.ln2"); ffn(f"enc.{i}.ffn")
    ln("enc.final_ln")
    for i in range(cfg.dec_layers):
        ln(f"dec.{i}.ln1"); attn(f"dec.{i}.attn"); ln(f"dec.{i}.ln2")
        attn(f"dec.{i}.cross"); ln(f"dec.{i}.ln3"); ffn(f"dec.{i}.ffn")
    ln("dec.final_ln")
    return out


def init_params(cfg: Config, seed: int, std: float = 0.02):
    """BASELINE init "N(0,0.02) from seed s".

    One `default_rng(seed)` stream, parameters visited in layout order, every
    matrix drawn N(0, std) in float64; biases / LN shifts 0, LN gains 1.
    """
    rng = np.random.default_rng(seed)
    params = {}
    for name, shape, kind in param_layout(cfg):
        if kind == "matrix":
            params[name] = rng.normal(0.0, std, size=shape)
        elif kind == "ones":
            params[name] = np.ones(shape)
        else:
            params[name] = np.zeros(shape)
    return params


def pe_table(n_positions, d_model, dtype=np.float64):
    """Sinusoidal table: sin on even columns, cos on odd (model.py:104-112)."""
    pos = np.arange(n_positions, dtype=np.float64)[:, None]
    i = np.arange(d_model // 2, dtype=np.float64)[None, :]
    ang = pos / np.power(10000.0, 2 * i / d_model)
    t = np.zeros((n_positions, d_model), dtype=np.float64)
    t[:, 0::2] = np.sin(ang)
    t[:, 1::2] = np.cos(ang)
    return t.astype(dtype)


# ---------------------------------------------------------------------------
# numerics (kernels.py:30-57)
# ---------------------------------------------------------------------------


def layer_norm(x, g, b):
    mu = x.mean(axis=-1, keepdims=True)
    var = x.var(axis=-1, keepdims=True)
    inv = 1.0 / np.sqrt(var + LN_EPS)
    return (x - mu) * inv * g + b


def softmax(x):
    e = np.exp(x - x.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def log_softmax(x):
    """Full-row log-softmax the way step() forms it (infer.py:296-301)."""
    z = x - x.max(axis=-1, keepdims=True)
    return z - np.log(np.exp(z).sum(axis=-1, keepdims=True))


# ---------------------------------------------------------------------------
# session
# ---------------------------------------------------------------------------


@dataclass
class Cache:
    """Self-attention K/V of one in-flight causal decode (infer.py:109-124)."""

    beam: int
    cap: int
    keys: list
    values: list
    length: int = 0
    last_position: int | None = None


class Oracle:
    """Forward-only HRT session in float32 or float64 (infer.py:140-418)."""

    def __init__(self, cfg: Config, params: dict, dtype=np.float32):
        self.cfg = cfg
        self.dtype = np.dtype(dtype)
        self.p = {k: np.ascontiguousarray(v, dtype=self.dtype) for k, v in params.items()}
        self.pe = pe_table(cfg.pe_rows, cfg.d_model, self.dtype)
        self.scale = math.sqrt(cfg.d_model)
        self.att_scale = 1.0 / math.sqrt(cfg.d_head)
        self.memory = None
        self.cross_k = []
        self.cross_v = []
        self.decoder_calls = 0

    # -- helpers ------------------------------------------------------------
    def _lin(self, x, prefix, w, b):
        return x @ self.p[f"{prefix}.{w}"] + self.p[f"{prefix}.{b}"]

    def _ln(self, x, prefix):
        return layer_norm(x, self.p[f"{prefix}.g"], self.p[f"{prefix}.b"])

    def _embed(self, ids, positions):
        x = self.p["embed"][np.asarray(ids, dtype=np.int64)]
        x = x * self.dtype.type(self.scale)
        return x + self.pe[np.asarray(positions, dtype=np.int64)]

    def _split(self, x):
        # (..., T, d) -> (..., h, T, dh)
        h, dh = self.cfg.n_heads, self.cfg.d_head
        s = x.shape[:-1] + (h, dh)
        return np.swapaxes(x.reshape(s), -2, -3)

    def _merge(self, x):
        x = np.swapaxes(x, -2, -3)
        return x.reshape(x.shape[:-2] + (self.cfg.d_model,))

    def _attend(self, q, k, v, bias=None):
        sc = (q @ np.swapaxes(k, -1, -2)) * self.dtype.type(self.att_scale)
        if bias is not None:
            sc = sc + bias
        return softmax(sc) @ v

    def _ffn(self, x, prefix):
        hdn = np.maximum(self._lin(x, prefix, "w1", "b1"), 0.0)
        return self._lin(hdn, prefix, "w2", "b2")

    # -- encoder (infer.py:176-221) ----------------------------------------
    def encode(self, src):
        c = self.cfg
        src = np.asarray(src, dtype=np.int64)
        s = len(src)
        if s > c.max_len:
            raise OracleError(f"source length {s} exceeds max_len {c.max_len}")
        x = self._embed(src, np.arange(s))
        for i in range(c.enc_layers):
            pre = f"enc.{i}"
            y = self._ln(x, f"{pre}.ln1")
            q = self._split(self._lin(y, f"{pre}.attn", "wq", "bq"))
            k = self._split(self._lin(y, f"{pre}.attn", "wk", "bk"))
            v = self._split(self._lin(y, f"{pre}.attn", "wv", "bv"))
            x = x + self._lin(self._merge(self._attend(q, k, v)), f"{pre}.attn", "wo", "bo")
            x = x + self._ffn(self._ln(x, f"{pre}.ln2"), f"{pre}.ffn")
        mem = self._ln(x, "enc.final_ln")
        self.memory = mem
        self.cross_k = [self._lin(mem, f"dec.{i}.cross", "wk", "bk") for i in range(c.dec_layers)]
        self.cross_v = [self._lin(mem, f"dec.{i}.cross", "wv", "bv") for i in range(c.dec_layers)]
        return mem

    # -- one decoder layer, shared by the incremental and parallel passes --
    def _decoder_layer(self, i, x, self_kv, self_bias):
        """x: (..., T, d).  self_kv(i, k, v) -> (K, V) keys/values to attend."""
        pre = f"dec.{i}"
        y = self._ln(x, f"{pre}.ln1")
        q = self._lin(y, f"{pre}.attn", "wq", "bq")
        k = self._lin(y, f"{pre}.attn", "wk", "bk")
        v = self._lin(y, f"{pre}.attn", "wv", "bv")
        kk, vv = self_kv(i, k, v)
        ctx = self._attend(self._split(q), self._split(kk), self._split(vv), self_bias)
        x = x + self._lin(self._merge(ctx), f"{pre}.attn", "wo", "bo")
        y = self._ln(x, f"{pre}.ln2")
        q = self._split(self._lin(y, f"{pre}.cross", "wq", "bq"))
        ctx = self._attend(q, self._split(self.cross_k[i]), self._split(self.cross_v[i]))
        x = x + self._lin(self._merge(ctx), f"{pre}.cross", "wo", "bo")
        return x + self._ffn(self._ln(x, f"{pre}.ln3"), f"{pre}.ffn")

    def _logits(self, x):
        return self._ln(x, "dec.final_ln") @ self.p["embed"].T

    # -- incremental causal decoding (infer.py:225-318) --------------------
    def start_cache(self, beam, cap):
        d, n = self.cfg.d_model, self.cfg.dec_layers
        z = lambda: np.zeros((beam, cap, d), dtype=self.dtype)  # noqa: E731
        return Cache(beam, cap, [z() for _ in range(n)], [z() for _ in range(n)])

    def step(self, cache: Cache, tokens, position):
        """Feed one token per beam row at `position`; (beam, V) log-probs."""
        if cache.last_position is not None and position <= cache.last_position:
            raise OracleError("new position must exceed all cached positions")
        t = cache.length
        if t >= cache.cap:
            raise OracleError("decoder cache capacity exceeded")
        x = self._embed(tokens, np.full(cache.beam, position))[:, None, :]  # (beam, 1, d)

        def self_kv(i, k, v):
            cache.keys[i][:, t] = k[:, 0]
            cache.values[i][:, t] = v[:, 0]
            return cache.keys[i][:, : t + 1], cache.values[i][:, : t + 1]

        for i in range(self.cfg.dec_layers):
            x = self._decoder_layer(i, x, self_kv, None)
        logp = log_softmax(self._logits(x[:, 0]))
        cache.length = t + 1
        cache.last_position = position
        self.decoder_calls += 1
        return logp

    def reorder(self, cache: Cache, parents):
        parents = np.asarray(list(parents), dtype=np.int64)
        if np.array_equal(parents, np.arange(cache.beam)):
            return
        t = cache.length
        for i in range(self.cfg.dec_layers):
            cache.keys[i][:, :t] = cache.keys[i][parents, :t]
            cache.values[i][:, :t] = cache.values[i][parents, :t]

    # -- one-shot parallel decoding (infer.py:322-399) ---------------------
    def parallel_logits(self, ids, positions, mode, pad_mask=None):
        ids = np.atleast_2d(np.asarray(ids, dtype=np.int64))
        positions = np.atleast_2d(np.asarray(positions, dtype=np.int64))
        bsz, t = ids.shape
        x = self._embed(ids, positions)
        bias = np.zeros((bsz, 1, t, t), dtype=self.dtype)
        if mode == "causal":
            bias[:, :, np.triu_indices(t, k=1)[0], np.triu_indices(t, k=1)[1]] = NEG_BIG
        elif mode != "full":
            raise OracleError(f"unknown mode {mode!r}")
        if pad_mask is not None:
            keymask = ~np.asarray(pad_mask, dtype=bool)
            bias = bias + np.where(keymask, NEG_BIG, 0.0).astype(self.dtype)[:, None, None, :]
        for i in range(self.cfg.dec_layers):
            x = self._decoder_layer(i, x, lambda _i, k, v: (k, v), bias)
        self.decoder_calls += 1
        return self._logits(x)

    @staticmethod
    def argmax_logprobs(logits, exclude=EXCLUDED_OUTPUT_IDS):
        """Argmax over the allowed set and its renormalised log-prob (infer.py:401-418)."""
        l = np.array(logits, copy=True)
        if exclude is not None:
            l[..., list(exclude)] = NEG_BIG
        amax = np.argmax(l, axis=-1)
        mx = l.max(axis=-1, keepdims=True)
        lp = -np.log(np.exp(l - mx).sum(axis=-1))
        return amax, lp


# ---------------------------------------------------------------------------
# search and selection (decoding.py)
# ---------------------------------------------------------------------------


@dataclass
class Hyp:
    """Partial anchor sequence (decoding.py:39-53)."""

    tokens: list = field(default_factory=list)
    score: float = 0.0
    finished: bool = False
    forced: bool = False
    is_greedy: bool = False
    row: int = 0


@dataclass
class Translation:
    """Result record (decoding.py:56-68)."""

    tokens: list
    skip_at_score: float
    skip_cmlm_score: float
    score: float
    decoder_calls: int
    forced: bool = False
    anchors: list = field(default_factory=list)


def truncate_at_eos(tokens):
    """Prefix strictly before the first EOS (decoding.py:71-76)."""
    tokens = list(tokens)
    return tokens[: tokens.index(EOS)] if EOS in tokens else tokens


def allowed_row(logp_row):
    """fp64 copy with excluded ids at -inf (decoding.py:84-87)."""
    r = np.array(logp_row, dtype=np.float64)
    r[list(EXCLUDED_OUTPUT_IDS)] = -np.inf
    return r


def beam_search(sess: Oracle, bos, interval, beam, max_steps):
    """Causal beam search over grid positions (decoding.py:90-155).

    Returns (finished hypotheses, steps).
    """
    cache = sess.start_cache(beam, max_steps + 1)
    live = [Hyp(is_greedy=True, row=0)]
    finished = []
    steps = 0
    feed = np.full(beam, bos, dtype=np.int64)
    for t in range(max_steps):
        for h in live:
            feed[h.row] = bos if t == 0 else h.tokens[-1]
        logp = sess.step(cache, feed, t * interval)
        steps += 1
        last = t == max_steps - 1
        cands = []  # (score, token, parent, greedy)
        for h in live:
            row = allowed_row(logp[h.row])
            g_tok = int(np.argmax(row))
            picks = [EOS] if last else np.argsort(-row, kind="stable")[: beam + 1]
            for tok in picks:
                tok = int(tok)
                cands.append((h.score + float(row[tok]), tok, h, h.is_greedy and (last or tok == g_tok)))
        cands.sort(key=lambda c: (-c[0], c[1]))

        def child(score, tok, parent, greedy):
            return Hyp(parent.tokens + [tok], score, tok == EOS, last and tok == EOS, greedy)

        new_live, parents = [], []
        for rank, (score, tok, parent, greedy) in enumerate(cands):
            if tok == EOS:
                if rank < beam or greedy:
                    finished.append(child(score, tok, parent, greedy))
            elif len(new_live) < beam:
                new_live.append(child(score, tok, parent, greedy))
                parents.append(parent.row)
        greedy_done = any(h.is_greedy for h in finished)
        if not greedy_done and not any(h.is_greedy for h in new_live):
            gc = next((c for c in cands if c[3] and c[1] != EOS), None)
            if gc is not None and new_live:
                new_live[-1] = child(gc[0], gc[1], gc[2], True)
                parents[-1] = gc[2].row
        if not new_live or (len(finished) >= beam and greedy_done):
            break
        sess.reorder(cache, parents + [0] * (beam - len(parents)))
        for j, h in enumerate(new_live):
            h.row = j
        live = new_live
    return finished, steps


def build_stage2_input(anchors, k):
    """(k-1) MASKs before every anchor; positions 1..k*m (decoding.py:208-217)."""
    anchors = list(anchors)
    if not anchors or anchors[-1] != EOS:
        raise OracleError("stage-II input requires anchors ending with EOS")
    ids = []
    for z in anchors:
        ids += [MASK] * (k - 1) + [z]
    return ids, list(range(1, len(ids) + 1))


def tmax_for(n_src_words):
    """BASELINE target cap floor(1.2*n + 10)."""
    return int(math.floor(1.2 * n_src_words + 10))


def max_steps_for(n_src_words, k):
    return int(math.ceil(tmax_for(n_src_words) / k))


def hrt_translate(sess: Oracle, source, k, b_at=1, b_nat=1, length_penalty=0.6, max_steps=None):
    """Two-stage decode (decoding.py:249-302), with an optional Stage-I cap."""
    if b_nat < 1 or b_at < b_nat:
        raise OracleError("need b_at >= b_nat >= 1")
    c = sess.cfg
    if k not in c.chunk_sizes:
        raise OracleError(f"chunk size k={k} not supported")
    sess.encode(list(source)[: c.max_len])
    if max_steps is None:
        max_steps = math.ceil(c.max_len / k)  # decoding.py:202-203
    finished, steps = beam_search(sess, BOS_K[k], k, b_at, max_steps)
    finished.sort(key=lambda h: -h.score)
    cands = finished[:b_nat]
    greedy = next((h for h in finished if h.is_greedy), None)
    if greedy is not None and not any(h is greedy for h in cands):
        cands[-1] = greedy

    stage2 = [build_stage2_input(h.tokens, k) for h in cands]
    t_max = max(len(s[0]) for s in stage2)
    b = len(cands)
    ids = np.full((b, t_max), PAD, dtype=np.int64)
    pos = np.tile(np.arange(1, t_max + 1, dtype=np.int64), (b, 1))
    pad_mask = np.zeros((b, t_max), dtype=bool)
    for i, (s_ids, _) in enumerate(stage2):
        ids[i, : len(s_ids)] = s_ids
        pad_mask[i, : len(s_ids)] = True
    logits = sess.parallel_logits(ids, pos, "full", pad_mask=pad_mask)
    amax, lp = sess.argmax_logprobs(logits)

    best = None
    for i, (hyp, (s_ids, _)) in enumerate(zip(cands, stage2)):
        filled, s_cmlm = [], 0.0
        for j, tok in enumerate(s_ids):
            if tok == MASK:
                filled.append(int(amax[i, j]))
                s_cmlm += float(lp[i, j])
            else:
                filled.append(tok)
        score = (hyp.score + s_cmlm) / len(s_ids) ** length_penalty
        if best is None or score > best[0]:
            best = (score, hyp, filled, s_cmlm)
    score, hyp, filled, s_cmlm = best
    return Translation(
        tokens=truncate_at_eos(filled)[: c.max_len],
        skip_at_score=hyp.score,
        skip_cmlm_score=s_cmlm,
        score=score,
        decoder_calls=steps + 1,
        forced=hyp.forced,
        anchors=list(hyp.tokens),
    )


def at_translate(sess: Oracle, source, beam=1, length_penalty=0.6, max_len=None):
    """Autoregressive baseline from BOS (decoding.py:163-185)."""
    c = sess.cfg
    sess.encode(list(source)[: c.max_len])
    finished, steps = beam_search(sess, BOS, 1, beam, max_len or c.max_len)
    best = max(finished, key=lambda h: h.score / len(h.tokens) ** length_penalty)
    return Translation(
        tokens=truncate_at_eos(best.tokens),
        skip_at_score=best.score,
        skip_cmlm_score=0.0,
        score=best.score / len(best.tokens) ** length_penalty,
        decoder_calls=steps,
        forced=best.forced,
        anchors=list(best.tokens),
    )


# ---------------------------------------------------------------------------
# parity accounting (SURVEY §8(c) protocol, steps 3-4): teacher-forced
# agreement with top-2 margins. Not part of the reference; built from its
# own pieces -- Stage-I rows come from a causal parallel_logits pass over the
# anchor prefix, which equals incremental `step` (test_acceptance.py:211-231),
# and Stage-II rows from the full pass of decoding.py:268-285.
# ---------------------------------------------------------------------------


def _top2_margin(row):
    """(argmax, top1 - top2) of a logits / log-prob row over the allowed set."""
    r = allowed_row(row)
    i = int(np.argmax(r))
    top1 = r[i]
    r[i] = -np.inf
    return i, float(top1 - r.max())


def greedy_teacher_forced(sess: Oracle, source, k, tokens, max_steps, tie=1e-3):
    """Score an engine's greedy HRT output against the oracle, position by
    position, with the engine's own prefix fed to the oracle (so one flip does
    not cascade). `tokens` is the engine's Translation.tokens.

    Returns counts: s1 / s2 positions compared, agreements, and near-ties
    (positions whose oracle top-2 margin is below `tie`), plus `bad`, the
    disagreements that are NOT near-ties (must be 0 for an exact fp32 path).
    Stage II is compared only when the anchors can be read back from `tokens`
    (no EOS fill truncated the output).
    """
    c = sess.cfg
    out = dict(s1=0, s1_agree=0, s1_ties=0, s2=0, s2_agree=0, s2_ties=0, bad=0)
    sess.encode(list(source)[: c.max_len])
    tokens = list(tokens)
    n = len(tokens)
    complete = (n + 1) % k == 0 and (n + 1) // k <= max_steps
    anchors = tokens[k - 1:: k] + ([EOS] if complete else [])
    if not anchors:
        return out
    m = len(anchors)
    feed = [BOS_K[k]] + anchors[: m - 1]
    logits = sess.parallel_logits([feed], [[t * k for t in range(m)]], "causal")[0]
    for t in range(m):
        if t == max_steps - 1:  # forced EOS at the cap (decoding.py:108)
            continue
        if not complete and t == m - 1 and anchors[t] == EOS:
            continue
        am, margin = _top2_margin(logits[t])
        out["s1"] += 1
        if am == anchors[t]:
            out["s1_agree"] += 1
        elif margin < tie:
            out["s1_ties"] += 1
        else:
            out["bad"] += 1
    if not complete:
        return out
    ids, pos = build_stage2_input(anchors, k)
    logits = sess.parallel_logits([ids], [pos], "full")[0]
    filled = tokens + [EOS]
    for j, tok in enumerate(ids):
        if tok != MASK or j >= len(filled):
            continue
        am, margin = _top2_margin(logits[j])
        out["s2"] += 1
        if am == filled[j]:
            out["s2_agree"] += 1
        elif margin < tie:
            out["s2_ties"] += 1
        else:
            out["bad"] += 1
    return out


def free_running_agreement(a, b):
    """Positional token agreement of two decodes: (agreeing positions, max length)."""
    return sum(x == y for x, y in zip(a, b)), max(len(a), len(b))
