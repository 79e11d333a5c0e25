"""Generate golden vectors by running the REAL reference package (build container only).

    PYTHONPATH=/root/reference/pkg/src python tools/make_golden.py

The reference (`/root/reference/pkg/src/hrt`, numpy backend) is imported
read-only and driven through its own public API; nothing here is shipped or
run on the GPU box. Outputs go to tests/golden/*.json and pin both
`oracle/hrt_oracle.py` (CPU tests) and the CUDA engine (GPU tests).

Weights follow the BASELINE rule: the reference model is
built, then every parameter is overwritten in `model.params` insertion order
from one `default_rng(seed)` stream (matrices N(0, 0.02), biases 0, LN gain
1). The per-sentence Stage-I cap (SURVEY Fact 1) is injected by wrapping the
reference's own `skip_at_stage(max_steps=...)` parameter; the rest of
`hrt_translate` runs unmodified.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import hrt  # noqa: E402
import hrt.decoding as D  # noqa: E402
from hrt.arena import Workspace  # noqa: E402
from hrt.infer import InferenceSession  # noqa: E402
from hrt.model import ModelConfig, TransformerModel  # noqa: E402

from paper_2212_01543_b200.workload import make_sources, stage1_caps  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")


def fill_params(model, seed, std=0.02):
    rng = np.random.default_rng(seed)
    for name, p in model.params.items():
        if p.data.ndim == 2:
            p.data[...] = rng.normal(0.0, std, size=p.data.shape)
        elif name.endswith(".g"):
            p.data[...] = 1.0
        else:
            p.data[...] = 0.0


def layout(model):
    return [[n, list(p.data.shape), float(np.sum(p.data))] for n, p in model.params.items()]


def translate_capped(session, src, k, b_at, b_nat, cap):
    """Reference hrt_translate with skip_at_stage's own max_steps set to `cap`."""
    orig = D.skip_at_stage
    if cap is not None:
        D.skip_at_stage = lambda s, kk, b, max_steps=None, ws=None: orig(s, kk, b, max_steps=cap, ws=ws)
    try:
        tr = D.hrt_translate(session, src, k, b_at=b_at, b_nat=b_nat, ws=Workspace())
    finally:
        D.skip_at_stage = orig
    return tr


def tr_dict(tr):
    return dict(tokens=[int(t) for t in tr.tokens], skip_at_score=tr.skip_at_score,
                skip_cmlm_score=tr.skip_cmlm_score, score=tr.score,
                decoder_calls=tr.decoder_calls, forced=bool(tr.forced))


def cfg_dict(c):
    return c.to_dict()


def session_vectors(model, src, ids, dtype=np.float64, steps=3, k=2):
    """encode memory, first greedy Stage-I log-prob rows, parallel logits."""
    s = InferenceSession(model, dtype=dtype)
    ws = Workspace()
    mem = s.encode(src, ws).copy()
    cache = s.start_cache(1, steps + 1, ws)
    feed, rows = [hrt.BOS_K[k]], []
    for t in range(steps):
        lp = s.step(cache, feed, t * k)[0].copy()
        rows.append(lp.tolist())
        row = D._allowed_row(lp)
        feed = [int(np.argmax(row))]
    ws2 = Workspace()
    s.encode(src, ws2)
    pos = np.arange(1, len(ids) + 1)[None, :]
    full = s.parallel_logits(np.asarray([ids]), pos, "full", ws2).copy()
    amax, lp = s.argmax_logprobs(full.copy(), exclude=D.EXCLUDED_OUTPUT_IDS)
    causal = s.parallel_logits(np.asarray([ids]), pos, "causal", ws2).copy()
    return dict(src=list(map(int, src)), ids=list(map(int, ids)), memory=mem.tolist(), step_logp=rows,
                step_k=k, parallel_full=full[0].tolist(), parallel_causal=causal[0].tolist(),
                fill_amax=amax[0].tolist(), fill_lp=lp[0].tolist())


def toy_case():
    cfg = ModelConfig(d_model=64, d_ff=128, n_heads=2, enc_layers=2, dec_layers=1, vocab_size=97, max_len=24)
    model = TransformerModel(cfg, seed=0)
    fill_params(model, 11)
    rng = np.random.default_rng(5)
    sources = [rng.integers(7, 97, size=int(n)).tolist() + [2] for n in rng.integers(1, 20, size=6)]
    session = InferenceSession(model, dtype=np.float64)
    runs = []
    for k in (2, 3, 4):
        for (b_at, b_nat) in ((1, 1), (3, 1), (3, 3)):
            for capped in (False, True):
                for si, src in enumerate(sources):
                    cap = stage1_caps([src], k)[0] if capped else None
                    cap = None if cap is None else min(cap, math.ceil(cfg.max_len / k))
                    tr = translate_capped(session, src, k, b_at, b_nat, cap)
                    runs.append(dict(src=si, k=k, b_at=b_at, b_nat=b_nat, max_steps=cap, out=tr_dict(tr)))
    vec = session_vectors(model, sources[0], [3, 20, 3, 31, 3, 2])
    return dict(name="toy", config=cfg_dict(cfg), seed=11, layout=layout(model), sources=sources,
                runs=runs, vectors=vec)


def tiny_trained_case():
    """The reference's own tiny_trained recipe (tests/conftest.py:80-89): natural EOS."""
    from hrt.data import generate_synthetic
    from hrt.training import CurriculumSchedule, train

    corpus = generate_synthetic("copy", 2000, (1, 6), 15, seed=3)
    cfg = ModelConfig(d_model=16, d_ff=64, n_heads=2, enc_layers=1, dec_layers=1, vocab_size=15, max_len=6)
    model = TransformerModel(cfg, seed=5)
    train(model, corpus, CurriculumSchedule(500), steps=500, k=2, batch_size=16, seed=0)
    params = {n: p.data.tolist() for n, p in model.params.items()}
    session = InferenceSession(model, dtype=np.float64)
    rng = np.random.default_rng(17)
    sources = [rng.integers(7, 15, size=int(rng.integers(1, 7))).tolist() for _ in range(24)]
    runs = []
    for k in (2, 3):
        for (b_at, b_nat) in ((1, 1), (4, 1), (4, 4)):
            for si, src in enumerate(sources):
                tr = translate_capped(session, src, k, b_at, b_nat, None)
                runs.append(dict(src=si, k=k, b_at=b_at, b_nat=b_nat, max_steps=None, out=tr_dict(tr)))
    at_runs = []
    for si, src in enumerate(sources[:8]):
        for beam in (1, 3):
            tr = D.at_translate(session, src, beam=beam, ws=Workspace())
            at_runs.append(dict(src=si, beam=beam, out=tr_dict(tr)))
    return dict(name="tiny_trained", config=cfg_dict(cfg), params=params, layout=layout(model),
                sources=sources, runs=runs, at_runs=at_runs)


def dh64_case():
    """d_head = 64 small model for the bf16 tcgen05 path and fp32 parity."""
    cfg = ModelConfig(d_model=128, d_ff=256, n_heads=2, enc_layers=2, dec_layers=1, vocab_size=1000, max_len=64)
    model = TransformerModel(cfg, seed=0)
    fill_params(model, 21)
    sources = make_sources(8, 2021, ("uniform", 3, 40), vocab_size=1000)
    out = dict(name="dh64", config=cfg_dict(cfg), seed=21, layout=layout(model), sources=sources, runs=[])
    for dt in ("f64", "f32"):
        session = InferenceSession(model, dtype=np.float64 if dt == "f64" else np.float32)
        for (k, b_at, b_nat) in ((2, 1, 1), (3, 1, 1), (2, 4, 1), (2, 4, 4)):
            caps = stage1_caps(sources, k)
            for si, src in enumerate(sources):
                tr = translate_capped(session, src, k, b_at, b_nat, caps[si])
                out["runs"].append(dict(dtype=dt, src=si, k=k, b_at=b_at, b_nat=b_nat, max_steps=caps[si],
                                        out=tr_dict(tr)))
    out["vectors"] = session_vectors(model, sources[0], [3, 40, 3, 41, 3, 2])
    return out


def c1_case(n_sent=3):
    """BASELINE config 1 shape (E6D1, d512, V32000), weights seed 0, inputs seed 1000."""
    cfg = ModelConfig(d_model=512, d_ff=2048, n_heads=8, enc_layers=6, dec_layers=1, vocab_size=32000, max_len=256)
    model = TransformerModel(cfg, seed=0)
    fill_params(model, 0)
    sources = make_sources(n_sent, 1000, ("uniform", 8, 64))
    caps = stage1_caps(sources, 2)
    out = dict(name="c1", config=cfg_dict(cfg), seed=0, layout=layout(model), sources=sources, runs=[])
    for dt in ("f64", "f32"):
        session = InferenceSession(model, dtype=np.float64 if dt == "f64" else np.float32)
        for si, src in enumerate(sources):
            tr = translate_capped(session, src, 2, 1, 1, caps[si])
            out["runs"].append(dict(dtype=dt, src=si, k=2, b_at=1, b_nat=1, max_steps=caps[si], out=tr_dict(tr)))
    # top-8 of the first 3 Stage-I log-prob rows of sentence 0, fp64
    s = InferenceSession(model, dtype=np.float64)
    ws = Workspace()
    s.encode(sources[0], ws)
    cache = s.start_cache(1, 4, ws)
    feed, tops = [hrt.BOS_K[2]], []
    for t in range(3):
        lp = s.step(cache, feed, 2 * t)[0]
        order = np.argsort(-lp, kind="stable")[:8]
        tops.append(dict(ids=order.tolist(), logp=lp[order].tolist(), eos=float(lp[2]),
                         lse_check=float(np.log(np.exp(lp).sum()))))
        feed = [int(np.argmax(D._allowed_row(lp)))]
    out["step_top8"] = tops
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    which = sys.argv[1:] or ["toy", "tiny_trained", "dh64", "c1", "ckpt"]
    if "ckpt" in which:
        which.remove("ckpt")
        write_tiny_checkpoint()
    makers = dict(toy=toy_case, tiny_trained=tiny_trained_case, dh64=dh64_case, c1=c1_case)
    for name in which:
        data = makers[name]()
        data["generator"] = "tools/make_golden.py (reference hrt %s, numpy backend=%s)" % (
            hrt.__version__, hrt.backend_name())
        path = os.path.join(OUT, f"{name}.json")
        with open(path, "w") as f:
            json.dump(data, f)
        print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")



def write_tiny_checkpoint():
    """The tiny_trained model saved by the reference's own save_checkpoint
    (HRTCKPT1 fixture for the loader tests) plus its vocabulary file."""
    from hrt.checkpoint import save_checkpoint
    from hrt.data import Vocabulary, save_vocab

    g = json.load(open(os.path.join(OUT, "tiny_trained.json")))
    cfg = ModelConfig.from_dict(g["config"])
    model = TransformerModel(cfg, seed=0)
    for n, p in model.params.items():
        p.data[...] = np.asarray(g["params"][n])
    save_checkpoint(model, os.path.join(OUT, "tiny_trained.ckpt"))
    save_vocab(Vocabulary.synthetic(cfg.vocab_size), os.path.join(OUT, "tiny_vocab.txt"))
    print("wrote tiny_trained.ckpt / tiny_vocab.txt")


if __name__ == "__main__":
    main()
