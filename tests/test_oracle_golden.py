"""Pin the CPU oracle against golden vectors produced by the real reference.

The fixtures (tests/golden/*.json) were written by tools/make_golden.py, which
drives the unmodified reference package; here the oracle must reproduce them
at float64 (tokens exact, floats to ~1e-12).
"""

import math

import numpy as np
import pytest

from oracle import hrt_oracle as O


def make_oracle(g, dtype=np.float64):
    c = g["config"]
    cfg = O.Config(**{k: (tuple(v) if k == "chunk_sizes" else v) for k, v in c.items()})
    if "params" in g:
        params = {k: np.asarray(v, dtype=np.float64) for k, v in g["params"].items()}
    else:
        params = O.init_params(cfg, g["seed"])
    return O.Oracle(cfg, params, dtype=dtype), cfg, params


@pytest.mark.parametrize("name", ["toy", "tiny_trained", "dh64", "c1"])
def test_param_layout_matches_reference(golden, name):
    g = golden(name)
    _, cfg, params = make_oracle(g)
    lay = O.param_layout(cfg)
    assert [n for n, _, _ in lay] == [row[0] for row in g["layout"]]
    assert [list(s) for _, s, _ in lay] == [row[1] for row in g["layout"]]
    for (n, _, _), row in zip(lay, g["layout"]):
        assert abs(float(np.sum(params[n])) - row[2]) <= 1e-9 * max(1.0, abs(row[2]))


@pytest.mark.parametrize("name", ["toy", "dh64"])
def test_session_vectors(golden, name):
    g = golden(name)
    orc, cfg, _ = make_oracle(g)
    v = g["vectors"]
    mem = orc.encode(v["src"])
    assert np.abs(mem - np.asarray(v["memory"])).max() < 1e-12
    k = v["step_k"]
    cache = orc.start_cache(1, len(v["step_logp"]) + 1)
    feed = [O.BOS_K[k]]
    for t, ref in enumerate(v["step_logp"]):
        lp = orc.step(cache, feed, t * k)[0]
        assert np.abs(lp - np.asarray(ref)).max() < 1e-11
        feed = [int(np.argmax(O.allowed_row(lp)))]
    pos = np.arange(1, len(v["ids"]) + 1)[None, :]
    full = orc.parallel_logits([v["ids"]], pos, "full")[0]
    assert np.abs(full - np.asarray(v["parallel_full"])).max() < 1e-11
    causal = orc.parallel_logits([v["ids"]], pos, "causal")[0]
    assert np.abs(causal - np.asarray(v["parallel_causal"])).max() < 1e-11
    amax, lp = orc.argmax_logprobs(full[None])
    assert amax[0].tolist() == v["fill_amax"]
    assert np.abs(lp[0] - np.asarray(v["fill_lp"])).max() < 1e-12


def _check_run(orc, g, run):
    src = g["sources"][run["src"]]
    tr = O.hrt_translate(orc, src, run["k"], run["b_at"], run["b_nat"], max_steps=run["max_steps"])
    ref = run["out"]
    assert tr.tokens == ref["tokens"], (run, tr.tokens, ref["tokens"])
    assert tr.decoder_calls == ref["decoder_calls"]
    assert tr.forced == ref["forced"]
    tol = 1e-9 if orc.dtype == np.float64 else 1e-4
    for key in ("skip_at_score", "skip_cmlm_score", "score"):
        assert abs(getattr(tr, key) - ref[key]) <= tol * max(1.0, abs(ref[key])), key


@pytest.mark.parametrize("name", ["toy", "tiny_trained"])
def test_translations(golden, name):
    g = golden(name)
    orc, _, _ = make_oracle(g)
    for run in g["runs"]:
        _check_run(orc, g, run)


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_dh64_translations(golden, dt):
    g = golden("dh64")
    orc, _, _ = make_oracle(g, np.float64 if dt == "f64" else np.float32)
    for run in g["runs"]:
        if run["dtype"] == dt:
            _check_run(orc, g, run)


def test_at_translate_tiny_trained(golden):
    g = golden("tiny_trained")
    orc, _, _ = make_oracle(g)
    for run in g["at_runs"]:
        tr = O.at_translate(orc, g["sources"][run["src"]], beam=run["beam"])
        assert tr.tokens == run["out"]["tokens"]
        assert abs(tr.score - run["out"]["score"]) < 1e-9
        assert tr.decoder_calls == run["out"]["decoder_calls"]


@pytest.mark.slow
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_c1_translations(golden, dt):
    g = golden("c1")
    orc, _, _ = make_oracle(g, np.float64 if dt == "f64" else np.float32)
    for run in g["runs"]:
        if run["dtype"] == dt:
            _check_run(orc, g, run)


def test_c1_step_top8(golden):
    g = golden("c1")
    orc, _, _ = make_oracle(g)
    orc.encode(g["sources"][0])
    cache = orc.start_cache(1, 4)
    feed = [O.BOS_K[2]]
    for t, ref in enumerate(g["step_top8"]):
        lp = orc.step(cache, feed, 2 * t)[0]
        order = np.argsort(-lp, kind="stable")[:8]
        assert order.tolist() == ref["ids"]
        assert np.abs(lp[order] - np.asarray(ref["logp"])).max() < 1e-11
        assert abs(lp[2] - ref["eos"]) < 1e-11
        feed = [int(np.argmax(O.allowed_row(lp)))]


def test_stage2_layout_worked_example():
    # reference tests/test_decoding.py:57-61 layout law
    ids, pos = O.build_stage2_input([10, 11, 12, O.EOS], 2)
    assert ids == [O.MASK, 10, O.MASK, 11, O.MASK, 12, O.MASK, O.EOS]
    assert pos == list(range(1, 9))
    with pytest.raises(O.OracleError):
        O.build_stage2_input([10, 11], 2)


def test_truncate_at_eos_fuzz():
    rng = np.random.default_rng(0)
    for _ in range(1000):
        toks = rng.integers(0, 12, size=rng.integers(0, 20)).tolist()
        out = O.truncate_at_eos(toks)
        assert O.EOS not in out and out == toks[: len(out)]


def test_caps():
    assert O.max_steps_for(36, 2) == math.ceil(math.floor(1.2 * 36 + 10) / 2)
