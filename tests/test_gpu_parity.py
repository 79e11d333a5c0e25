"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle and
the reference golden vectors.

Tolerances (BASELINE north star): fp32 logits / log-probs within 1e-3
relative to the row's max magnitude; token sequences identical (any mismatch
must sit at a top-2 margin < 1e-3, which none of these fixtures has); scores
within 1e-3 relative. bf16 is reported as a token agreement rate.
"""

import math

import numpy as np
import pytest

from oracle import hrt_oracle as O

pytestmark = pytest.mark.gpu

REL = 1e-3


@pytest.fixture(scope="module")
def hrt():
    import paper_2212_01543_b200 as hrt
    from paper_2212_01543_b200 import build

    build.build(verbose=False)
    return hrt


def _model(hrt, g):
    cfg = hrt.ModelConfig.from_any(g["config"])
    if "params" in g:
        params = {k: np.asarray(v, dtype=np.float64) for k, v in g["params"].items()}
    else:
        params = hrt.init_params(cfg, g["seed"])
    return hrt.HRTModel(cfg, params)


def _oracle(g, model, dtype=np.float64):
    c = g["config"]
    cfg = O.Config(**{k: (tuple(v) if k == "chunk_sizes" else v) for k, v in c.items()})
    return O.Oracle(cfg, model.params, dtype=dtype)


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


@pytest.mark.parametrize("name", ["toy", "dh64"])
def test_protocol_session_vectors(hrt, golden, name):
    g = golden(name)
    model = _model(hrt, g)
    sess = hrt.CudaSession(model, dtype=np.float32, max_beam=4)
    v = g["vectors"]
    mem = sess.encode(v["src"])
    assert _rel(mem, v["memory"]) < REL
    k = v["step_k"]
    cache = sess.start_cache(1, len(v["step_logp"]) + 1)
    feed = [O.BOS_K[k]]
    for t, ref in enumerate(v["step_logp"]):
        lp = sess.step(cache, feed, t * k)[0]
        assert _rel(lp, ref) < REL, t
        feed = [int(np.argmax(O.allowed_row(np.asarray(ref))))]
    pos = np.arange(1, len(v["ids"]) + 1)[None, :]
    full = sess.parallel_logits([v["ids"]], pos, "full")[0]
    assert _rel(full, v["parallel_full"]) < REL
    amax, lp = sess.argmax_logprobs(full[None], exclude=O.EXCLUDED_OUTPUT_IDS)
    assert amax[0].tolist() == v["fill_amax"]
    assert _rel(lp[0], v["fill_lp"]) < REL
    causal = sess.parallel_logits([v["ids"]], pos, "causal")[0]
    assert _rel(causal, v["parallel_causal"]) < REL


def test_protocol_errors(hrt, golden):
    g = golden("toy")
    sess = hrt.CudaSession(_model(hrt, g), dtype=np.float32)
    sess.encode([10, 11, 12, 2])
    cache = sess.start_cache(1, 2)
    sess.step(cache, [4], 2)
    with pytest.raises(hrt.InferenceError):
        sess.step(cache, [7], 2)
    sess.step(cache, [7], 3)
    with pytest.raises(hrt.InferenceError):
        sess.step(cache, [8], 4)
    with pytest.raises(hrt.InferenceError):
        sess.encode(list(range(7, 7 + g["config"]["max_len"] + 1)))


def test_reorder_continues_from_parent_rows(hrt, golden):
    """reference tests/test_infer.py:123-141 on the engine."""
    g = golden("toy")
    sess = hrt.CudaSession(_model(hrt, g), dtype=np.float32, max_beam=4)
    src = [20, 30, 40, 50, 2]
    sess.encode(src)
    cache = sess.start_cache(2, 6)
    sess.step(cache, [1, 1], 0)
    sess.step(cache, [7, 8], 1)
    sess.reorder(cache, [1, 1])
    after = sess.step(cache, [9, 9], 2).copy()
    assert np.abs(after[0] - after[1]).max() == 0.0
    sess.encode(src)
    c2 = sess.start_cache(1, 6)
    sess.step(c2, [1], 0)
    sess.step(c2, [8], 1)
    ref = sess.step(c2, [9], 2)
    assert np.abs(after[0] - ref[0]).max() < 1e-5
    # and against the fp64 oracle's own reorder (infer.py:307-318)
    orc = _oracle(g, _model(hrt, g))
    orc.encode(src)
    oc = orc.start_cache(2, 6)
    orc.step(oc, [1, 1], 0)
    orc.step(oc, [7, 8], 1)
    orc.reorder(oc, [1, 1])
    want = orc.step(oc, [9, 9], 2)
    assert _rel(after, want) < REL


def _check_translation(tr, ref, rel=REL):
    assert tr.tokens == ref["tokens"]
    assert tr.decoder_calls == ref["decoder_calls"]
    assert tr.forced == ref["forced"]
    for key in ("skip_at_score", "skip_cmlm_score", "score"):
        assert abs(getattr(tr, key) - ref[key]) <= rel * max(1.0, abs(ref[key])), key


@pytest.mark.parametrize("name", ["toy", "tiny_trained"])
def test_fused_greedy_matches_golden(hrt, golden, name):
    g = golden(name)
    model = _model(hrt, g)
    runs = [r for r in g["runs"] if r["b_at"] == 1]
    sess = hrt.CudaSession(model, dtype=np.float32, max_sentences=len(g["sources"]))
    for k in sorted({r["k"] for r in runs}):
        for capped in (False, True):
            sel = [r for r in runs if r["k"] == k and (r["max_steps"] is not None) == capped]
            if not sel:
                continue
            srcs = [g["sources"][r["src"]] for r in sel]
            caps = None if not capped else [r["max_steps"] for r in sel]
            out = hrt.hrt_translate_batch(sess, srcs, k, max_steps=caps)
            for tr, r in zip(out, sel):
                _check_translation(tr, r["out"])


@pytest.mark.parametrize("name", ["dh64", "c1"])
def test_fused_greedy_fp32_matches_reference(hrt, golden, name):
    g = golden(name)
    model = _model(hrt, g)
    runs = [r for r in g["runs"] if r["dtype"] == "f32" and r["b_at"] == 1]
    sess = hrt.CudaSession(model, dtype=np.float32, max_sentences=len(g["sources"]))
    for k in sorted({r["k"] for r in runs}):
        sel = [r for r in runs if r["k"] == k]
        out = hrt.hrt_translate_batch(sess, [g["sources"][r["src"]] for r in sel], k,
                                      max_steps=[r["max_steps"] for r in sel])
        for tr, r in zip(out, sel):
            _check_translation(tr, r["out"])
    # the single-sentence drop-in gives the same answers as the batch
    r = runs[0]
    tr = hrt.hrt_translate(sess, g["sources"][r["src"]], r["k"], max_steps=r["max_steps"])
    _check_translation(tr, r["out"])


def test_c1_first_steps_logp(hrt, golden):
    """BASELINE config-1 shape: Stage-I log-prob rows vs the fp64 reference."""
    g = golden("c1")
    sess = hrt.CudaSession(_model(hrt, g), dtype=np.float32)
    sess.encode(g["sources"][0])
    cache = sess.start_cache(1, 4)
    feed = [O.BOS_K[2]]
    for t, ref in enumerate(g["step_top8"]):
        lp = sess.step(cache, feed, 2 * t)[0]
        ids = np.asarray(ref["ids"])
        assert np.abs(lp[ids] - np.asarray(ref["logp"])).max() < REL * max(1.0, abs(ref["logp"][0]))
        assert abs(lp[2] - ref["eos"]) < REL * max(1.0, abs(ref["eos"]))
        feed = [int(ref["ids"][0]) if ref["ids"][0] not in O.EXCLUDED_OUTPUT_IDS else
                int(np.argmax(O.allowed_row(lp)))]


def _beam_runs(g):
    runs, seen = [], set()
    for r in g["runs"]:
        if r["b_at"] == 1 or r.get("dtype", "f32") not in ("f32", "f64"):
            continue
        key = (r["src"], r["k"], r["b_at"], r["b_nat"])
        if key not in seen:
            seen.add(key)
            runs.append(r)
    return runs


@pytest.mark.parametrize("name", ["tiny_trained", "dh64", "toy"])
def test_protocol_beam_matches_golden(hrt, golden, name):
    """Stage-I beam through the session protocol (device step/reorder kernels,
    host-side selection)."""
    from paper_2212_01543_b200 import decoding as PD

    g = golden(name)
    sess = hrt.CudaSession(_model(hrt, g), dtype=np.float32, max_beam=4)
    for r in _beam_runs(g)[::2]:
        tr = PD._protocol_translate(sess, g["sources"][r["src"]], r["k"], r["b_at"], r["b_nat"], 0.6,
                                    r["max_steps"])
        _check_translation(tr, r["out"])


@pytest.mark.parametrize("name", ["tiny_trained", "dh64", "toy"])
def test_fused_beam_matches_golden(hrt, golden, name):
    """Device beam search (b_at > 1) + multi-candidate Stage II (b_nat > 1), one
    fused batch per (k, b_at, b_nat) group."""
    g = golden(name)
    sess = hrt.CudaSession(_model(hrt, g), dtype=np.float32, max_beam=4, max_sentences=len(g["sources"]))
    groups = {}
    for r in _beam_runs(g):
        groups.setdefault((r["k"], r["b_at"], r["b_nat"], r["max_steps"] is None), []).append(r)
    for (k, b_at, b_nat, uncapped), rs in groups.items():
        caps = None if uncapped else [r["max_steps"] for r in rs]
        out = hrt.hrt_translate_batch(sess, [g["sources"][r["src"]] for r in rs], k, b_at, b_nat, max_steps=caps)
        for tr, r in zip(out, rs):
            _check_translation(tr, r["out"])


def test_bf16_token_agreement(hrt, golden):
    g = golden("dh64")
    model = _model(hrt, g)
    sess = hrt.CudaSession(model, dtype="bfloat16", max_sentences=len(g["sources"]))
    runs = [r for r in g["runs"] if r["dtype"] == "f64" and r["b_at"] == 1 and r["k"] == 2]
    out = hrt.hrt_translate_batch(sess, [g["sources"][r["src"]] for r in runs], 2,
                                  max_steps=[r["max_steps"] for r in runs])
    agree = total = 0
    for tr, r in zip(out, runs):
        ref = r["out"]["tokens"]
        total += max(len(ref), len(tr.tokens))
        agree += sum(a == b for a, b in zip(tr.tokens, ref))
        assert tr.decoder_calls == r["out"]["decoder_calls"]
    rate = agree / max(1, total)
    print(f"bf16 token agreement vs fp64 reference: {rate:.4f}")
    assert rate > 0.8


def test_batch_equals_single(hrt, golden):
    """Packed batch decode == per-sentence decode (padding isolation)."""
    g = golden("dh64")
    sess = hrt.CudaSession(_model(hrt, g), dtype=np.float32, max_sentences=8)
    srcs = g["sources"]
    batch = hrt.hrt_translate_batch(sess, srcs, 2)
    for s, b in zip(srcs, batch):
        one = hrt.hrt_translate(sess, s, 2)
        assert one.tokens == b.tokens
        assert abs(one.score - b.score) < 1e-5


def test_bf16_protocol_vectors_close(hrt, golden):
    """bf16 engine (tcgen05 GEMMs + mma.sync attention) tracks the fp64
    reference to bf16 precision on the d_head = 64 fixture."""
    g = golden("dh64")
    sess = hrt.CudaSession(_model(hrt, g), dtype="bfloat16", max_beam=4)
    v = g["vectors"]
    mem = sess.encode(v["src"])
    assert _rel(mem, v["memory"]) < 5e-2
    pos = np.arange(1, len(v["ids"]) + 1)[None, :]
    for mode, key in (("full", "parallel_full"), ("causal", "parallel_causal")):
        got = sess.parallel_logits([v["ids"]], pos, mode)[0]
        assert _rel(got, v[key]) < 5e-2, mode
    cache = sess.start_cache(1, len(v["step_logp"]) + 1)
    feed = [O.BOS_K[v["step_k"]]]
    for t, ref in enumerate(v["step_logp"]):
        lp = sess.step(cache, feed, t * v["step_k"])[0]
        assert _rel(lp, ref) < 5e-2, t
        feed = [int(np.argmax(O.allowed_row(np.asarray(ref))))]


def test_graph_loop_equals_eager(hrt, golden):
    """The captured Stage-I loop (unrolled plain graphs, the default) reproduces
    the step-by-step launch path exactly, for several batch buckets."""
    g = golden("dh64")
    eng = hrt.Engine(_model(hrt, g), dtype="bfloat16", max_sentences=64, max_beam=1)
    from paper_2212_01543_b200 import workload as W

    srcs = W.make_sources(37, 5, ("uniform", 3, 40), vocab_size=1000)
    caps = W.stage1_caps(srcs, 2)
    for n in (1, 5, 37):
        eng.set_option("graphs", 1)
        a = eng.translate_batch(srcs[:n], 2, max_steps=caps[:n])
        eng.set_option("graphs", 0)
        b = eng.translate_batch(srcs[:n], 2, max_steps=caps[:n])
        for x, y in zip(a, b):
            assert x.tokens == y.tokens
            assert x.score == y.score and x.decoder_calls == y.decoder_calls


def test_fused_beam_bf16_graph_equals_eager(hrt, golden):
    g = golden("dh64")
    eng = hrt.Engine(_model(hrt, g), dtype="bfloat16", max_sentences=16, max_beam=4)
    from paper_2212_01543_b200 import workload as W

    srcs = W.make_sources(13, 9, ("uniform", 3, 40), vocab_size=1000)
    caps = W.stage1_caps(srcs, 2)
    for b_at, b_nat in ((4, 1), (4, 4), (2, 2)):
        eng.set_option("graphs", 1)
        a = eng.translate_batch(srcs, 2, b_at, b_nat, max_steps=caps)
        eng.set_option("graphs", 0)
        b = eng.translate_batch(srcs, 2, b_at, b_nat, max_steps=caps)
        for x, y in zip(a, b):
            assert x.tokens == y.tokens and x.score == y.score and x.decoder_calls == y.decoder_calls


def test_splitk_equals_unsplit_and_is_deterministic(hrt, golden):
    """Split-K GEMMs (deterministic last-arriver reduction) change only fp32
    summation order: tokens match the unsplit engine and repeat bit-exactly."""
    g = golden("dh64")
    eng = hrt.Engine(_model(hrt, g), dtype="bfloat16", max_sentences=8, max_beam=4)
    srcs = g["sources"]
    runs = []
    for sk in (1, 1, 0):
        eng.set_option("splitk", sk)
        runs.append(eng.translate_batch(srcs, 2, 4, 2))
    for a, b in zip(runs[0], runs[1]):
        assert a.tokens == b.tokens and a.score == b.score
    agree = sum(x.tokens == y.tokens for x, y in zip(runs[0], runs[2]))
    assert agree >= len(srcs) - 1


def test_checkpoint_model_and_cli_translate(hrt, golden, tmp_path, capsys):
    """HRTCKPT1 (written by the reference) -> engine: greedy and beam outputs
    match the reference goldens; the CLI translate path prints them."""
    import os

    from paper_2212_01543_b200 import checkpoint as CK, cli

    here = os.path.join(os.path.dirname(__file__), "golden")
    m = CK.load_model(os.path.join(here, "tiny_trained.ckpt"))
    g = golden("tiny_trained")
    sess = hrt.CudaSession(m, dtype=np.float32, max_sentences=len(g["sources"]), max_beam=4)
    sel = [r for r in g["runs"] if r["k"] == 2 and r["b_at"] == 4 and r["b_nat"] == 4]
    out = hrt.hrt_translate_batch(sess, [g["sources"][r["src"]] for r in sel], 2, 4, 4)
    for tr, r in zip(out, sel):
        _check_translation(tr, r["out"])
    vocab = [ln.strip() for ln in open(os.path.join(here, "tiny_vocab.txt")) if ln.strip()]
    src = tmp_path / "src.txt"
    greedy = [r for r in g["runs"] if r["k"] == 2 and r["b_at"] == 1]
    src.write_text("\n".join(" ".join(vocab[t] for t in g["sources"][r["src"]]) for r in greedy) + "\n")
    cli.main(["translate", "--checkpoint", os.path.join(here, "tiny_trained.ckpt"), "--vocab",
              os.path.join(here, "tiny_vocab.txt"), "--input", str(src), "--batch", "8"])
    lines = capsys.readouterr().out.strip().split("\n")
    assert lines == [" ".join(vocab[t] for t in r["out"]["tokens"]) for r in greedy]


def _eos_prone_model(hrt, seed=41):
    """d=128 random model whose EOS embedding row points along the (centred)
    positional encoding of position 20, so greedy decodes stop at a natural EOS
    (decoding.py:149-150) around step 10 -- long before the batch's largest
    Stage-I cap (30) -- while the shortest sentences still hit their cap."""
    cfg = hrt.ModelConfig(d_model=128, d_ff=256, n_heads=2, enc_layers=2, dec_layers=1, vocab_size=1000, max_len=64)
    m = hrt.HRTModel.random(cfg, seed)
    u = O.pe_table(70, 128)[20]
    u = u - u.mean()
    m.params["embed"][2] = 0.12 * u / np.linalg.norm(u)
    return cfg, m


def test_natural_eos_graph_early_exit_matches_oracle(hrt):
    """Natural EOS on the captured (unrolled-graph) Stage-I loop: rows finish
    before their cap, the advance kernel drops the live row count to 0 once all
    have finished and the remaining captured steps exit at once. Graph and
    eager runs are bit-identical; the fp32 engine equals the fp64 oracle."""
    from paper_2212_01543_b200 import workload as W

    cfg, model = _eos_prone_model(hrt)
    srcs = W.make_sources(24, 8, ("uniform", 3, 40), vocab_size=1000)
    caps = W.stage1_caps(srcs, 2)
    ocfg = O.Config(128, 256, 2, 2, 1, 1000, 64)
    orc = O.Oracle(ocfg, model.params, dtype=np.float64)
    refs = [O.hrt_translate(orc, s, 2, max_steps=c) for s, c in zip(srcs, caps)]
    natural = sum(not r.forced for r in refs)
    assert natural >= len(srcs) // 2, natural  # the fixture does exercise natural EOS
    f32 = hrt.CudaSession(model, dtype=np.float32, max_sentences=len(srcs))
    for tr, r in zip(hrt.hrt_translate_batch(f32, srcs, 2, max_steps=caps), refs):
        assert tr.tokens == r.tokens and tr.decoder_calls == r.decoder_calls and tr.forced == r.forced
    eng = hrt.Engine(model, dtype="bfloat16", max_sentences=len(srcs), max_beam=4)
    # the captured loop computes only rows up to the last unfinished one: far fewer row-steps
    # than the cap-based schedule (sum of the caps)
    before = eng.stats()["stage1_row_steps"]
    out = eng.translate_batch(srcs, 2, max_steps=caps)
    rows = eng.stats()["stage1_row_steps"] - before
    steps_taken = sum(t.decoder_calls - 1 for t in out)
    assert steps_taken <= rows < 0.8 * sum(caps), (steps_taken, rows, sum(caps))  # measured: 253 vs 413
    for n in (1, 7, 24):  # n = 1: a single row finishes early -> every later step is skipped
        for b_at in (1, 4):
            eng.set_option("graphs", 1)
            a = eng.translate_batch(srcs[:n], 2, b_at, 1, max_steps=caps[:n])
            eng.set_option("graphs", 0)
            b = eng.translate_batch(srcs[:n], 2, b_at, 1, max_steps=caps[:n])
            for x, y in zip(a, b):
                assert x.tokens == y.tokens and x.score == y.score and x.decoder_calls == y.decoder_calls
    eng.set_option("graphs", 1)


def test_while_node_graph_equals_eager(hrt, golden):
    """The conditional WHILE-node Stage-I graph (option graph_unroll=0, the
    first design) reproduces the eager launch path exactly."""
    from paper_2212_01543_b200 import workload as W

    g = golden("dh64")
    eng = hrt.Engine(_model(hrt, g), dtype="bfloat16", max_sentences=40, max_beam=4)
    srcs = W.make_sources(37, 5, ("uniform", 3, 40), vocab_size=1000)
    caps = W.stage1_caps(srcs, 2)
    for b_at in (1, 4):
        eng.set_option("graphs", 0)
        ref = eng.translate_batch(srcs, 2, b_at, 1, max_steps=caps)
        eng.set_option("graphs", 1)
        eng.set_option("graph_unroll", 0)
        got = eng.translate_batch(srcs, 2, b_at, 1, max_steps=caps)
        eng.set_option("graph_unroll", 16)
        for x, y in zip(got, ref):
            assert x.tokens == y.tokens and x.score == y.score and x.decoder_calls == y.decoder_calls


def test_prefill_attention_all_heads_matches_per_head_kernel(hrt, golden):
    """All-heads-per-CTA prefill attention (cp.async + ldmatrix.trans) vs the
    per-head mma.sync kernel: encoder memory and Stage-II logits agree to bf16
    rounding, decoded tokens agree."""
    g = golden("dh64")
    sess = hrt.CudaSession(_model(hrt, g), dtype="bfloat16", max_sentences=8)
    v = g["vectors"]
    pos = np.arange(1, len(v["ids"]) + 1)[None, :]
    res = {}
    for on in (2, 0):
        sess.engine.set_option("attn_heads", on)
        mem = np.array(sess.encode(v["src"]))
        full = np.array(sess.parallel_logits([v["ids"]], pos, "full")[0])
        causal = np.array(sess.parallel_logits([v["ids"]], pos, "causal")[0])
        toks = [t.tokens for t in hrt.hrt_translate_batch(sess, g["sources"], 2)]
        res[on] = (mem, full, causal, toks)
    sess.engine.set_option("attn_heads", 1)
    for a, b in zip(res[2][:3], res[0][:3]):
        assert _rel(a, b) < 2e-2
    agree = sum(x == y for x, y in zip(res[2][3], res[0][3]))
    assert agree >= len(g["sources"]) - 1


def test_small_batch_gemv_paths_match_and_fused_ln_is_exact(hrt):
    """Small-M GEMV path (mma.sync) vs tcgen05 GEMMs: tokens agree (bf16
    summation order differs); the LayerNorm fused into the GEMV prologue feeds
    a bit-identical operand, so fused and unfused runs match exactly."""
    from paper_2212_01543_b200 import workload as W

    cfg = hrt.ModelConfig(d_model=256, d_ff=512, n_heads=4, enc_layers=2, dec_layers=1, vocab_size=2000, max_len=64)
    eng = hrt.Engine(hrt.HRTModel.random(cfg, 5), dtype="bfloat16", max_sentences=8, max_beam=1)
    srcs = W.make_sources(8, 21, ("uniform", 3, 30), vocab_size=2000)
    caps = W.stage1_caps(srcs, 2)
    runs = {}
    for gemv, lnf in ((1, 0), (1, 1), (0, 0)):
        eng.set_option("gemv", gemv)
        eng.set_option("ln_fuse", lnf)
        runs[(gemv, lnf)] = eng.translate_batch(srcs, 2, max_steps=caps)
    eng.set_option("gemv", 1)
    eng.set_option("ln_fuse", 0)
    for a, b in zip(runs[(1, 0)], runs[(1, 1)]):
        assert a.tokens == b.tokens and a.score == b.score
    agree = tot = 0
    for a, b in zip(runs[(1, 0)], runs[(0, 0)]):
        assert a.decoder_calls == b.decoder_calls
        tot += max(len(a.tokens), len(b.tokens))
        agree += sum(x == y for x, y in zip(a.tokens, b.tokens))
    assert agree / tot > 0.95


def test_decode_attention_row_kernel_matches_head_kernel(hrt, golden):
    """CTA-per-row decode attention (all heads, staged K/V) vs the
    warp-per-(row, head) kernel, greedy and beam (history map in use)."""
    g = golden("dh64")
    eng = hrt.Engine(_model(hrt, g), dtype="bfloat16", max_sentences=8, max_beam=4)
    srcs = g["sources"]
    for b_at, b_nat in ((1, 1), (4, 2)):
        res = {}
        for mode in (2, 0):
            eng.set_option("attn_rows", mode)
            res[mode] = eng.translate_batch(srcs, 2, b_at, b_nat)
        eng.set_option("attn_rows", 1)
        agree = sum(a.tokens == b.tokens for a, b in zip(res[2], res[0]))
        assert agree >= len(srcs) - 1, (b_at, agree)
        for a, b in zip(res[2], res[0]):
            assert a.decoder_calls == b.decoder_calls


def test_at_translate_protocol_face_matches_reference(hrt, golden):
    """AT baseline (decoding.py:163-185) driven through the session protocol on
    the CUDA engine: the reference's own AT runs on the trained fixture."""
    import os

    from paper_2212_01543_b200 import checkpoint as CK

    here = os.path.join(os.path.dirname(__file__), "golden")
    g = golden("tiny_trained")
    runs = [r for r in g.get("at_runs", [])]
    if not runs:
        pytest.skip("fixture has no AT runs")
    sess = hrt.CudaSession(CK.load_model(os.path.join(here, "tiny_trained.ckpt")), dtype=np.float32, max_beam=4)
    for r in runs:
        tr = hrt.at_translate(sess, g["sources"][r["src"]], beam=r["beam"])
        assert tr.tokens == r["out"]["tokens"]
        assert abs(tr.score - r["out"]["score"]) <= 1e-3 * max(1.0, abs(r["out"]["score"]))


def test_edge_sources_match_reference(hrt, golden):
    """Edge inputs through the fused face vs the fp64 oracle (decoding.py:249-302):
    an EOS-only source, a source of exactly max_len, one longer than max_len
    (truncated as decoding.py:260 does), Stage-I caps of 1 (forced EOS at the
    first step), mixed caps and the uncapped default, every chunk size k, all in
    one ragged batch; the single-sentence face agrees; an empty batch is []."""
    g = golden("toy")
    model = _model(hrt, g)
    orc = _oracle(g, model)
    L, V = g["config"]["max_len"], g["config"]["vocab_size"]
    rng = np.random.default_rng(11)

    def body(n):
        return [int(x) for x in rng.integers(7, V, n)]

    srcs = [[2], body(L - 1) + [2], body(L + 6) + [2], body(3) + [2], [9, 2]]
    sess = hrt.CudaSession(model, dtype=np.float32, max_sentences=len(srcs))
    for k in g["config"]["chunk_sizes"]:
        for caps in (None, [1] * len(srcs), [1, 3, 2, 5, 4]):
            out = hrt.hrt_translate_batch(sess, srcs, k, max_steps=caps)
            assert len(out) == len(srcs)
            for i, (s, tr) in enumerate(zip(srcs, out)):
                ref = O.hrt_translate(orc, s, k, max_steps=None if caps is None else caps[i])
                assert tr.tokens == ref.tokens, (k, caps, i)
                assert tr.decoder_calls == ref.decoder_calls
                assert tr.forced == ref.forced
                for key in ("skip_at_score", "skip_cmlm_score", "score"):
                    assert abs(getattr(tr, key) - getattr(ref, key)) <= REL * max(1.0, abs(getattr(ref, key))), key
            one = hrt.hrt_translate(sess, srcs[2], k, max_steps=None if caps is None else caps[2])
            assert one.tokens == out[2].tokens and one.score == pytest.approx(out[2].score, rel=1e-6)
    assert hrt.hrt_translate_batch(sess, [], 2) == []
    with pytest.raises(hrt.DecodingError):
        hrt.hrt_translate_batch(sess, srcs, 5)


@pytest.mark.parametrize("b_at,b_nat,B", [(1, 1, 300), (4, 2, 96)])
def test_large_ragged_batch_matches_reference(hrt, golden, b_at, b_nat, B):
    """300 sentences in one fp32 fused call: ragged lengths (EOS-only up to past
    max_len), per-sentence caps from 1 up, so the live-row count crosses every
    row bucket (512 .. 1) and the kernel regimes chosen per bucket (SIMT GEMM,
    fp32 GEMV, row and head attention paths); every sentence must equal the fp64
    oracle's decode of it alone."""
    g = golden("dh64")
    model = _model(hrt, g)
    orc = _oracle(g, model)
    L, V = g["config"]["max_len"], g["config"]["vocab_size"]
    rng = np.random.default_rng(23)
    lens = rng.integers(0, L + 8, B)
    srcs = [[int(x) for x in rng.integers(7, V, n)] + [2] for n in lens]
    caps = [int(c) for c in rng.integers(1, 33, B)]
    sess = hrt.CudaSession(model, dtype=np.float32, max_sentences=B, max_beam=b_at)
    out = hrt.hrt_translate_batch(sess, srcs, 2, b_at, b_nat, max_steps=caps)
    bad = []
    for i, (s, c, tr) in enumerate(zip(srcs, caps, out)):
        ref = O.hrt_translate(orc, s, 2, b_at, b_nat, max_steps=c)
        if tr.tokens != ref.tokens or tr.decoder_calls != ref.decoder_calls or \
                abs(tr.score - ref.score) > REL * max(1.0, abs(ref.score)):
            bad.append(i)
    assert not bad, f"{len(bad)} of {B} sentences differ, first {bad[:5]}"


def test_bf16_c2_shape_large_batch(hrt):
    """C2 shape (E12D1, d512, V32000) at 192 sentences, so the tcgen05 paths the
    benchmark runs are exercised (encoder M ~ 5.6k rows: BN=256 tiles, CTA-pair
    multicast clusters, all-heads prefill attention; Stage I from 192 rows down
    through every bucket). The CTA-pair GEMM is bit-identical to the unpaired
    one; bf16 tokens agree with the (oracle-verified) fp32 engine."""
    from paper_2212_01543_b200 import workload as W

    spec = W.CONFIGS["c2"]
    model = hrt.HRTModel.random(spec["shape"], spec["seed"])
    srcs = W.make_sources(192, 77, spec["lengths"])
    caps = W.stage1_caps(srcs, 2)
    eng = hrt.Engine(model, dtype="bfloat16", max_sentences=len(srcs), max_beam=1)
    a = eng.translate_batch(srcs, 2, max_steps=caps)
    eng.set_option("cluster", 0)
    b = eng.translate_batch(srcs, 2, max_steps=caps)
    for x, y in zip(a, b):
        assert x.tokens == y.tokens and x.score == y.score
    # persistent grids sized to their rounds (option balance) vs the full grid: the units map
    # to other CTAs, the arithmetic of every tile is unchanged, so the results are bit-identical
    eng.set_option("cluster", 1)
    eng.set_option("balance", 0)
    bb = eng.translate_batch(srcs, 2, max_steps=caps)
    eng.set_option("balance", 1)
    for x, y in zip(a, bb):
        assert x.tokens == y.tokens and x.score == y.score
    # clusters of four CTAs sharing each weight tile (a quarter each, multicast), down to
    # 4-row-tile GEMMs so Stage-I / Stage-II / vocabulary launches take them too: same tiles,
    # same MMA order, bit-identical
    eng.set_option("cluster4", 1)
    eng.set_option("cluster4_min_mtiles", 4)
    c4 = eng.translate_batch(srcs, 2, max_steps=caps)
    eng.set_option("cluster4", 0)
    eng.set_option("cluster4_min_mtiles", 32)
    for x, y in zip(a, c4):
        assert x.tokens == y.tokens and x.score == y.score
    # residual + LayerNorm fused into the tcgen05 epilogue (cluster of d / 256 CTAs exchanging
    # row statistics over DSMEM): only the LN summation order differs from GEMM + LN kernel
    eng.set_option("cluster", 1)
    eng.set_option("ln_row", 0)
    eng.set_option("ln_epi", 1)
    e = eng.translate_batch(srcs, 2, max_steps=caps)
    eng.set_option("ln_epi", 0)
    same = sum(p == q for x, y in zip(a, e) for p, q in zip(x.tokens, y.tokens))
    assert same / sum(max(len(x.tokens), len(y.tokens)) for x, y in zip(a, e)) > 0.98
    # the default full-row residual + LayerNorm epilogue (ln_row = 1, one CTA per 128-row block
    # holding all 512 columns) against GEMM + LN kernel: again only the LN summation order differs
    u = eng.translate_batch(srcs, 2, max_steps=caps)
    eng.set_option("ln_row", 1)
    same = sum(p == q for x, y in zip(a, u) for p, q in zip(x.tokens, y.tokens))
    assert same / sum(max(len(x.tokens), len(y.tokens)) for x, y in zip(a, u)) > 0.98
    f32 = hrt.Engine(model, dtype="float32", max_sentences=len(srcs), max_beam=1)
    c = f32.translate_batch(srcs, 2, max_steps=caps)
    agree = total = 0
    for x, y in zip(a, c):
        assert x.decoder_calls == y.decoder_calls
        total += max(len(x.tokens), len(y.tokens))
        agree += sum(p == q for p, q in zip(x.tokens, y.tokens))
    rate = agree / total
    print(f"C2 bf16 vs fp32 token agreement: {rate:.4f}")
    assert rate > 0.9


def test_arena_high_water_and_overflow(hrt, golden):
    """Arena contract (arena.py:38-42, reference tests/test_infer.py:173-183):
    the capacity is the closed-form estimate, no call's phase footprint exceeds
    it, and requests past the capacity raise ArenaOverflowError."""
    g = golden("dh64")
    model = _model(hrt, g)
    sess = hrt.CudaSession(model, dtype=np.float32, max_sentences=4, max_beam=3)
    est = hrt.estimate_max_bytes(model.config, "float32", max_sentences=4, max_beam=3)
    st = sess.engine.stats()
    assert st["arena_bytes"] == est["max"] and st["arena_high_water"] == 0
    rng = np.random.default_rng(3)
    L = g["config"]["max_len"]
    for _ in range(10):
        srcs = [[int(x) for x in rng.integers(7, 1000, int(rng.integers(1, L + 1)))] + [2]
                for _ in range(int(rng.integers(1, 5)))]
        hrt.hrt_translate_batch(sess, srcs, 2, b_at=3, b_nat=2)
    st = sess.engine.stats()
    assert 0 < st["arena_high_water"] <= st["arena_bytes"]
    with pytest.raises(hrt.ArenaOverflowError):
        hrt.hrt_translate_batch(sess, [[9, 2]] * 5, 2)
    small = hrt.CudaSession(model, dtype=np.float32, max_sentences=4, max_src_tokens=16)
    with pytest.raises(hrt.ArenaOverflowError):
        hrt.hrt_translate_batch(small, [list(range(7, 17)) + [2]] * 2, 2)
    assert hrt.hrt_translate_batch(small, [list(range(7, 14)) + [2]] * 2, 2)  # 16 tokens fit
    # out-of-range source ids fail like the reference's np.take (IndexError -> ModelError/ValueError)
    with pytest.raises(ValueError):
        hrt.hrt_translate_batch(sess, [[9, 1000, 2]], 2)
    # a source longer than max_len is truncated (decoding.py:260), also on a one-sentence session
    one = hrt.CudaSession(model, dtype=np.float32)
    long_src = [int(x) for x in rng.integers(7, 1000, L + 20)] + [2]
    a = hrt.hrt_translate(one, long_src, 2)
    b = hrt.hrt_translate(one, long_src[:L], 2)
    assert a.tokens == b.tokens and a.score == b.score


def test_skip_cmlm_fill_matches_reference(hrt, golden):
    """Single-candidate Stage II wrapper (decoding.py:220-239) on the CUDA
    session: fills and their renormalised log-probs vs the fp64 oracle."""
    g = golden("toy")
    model = _model(hrt, g)
    orc = _oracle(g, model)
    sess = hrt.CudaSession(model, dtype=np.float32)
    from paper_2212_01543_b200 import decoding as PD

    for src in g["sources"][:4]:
        for k in (2, 3):
            ref = O.hrt_translate(orc, src, k)  # the reference's default cap, ceil(max_len / k)
            sess.encode(src)
            stage2 = PD.build_stage2_input(ref.anchors, k)
            filled, lps = PD.skip_cmlm_fill(sess, stage2)
            ids, pos = O.build_stage2_input(ref.anchors, k)
            orc.encode(src)
            amax, lp = orc.argmax_logprobs(orc.parallel_logits([ids], [pos], "full"))
            want = [int(amax[0, j]) if t == O.MASK else t for j, t in enumerate(ids)]
            assert filled == want
            want_lp = [float(lp[0, j]) for j, t in enumerate(ids) if t == O.MASK]
            assert np.allclose(lps, want_lp, rtol=REL, atol=REL)
            assert abs(sum(lps) - ref.skip_cmlm_score) <= REL * max(1.0, abs(ref.skip_cmlm_score))


def test_fused_at_matches_reference(hrt, golden):
    """Fused greedy AT baseline (hrt_at_translate_batch: interval 1 from BOS on
    the captured Stage-I loop, no Stage II; decoding.py:163-185) vs the fp64
    oracle's at_translate; bf16 graph replay == bf16 eager launches."""
    from paper_2212_01543_b200 import workload as W

    g = golden("dh64")
    model = _model(hrt, g)
    orc = _oracle(g, model)
    srcs = W.make_sources(12, 31, ("uniform", 3, 40), vocab_size=1000)
    caps = [W.tmax_for(len(s) - 1) for s in srcs]  # the BASELINE target cap, one token per step
    sess = hrt.CudaSession(model, dtype=np.float32, max_sentences=len(srcs))
    out = hrt.at_translate_batch(sess, srcs, max_len=caps)
    for s, c, tr in zip(srcs, caps, out):
        ref = O.at_translate(orc, s, beam=1, max_len=c)
        assert tr.tokens == ref.tokens and tr.decoder_calls == ref.decoder_calls and tr.forced == ref.forced
        assert abs(tr.score - ref.score) <= REL * max(1.0, abs(ref.score))
        assert abs(tr.skip_at_score - ref.skip_at_score) <= REL * max(1.0, abs(ref.skip_at_score))
    one = hrt.at_translate(sess, srcs[3], max_len=caps[3])
    assert one.tokens == out[3].tokens
    eng = hrt.Engine(model, dtype="bfloat16", max_sentences=len(srcs))
    eng.set_option("graphs", 1)
    a = eng.at_translate_batch(srcs, max_steps=caps)
    eng.set_option("graphs", 0)
    b = eng.at_translate_batch(srcs, max_steps=caps)
    for x, y in zip(a, b):
        assert x.tokens == y.tokens and x.score == y.score and x.decoder_calls == y.decoder_calls
    with pytest.raises(hrt.ModelError):
        eng.lib  # noqa: B018 -- the C ABI rejects fused AT beam search
        import ctypes as C

        from paper_2212_01543_b200 import _lib

        o = eng.alloc_outputs(1)
        ho = _lib.HrtTranslateOut(*[o[k].ctypes.data for k in ("tokens", "lens", "scores", "calls", "forced")])
        ids = np.array([9, 2], np.int32)
        eng._check(eng.lib.hrt_at_translate_batch(eng._h, ids.ctypes.data, np.array([2], np.int32).ctypes.data_as(
            C.POINTER(C.c_int32)), 1, 2, 0.6, None, C.byref(ho), 0))


def test_integration_stub_drives_protocol_search(hrt, golden, tmp_path):
    """the ctypes stub a maintainer adds to the reference
    package (hrt/cuda.py) is executed as written against libhrt_b200.so, and
    the protocol-level search (a restatement of the reference's
    decoding.py:90-155 / :249-302 that drives any session object) reproduces
    the reference goldens through it, greedy and beam."""
    import os
    import re
    import sys
    import types

    from paper_2212_01543_b200 import _lib, decoding as PD

    doc = open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# hrt/cuda.py.*?)```", doc, re.S).group(1)
    code = code.replace('C.CDLL("libhrt_b200.so")', f'C.CDLL({_lib.LIB_PATH!r})')
    # the reference package's exception modules, as the stub imports them
    pkg = types.ModuleType("hrt")
    pkg.__path__ = []
    mods = {"infer": ("InferenceError", RuntimeError), "model": ("ModelError", ValueError),
            "decoding": ("DecodingError", ValueError), "arena": ("ArenaOverflowError", MemoryError)}
    saved = {n: sys.modules.get(n) for n in ["hrt"] + [f"hrt.{m}" for m in mods]}
    try:
        sys.modules["hrt"] = pkg
        for m, (cls, base) in mods.items():
            mod = types.ModuleType(f"hrt.{m}")
            setattr(mod, cls, type(cls, (base,), {}))
            sys.modules[f"hrt.{m}"] = mod
        stub = types.ModuleType("hrt.cuda")
        stub.__package__ = "hrt"
        exec(compile(code, "INTEGRATION.md:hrt/cuda.py", "exec"), stub.__dict__)
        g = golden("toy")
        sess = stub.CudaInferenceSession(_model(hrt, g), dtype=0, max_beam=4)
        runs = [r for r in g["runs"] if r.get("dtype", "f32") in ("f32", "f64")][::9]
        assert any(r["b_at"] > 1 for r in runs) and any(r["b_at"] == 1 for r in runs)
        for r in runs:
            tr = PD._protocol_translate(sess, g["sources"][r["src"]], r["k"], r["b_at"], r["b_nat"], 0.6,
                                        r["max_steps"])
            _check_translation(tr, r["out"])
        assert sess.decoder_calls > 0
        with pytest.raises(sys.modules["hrt.infer"].InferenceError):
            sess.start_cache(1, 3)
            sess.step(1, [4], 2)
            sess.step(1, [5], 2)  # non-increasing position (infer.py:244)
    finally:
        for n, m in saved.items():
            if m is None:
                sys.modules.pop(n, None)
            else:
                sys.modules[n] = m


def test_cluster_decode_kernel_matches_per_kernel_path(hrt):
    """Stage-I decoder layers on one 16-CTA cluster (decode_cluster.cuh: DSMEM
    exchange, cluster barriers, bulk-copied weight ring) vs the per-kernel
    chain, at the C2 shape for batches of 1 and 3 rows (row buckets 1 and 4):
    same decoder calls, tokens agree (bf16 summation order only), and graph
    replay equals eager launches; the teacher-forced agreement with the fp64
    oracle stays at the bf16 floor."""
    from paper_2212_01543_b200 import workload as W

    spec = W.CONFIGS["c2"]
    model = hrt.HRTModel.random(spec["shape"], spec["seed"])
    srcs = W.make_sources(6, 4242, spec["lengths"])
    caps = W.stage1_caps(srcs, 2)
    eng = hrt.Engine(model, dtype="bfloat16", max_sentences=4, max_beam=1)
    res = {}
    for mode in (0, 2):
        eng.set_option("cluster_decode", mode)
        for g in (1, 0):
            eng.set_option("graphs", g)
            out = []
            for B in (1, 3):
                for i in range(0, len(srcs), B):
                    out += eng.translate_batch(srcs[i:i + B], 2, max_steps=caps[i:i + B])
            res[(mode, g)] = out
    eng.set_option("graphs", 1)
    eng.set_option("cluster_decode", 1)
    for x, y in zip(res[(2, 1)], res[(2, 0)]):
        assert x.tokens == y.tokens and x.score == y.score
    agree = tot = 0
    for x, y in zip(res[(2, 1)], res[(0, 1)]):
        assert x.decoder_calls == y.decoder_calls
        tot += max(len(x.tokens), len(y.tokens))
        agree += sum(p == q for p, q in zip(x.tokens, y.tokens))
    # free-running: one near-tie flip re-routes the rest of a sentence, so the bar is the
    # teacher-forced agreement with the fp64 oracle below (per-position, no cascade)
    assert agree / tot > 0.85
    sh = spec["shape"]
    orc = O.Oracle(O.Config(sh.d_model, sh.d_ff, sh.n_heads, sh.enc_layers, sh.dec_layers, sh.vocab_size, sh.max_len),
                   model.params, dtype=np.float64)
    tf = dict(s1=0, s1_agree=0, s2=0, s2_agree=0)
    for s, c, x in zip(srcs, caps, res[(2, 1)][: len(srcs)]):
        r = O.greedy_teacher_forced(orc, s, 2, x.tokens, c)
        for k in tf:
            tf[k] += r[k]
    rate = (tf["s1_agree"] + tf["s2_agree"]) / (tf["s1"] + tf["s2"])
    print(f"cluster decode bf16 teacher-forced agreement vs fp64 oracle: {rate:.4f}")
    assert rate > 0.97

