"""CPU-side checks: the C ABI library loads and exports every declared symbol,
host logic (layout, init, workload, schedule) matches the oracle, and the
product-side search/selection logic reproduces the oracle when it drives a
numpy session (no GPU)."""

import math
import re
import os

import numpy as np
import pytest

import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import _lib, build, decoding as PD, workload as W
from oracle import hrt_oracle as O

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib_path():
    return build.build(verbose=False)


def test_header_symbols_are_exported(lib_path):
    hdr = open(os.path.join(REPO, "include", "hrt_b200.h")).read()
    declared = set(re.findall(r"\b(hrt_[a-z_]+)\s*\(", hdr))
    assert declared == set(_lib.EXPORTED)
    assert set(_lib.exported_symbols(lib_path)) == declared


def test_param_count_matches_layout(lib_path):
    lib = _lib.load(lib_path)
    import ctypes as C

    for shape in (W.C1, W.C2, W.C4, hrt.ModelConfig(d_model=16, d_ff=64, n_heads=2, enc_layers=1, vocab_size=15,
                                                   max_len=6)):
        cfg = hrt.ModelConfig.from_any(shape)
        c = _lib.HrtConfig(cfg.d_model, cfg.d_ff, cfg.n_heads, cfg.enc_layers, cfg.dec_layers, cfg.vocab_size,
                           cfg.max_len, 4, 1, 1, 1, 0)
        n = lib.hrt_param_count(C.byref(c))
        assert n == sum(int(np.prod(s)) for _, s in hrt.param_layout(cfg))
    # BASELINE parameter totals
    assert sum(int(np.prod(s)) for _, s in hrt.param_layout(hrt.ModelConfig.from_any(W.C1))) == 39_504_384
    assert sum(int(np.prod(s)) for _, s in hrt.param_layout(hrt.ModelConfig.from_any(W.C2))) == 58_418_688
    assert sum(int(np.prod(s)) for _, s in hrt.param_layout(hrt.ModelConfig.from_any(W.C4))) == 217_520_128


def test_layout_and_init_match_oracle():
    cfg = hrt.ModelConfig(d_model=64, d_ff=128, n_heads=2, enc_layers=2, dec_layers=2, vocab_size=97, max_len=24)
    ocfg = O.Config(64, 128, 2, 2, 2, 97, 24)
    assert [(n, tuple(s)) for n, s in hrt.param_layout(cfg)] == [(n, tuple(s)) for n, s, _ in O.param_layout(ocfg)]
    a, b = hrt.init_params(cfg, 3), O.init_params(ocfg, 3)
    assert all(np.array_equal(a[k], b[k]) for k in a)


def test_flat_params_order_and_shape_checks():
    cfg = hrt.ModelConfig(d_model=16, d_ff=32, n_heads=2, enc_layers=1, vocab_size=15, max_len=6)
    m = hrt.HRTModel.random(cfg, 1)
    blob = hrt.model.flat_params(m)
    assert blob.dtype == np.float32 and blob.size == sum(int(np.prod(s)) for _, s in hrt.param_layout(cfg))
    assert np.array_equal(blob[: 15 * 16], m.params["embed"].astype(np.float32).reshape(-1))
    bad = hrt.HRTModel(cfg, dict(m.params, embed=np.zeros((3, 3))))
    with pytest.raises(hrt.ModelError):
        hrt.model.flat_params(bad)


def test_workload_generators():
    a = W.make_sources(200, 1000, ("uniform", 8, 64))
    b = W.make_sources(200, 1000, ("uniform", 8, 64))
    assert a == b
    for s in a:
        assert s[-1] == W.EOS and 8 <= len(s) - 1 <= 64
        assert all(4 <= t < 32000 for t in s[:-1])
    ln = W.make_sources(4000, 1001, ("lognormal", 28.0, 0.5))
    n = np.array([len(s) - 1 for s in ln])
    assert n.min() >= 4 and n.max() <= 200 and 25 < n.mean() < 31
    assert W.max_steps_for(36, 2) == math.ceil(math.floor(1.2 * 36 + 10) / 2) == O.max_steps_for(36, 2)


def test_engine_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = hrt.ModelConfig(d_model=16, d_ff=32, n_heads=2, enc_layers=1, vocab_size=15, max_len=6)
    with pytest.raises(hrt.EngineCudaError):
        hrt.CudaSession(hrt.HRTModel.random(cfg, 1))


def test_stage2_and_scoring_helpers():
    s = PD.build_stage2_input([10, 11, 12, hrt.EOS], 2)
    assert s.ids == [hrt.MASK, 10, hrt.MASK, 11, hrt.MASK, 12, hrt.MASK, hrt.EOS]
    assert s.positions == list(range(1, 9))
    with pytest.raises(hrt.DecodingError):
        PD.build_stage2_input([10], 2)
    h = PD.Hypothesis(tokens=[hrt.EOS], positions=[2], score=math.log(0.7), finished=True)
    assert abs(PD.combined_score(h, [math.log(0.4)], 2) - (math.log(0.7) + math.log(0.4)) / 2 ** 0.6) < 1e-12
    for bad in (hrt.MASK, hrt.PAD, hrt.EOS):
        with pytest.raises(hrt.DecodingError):
            PD.Translation([7, bad], 0.0, 0.0, 0.0, 1)
    assert PD.truncate_at_eos([7, 8, hrt.EOS, 9]) == [7, 8]


class OracleSession:
    """The session protocol backed by the numpy oracle (test double): lets
    the product-side host search run on CPU against the reference semantics."""

    def __init__(self, orc):
        self.o = orc
        self.config = hrt.ModelConfig(orc.cfg.d_model, orc.cfg.d_ff, orc.cfg.n_heads, orc.cfg.enc_layers,
                                      orc.cfg.dec_layers, orc.cfg.vocab_size, orc.cfg.max_len)
        self.decoder_calls = 0

    def encode(self, src, ws=None):
        return self.o.encode(src)

    def start_cache(self, beam, cap, ws=None, phase=None):
        return self.o.start_cache(beam, cap)

    def step(self, cache, tokens, position):
        self.decoder_calls += 1
        return self.o.step(cache, tokens, position)

    def reorder(self, cache, parents):
        self.o.reorder(cache, parents)

    def parallel_logits(self, ids, positions, mode, ws=None, pad_mask=None, phase=None):
        self.decoder_calls += 1
        return self.o.parallel_logits(ids, positions, mode, pad_mask)

    def argmax_logprobs(self, logits, exclude=None):
        return self.o.argmax_logprobs(logits, exclude)


@pytest.mark.parametrize("name", ["tiny_trained", "toy"])
def test_product_search_matches_golden_on_cpu(golden, name):
    g = golden(name)
    c = g["config"]
    ocfg = O.Config(**{k: (tuple(v) if k == "chunk_sizes" else v) for k, v in c.items()})
    params = ({k: np.asarray(v) for k, v in g["params"].items()} if "params" in g else O.init_params(ocfg, g["seed"]))
    sess = OracleSession(O.Oracle(ocfg, params, np.float64))
    for r in g["runs"][::3]:
        tr = PD.hrt_translate(sess, g["sources"][r["src"]], r["k"], r["b_at"], r["b_nat"], max_steps=r["max_steps"])
        assert tr.tokens == r["out"]["tokens"]
        assert abs(tr.score - r["out"]["score"]) < 1e-9
        assert tr.decoder_calls == r["out"]["decoder_calls"] and tr.forced == r["out"]["forced"]
    if name == "tiny_trained":
        for r in g["at_runs"]:
            tr = PD.at_translate(sess, g["sources"][r["src"]], beam=r["beam"])
            assert tr.tokens == r["out"]["tokens"] and abs(tr.score - r["out"]["score"]) < 1e-9


def test_hrtckpt1_loader_reads_reference_checkpoint(golden, tmp_path):
    """tests/golden/tiny_trained.ckpt was written by the reference's own
    save_checkpoint (checkpoint.py:24-35); the loader must reproduce its
    parameters exactly and round-trip through save_checkpoint."""
    from paper_2212_01543_b200 import checkpoint as CK

    g = golden("tiny_trained")
    m = CK.load_model(os.path.join(REPO, "tests", "golden", "tiny_trained.ckpt"))
    assert m.config.d_model == 16 and m.config.vocab_size == 15 and m.config.max_len == 6
    for n, v in g["params"].items():
        assert np.array_equal(m.params[n], np.asarray(v))
    p = tmp_path / "rt.ckpt"
    CK.save_checkpoint(m, p)
    assert open(p, "rb").read() == open(os.path.join(REPO, "tests", "golden", "tiny_trained.ckpt"), "rb").read()
    bad = tmp_path / "bad.ckpt"
    bad.write_bytes(b"NOTACKPT" + b"\0" * 16)
    with pytest.raises(CK.CheckpointError):
        CK.load_model(bad)


def test_cli_parser():
    from paper_2212_01543_b200 import cli

    a = cli.build_parser().parse_args(["translate", "--checkpoint", "m", "--vocab", "v", "--b-at", "4"])
    assert a.b_at == 4 and a.k == 2 and a.input == "-"
    a = cli.build_parser().parse_args(["bench", "--checkpoint", "m", "--vocab", "v", "--corpus", "c"])
    assert a.runs == 5


def test_bench_reference_arm_contract():
    """bench.py --impl reference (the reference CPU path, runnable without a GPU)
    prints one JSON line with the contract keys the driver reads."""
    import json
    import os
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HRT_REF_SENTENCES="1")
    out = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1"], capture_output=True, text=True, env=env, timeout=600, cwd=repo)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0


def test_arena_estimate_closed_form(lib_path):
    """estimate_max_bytes (infer.py:78-96; reference tests/test_infer.py:163-171):
    every phase reported, max = the largest phase, monotone in the capacity
    knobs, phases alias (max < sum). Host-only call into the C ABI."""
    cfg = W.C2
    est = hrt.estimate_max_bytes(cfg, "bfloat16", max_sentences=64, max_beam=1)
    assert set(est) == {"encoder", "skip-at", "skip-cmlm", "max"}
    assert est["max"] == max(v for k, v in est.items() if k != "max")
    assert est["max"] < est["encoder"] + est["skip-at"] + est["skip-cmlm"]
    big = hrt.estimate_max_bytes(cfg, "bfloat16", max_sentences=128, max_beam=1)
    assert all(big[k] >= est[k] for k in est) and big["max"] > est["max"]
    beam = hrt.estimate_max_bytes(cfg, "bfloat16", max_sentences=64, max_beam=4)
    assert beam["skip-at"] > est["skip-at"] and beam["encoder"] == est["encoder"]
    tok = hrt.estimate_max_bytes(cfg, "bfloat16", max_sentences=64, max_beam=1, max_src_tokens=1000)
    assert tok["encoder"] < est["encoder"]
    # fp32 activations are wider than bf16 ones
    assert hrt.estimate_max_bytes(cfg, "float32", max_sentences=64, max_beam=1)["encoder"] > est["encoder"]
    # encoder phase lower bound: fp32 residual + bf16 y / qkv / ctx / hidden for every token slot
    me = 64 * cfg.max_len
    assert est["encoder"] >= me * (4 * 512 + 2 * (512 + 3 * 512 + 512 + 2048))


def test_teacher_forced_accounting_flags_real_mismatches():
    """oracle.greedy_teacher_forced: an oracle decode scores 100 % against
    itself; flipping one anchor or one fill is counted as a (non-tie) miss."""
    cfg = O.Config(64, 128, 2, 2, 1, 97, 24)
    orc = O.Oracle(cfg, O.init_params(cfg, 5), dtype=np.float64)
    src = [11, 40, 7, 93, 2]
    cap = O.max_steps_for(len(src) - 1, 2)
    tr = O.hrt_translate(orc, src, 2, max_steps=cap)
    r = O.greedy_teacher_forced(orc, src, 2, tr.tokens, cap)
    assert r["bad"] == 0 and r["s1"] == r["s1_agree"] > 0 and r["s2"] == r["s2_agree"] > 0
    for j in (0, 1):  # a fill (position 0) and an anchor (position 1)
        toks = list(tr.tokens)
        toks[j] = 50 if toks[j] != 50 else 51
        r = O.greedy_teacher_forced(orc, src, 2, toks, cap)
        assert r["bad"] + r["s1_ties"] + r["s2_ties"] >= 1


def test_abi_rejects_null_engine_without_touching_cuda(lib_path):
    """Every engine call given a NULL handle returns HRT_ERR_INVALID with a message
    (no dereference, no CUDA call: runs on a host without a GPU)."""
    import ctypes as C

    lib = _lib.load(lib_path)
    assert lib.hrt_synchronize(None) == _lib.HRT_ERR_INVALID
    assert b"null engine" in lib.hrt_last_error(None)
    assert lib.hrt_set_option(None, b"graph_unroll", 16) == _lib.HRT_ERR_INVALID
    assert lib.hrt_reorder(None, None) == _lib.HRT_ERR_INVALID
    assert lib.hrt_phase_times(None, None) == _lib.HRT_ERR_INVALID
    assert lib.hrt_translate_batch(None, None, None, 0, 2, 1, 1, C.c_float(1.0), None, None, 0) == _lib.HRT_ERR_INVALID
    assert lib.hrt_stream(None) is None
    assert lib.hrt_get_stats(None, None) == _lib.HRT_ERR_INVALID
