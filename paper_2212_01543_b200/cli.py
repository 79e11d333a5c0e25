"""Command line for the B200 engine, mirroring the reference's `hrt translate`
and `hrt bench` (cli.py:150-197) on the fused batch path.

    python -m paper_2212_01543_b200 translate --checkpoint m.ckpt --vocab v.txt --input src.txt [--jsonl out.jsonl]
    python -m paper_2212_01543_b200 bench --checkpoint m.ckpt --vocab v.txt --corpus pairs.tsv

Vocabulary / corpus files use the reference formats (data.py:178-209): one
token per line in id order; TSV "source<TAB>target" lines of whitespace-split
tokens. Sentences are decoded in batches of --batch through one fused call.
"""

from __future__ import annotations

import argparse
import json
import sys
import time

from . import checkpoint
from .decoding import hrt_translate_batch
from .engine import CudaSession


def load_vocab(path):
    with open(path, encoding="utf-8") as f:
        tokens = [line.rstrip("\n") for line in f if line.strip()]
    return tokens, {t: i for i, t in enumerate(tokens)}


def encode(line, index):
    try:
        return [index[t] for t in line.split()]
    except KeyError as ex:
        raise SystemExit(f"unknown token {ex.args[0]!r}")


def _session(args, n):
    model = checkpoint.load_model(args.checkpoint)
    return CudaSession(model, dtype=args.dtype, device=args.device, max_sentences=n, max_beam=max(1, args.b_at))


def _batches(seq, n):
    for i in range(0, len(seq), n):
        yield seq[i: i + n]


def cmd_translate(args):
    tokens, index = load_vocab(args.vocab)
    src = sys.stdin if args.input == "-" else open(args.input, encoding="utf-8")
    lines = [ln.strip() for ln in src if ln.strip()]
    sess = _session(args, args.batch)
    jsonl = open(args.jsonl, "w", encoding="utf-8") if args.jsonl else None
    for chunk in _batches(lines, args.batch):
        t0 = time.perf_counter()
        outs = hrt_translate_batch(sess, [encode(ln, index) for ln in chunk], args.k, args.b_at, args.b_nat,
                                   args.length_penalty)
        wall = (time.perf_counter() - t0) / max(1, len(chunk))
        for ln, tr in zip(chunk, outs):
            text = " ".join(tokens[t] for t in tr.tokens)
            print(text)
            if jsonl:
                jsonl.write(json.dumps({"source": ln, "output": text, "score": tr.score,
                                        "skip_at_score": tr.skip_at_score, "skip_cmlm_score": tr.skip_cmlm_score,
                                        "decoder_calls": tr.decoder_calls, "wall_time": wall,
                                        "forced": tr.forced}) + "\n")
    if jsonl:
        jsonl.close()


def cmd_bench(args):
    tokens, index = load_vocab(args.vocab)
    with open(args.corpus, encoding="utf-8") as f:
        sources = [encode(ln.split("\t")[0], index) for ln in f if ln.strip()]
    sess = _session(args, args.batch)
    for chunk in _batches(sources[: args.batch], args.batch):  # warm-up (bench.py:81-82)
        hrt_translate_batch(sess, chunk, args.k, args.b_at, args.b_nat)
    secs, words = [], 0
    for _ in range(args.runs):
        t0 = time.monotonic()
        for chunk in _batches(sources, args.batch):
            words_run = sum(len(t.tokens) for t in hrt_translate_batch(sess, chunk, args.k, args.b_at, args.b_nat))
            words += words_run
        secs.append(time.monotonic() - t0)
    src_tokens = sum(len(s) for s in sources)
    report = {"mode": "hrt", "k": args.k, "b_at": args.b_at, "b_nat": args.b_nat, "runs": args.runs,
              "sentences": len(sources), "source_tokens": src_tokens, "seconds_mean": sum(secs) / len(secs),
              "wps_mean": src_tokens * len(secs) / sum(secs), "target_wps_mean": words / sum(secs),
              "run_seconds": secs, "engine": f"B200 fused path, dtype {args.dtype}, batch {args.batch}"}
    text = json.dumps(report, indent=2)
    if args.json:
        with open(args.json, "w", encoding="utf-8") as f:
            f.write(text + "\n")
    print(text)


def build_parser():
    p = argparse.ArgumentParser(prog="paper_2212_01543_b200")
    sub = p.add_subparsers(dest="cmd", required=True)
    for name, fn in (("translate", cmd_translate), ("bench", cmd_bench)):
        s = sub.add_parser(name)
        s.set_defaults(fn=fn)
        s.add_argument("--checkpoint", required=True)
        s.add_argument("--vocab", required=True)
        s.add_argument("--k", type=int, default=2)
        s.add_argument("--b-at", dest="b_at", type=int, default=1)
        s.add_argument("--b-nat", dest="b_nat", type=int, default=1)
        s.add_argument("--length-penalty", type=float, default=0.6)
        s.add_argument("--dtype", default="float32")
        s.add_argument("--device", type=int, default=0)
        s.add_argument("--batch", type=int, default=256)
        if name == "translate":
            s.add_argument("--input", default="-")
            s.add_argument("--jsonl", default=None)
        else:
            s.add_argument("--corpus", required=True)
            s.add_argument("--runs", type=int, default=5)
            s.add_argument("--json", default=None)
    return p


def main(argv=None):
    args = build_parser().parse_args(argv)
    args.fn(args)


if __name__ == "__main__":
    main()
