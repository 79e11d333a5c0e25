"""Phase times of one C2 batch under engine option variants:
python tools/phase_opts.py <batch> [opt=val,opt=val ...] -- device ms (best of 4) + token agreement vs the first variant."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W

B = int(sys.argv[1])
spec = W.CONFIGS[os.environ.get("CFG", "c2")]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=B,
                 max_beam=spec["beam"])
srcs = W.make_sources(B, spec["seed"] + 1000, spec["lengths"])
caps = W.stage1_caps(srcs, spec["k"])
ids = np.concatenate([np.asarray(s, np.int32) for s in srcs])
lens = [len(s) for s in srcs]
ref = None
for variant in sys.argv[2:] or ["base"]:
    if variant != "base":
        for kv in variant.split(","):
            k, v = kv.split("=")
            eng.set_option(k, int(v))
    best = None
    for _ in range(4):
        out = eng.translate_arrays(ids, lens, k=spec["k"], b_at=spec["beam"], max_steps=caps)
        ph = eng.phase_times()
        tot = sum(ph.values())
        if best is None or tot < best[0]:
            best = (tot, ph)
    toks = [out["tokens"][i, : out["lens"][i]].tolist() for i in range(B)]
    if ref is None:
        ref = toks
    agree = sum(sum(a == b for a, b in zip(x, y)) for x, y in zip(toks, ref)) / max(1, sum(max(len(x), len(y)) for x, y in zip(toks, ref)))
    words = int(out["lens"].sum())
    print(f"B={B} {variant:28s} total {best[0]:.3f} ms ({words / best[0] / 1e3:.3f} M w/s)  " +
          "  ".join(f"{k} {v:.3f}" for k, v in best[1].items()) + f"  agree-vs-first {agree:.4f}", flush=True)
