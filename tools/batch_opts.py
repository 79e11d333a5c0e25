"""Fused-batch phase times under engine option variants (config c2):
python tools/batch_opts.py B opt=val,opt=val ...   (variants apply cumulatively)"""
import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
B = int(sys.argv[1])
spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=B, max_beam=1)
srcs = W.make_sources(B, 1001, spec["lengths"])
caps = W.stage1_caps(srcs, 2)
ids = np.concatenate([np.asarray(s, np.int32) for s in srcs]); lens = [len(s) for s in srcs]
ref = None
for variant in sys.argv[2:] or ["base"]:
    if variant != "base":
        for kv in variant.split(","):
            k, v = kv.split("=")
            eng.set_option(k, int(v))
    best = None
    for rep in range(4):
        out = eng.translate_arrays(ids, lens, k=2, max_steps=caps)
        pt = eng.phase_times()
        if rep and (best is None or sum(pt.values()) < sum(best.values())):
            best = pt
    toks = out["tokens"] if isinstance(out, dict) else out[0]
    same = "" if ref is None else ("  tokens identical" if np.array_equal(np.asarray(toks), ref) else "  TOKENS DIFFER")
    if ref is None:
        ref = np.asarray(toks).copy()
    print(f"{variant:30s} total {sum(best.values()):7.3f} ms  " + "  ".join(f"{k} {v:.3f}" for k, v in best.items()) + same)
