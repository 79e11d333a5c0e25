"""Batch-1 device phases under engine-option variants, interleaved A/B:
python tools/b1_opt_ab.py attn_meta_pre=0 attn_meta_pre=1"""
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
import paper_2212_01543_b200 as hrt  # noqa: E402
from paper_2212_01543_b200 import workload as W  # noqa: E402

spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=8, max_beam=1)
srcs = W.make_sources(32, 1001, spec["lengths"])
caps = W.stage1_caps(srcs, 2)
ids1 = [np.asarray(s, np.int32) for s in srcs]
out1 = eng.alloc_outputs(1)
variants = [dict(kv.split("=") for kv in v.split(",")) for v in sys.argv[1:]]
res = {i: {"encoder": [], "stage1": [], "stage2": []} for i in range(len(variants))}
toks = {}
for rep in range(4):
    for vi, v in enumerate(variants):
        for n, x in v.items():
            eng.set_option(n, int(x))
        for i in range(32):
            eng.translate_arrays(ids1[i], [len(ids1[i])], k=2, max_steps=[caps[i]], out=out1)
            if rep > 0:
                for kk, t in eng.phase_times().items():
                    res[vi][kk].append(t)
            toks.setdefault(vi, []).append(out1["tokens"][0, : int(out1["lens"][0])].tolist())
for vi, v in enumerate(variants):
    same = all(a == b for a, b in zip(toks[vi], toks[0]))
    print(sys.argv[1 + vi], {kk: round(float(np.mean(x)), 4) for kk, x in res[vi].items()}, "ms; tokens equal to first:", same)
