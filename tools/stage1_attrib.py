"""Graph-mode Stage-I time with kernel groups dropped (debug attribution)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W

spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=1024, max_beam=1)
for B in (1, 64, 1024):
    srcs = W.make_sources(B, 1001, spec["lengths"])
    caps = [30] * B
    ids = np.concatenate([np.asarray(s, np.int32) for s in srcs])
    lens = [len(s) for s in srcs]
    for mask, name in ((0, "full"), (1, "-LN"), (2, "-attn"), (4, "-gemm"), (8, "-vocab"), (16, "-select"),
                       (32, "-embed"), (63, "-all")):
        eng.set_option("stage1_skip", mask)
        t = []
        for _ in range(4):
            eng.translate_arrays(ids, lens, k=2, max_steps=caps)
            t.append(eng.phase_times()["stage1"])
        print(f"B={B:5d} {name:8s} stage1 {min(t[1:]):8.3f} ms  per step {1000*min(t[1:])/30:7.1f} us", flush=True)
eng.set_option("stage1_skip", 0)
