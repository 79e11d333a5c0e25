import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=32, max_beam=1)
eng.set_option("mega", 1)
eng.set_option("mega_trace", 1)
for B in (1, 8):
    srcs = W.make_sources(B, 1001, spec["lengths"])
    ids = np.concatenate([np.asarray(s, np.int32) for s in srcs]); lens = [len(s) for s in srcs]
    for _ in range(3):
        eng.translate_arrays(ids, lens, k=2, max_steps=[30] * B)
    tr = eng.debug_trace()
    tr = tr[tr > 0]
    d = np.diff(tr) / 1000.0
    names = ["qkv", "self", "wo", "qc", "cross", "woc", "w1", "w2", "vocab", "select"]
    print("B", B, "step total us", (tr[-1] - tr[0]) / 1000.0, [f"{n}:{x:.1f}" for n, x in zip(names, d)])
