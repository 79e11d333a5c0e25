"""Eager Stage-I run at uniform live rows for ncu captures of decode-regime kernels."""
import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=B, max_beam=1)
eng.set_option("graphs", 0)
srcs = W.make_sources(B, 1001, spec["lengths"])
ids = np.concatenate([np.asarray(s, np.int32) for s in srcs]); lens = [len(s) for s in srcs]
for _ in range(2):
    eng.translate_arrays(ids, lens, k=2, max_steps=[6] * B)
