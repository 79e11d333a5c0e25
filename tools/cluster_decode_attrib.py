"""Batch-1 Stage-I kernels timed one by one (eager launches, CUDA events per launch):
cluster decode kernel vs the per-kernel chain it replaces."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=8, max_beam=1)
srcs = W.make_sources(4, 1001, spec["lengths"])
eng.set_option("graphs", 0)
for cd in (0, 1):
    eng.set_option("cluster_decode", cd)
    for s in srcs:
        eng.translate_batch([s], 2, max_steps=[30])
    eng.timing_enable("all", True)
    for s in srcs:
        eng.translate_batch([s], 2, max_steps=[30])
    rep = eng.timing_report()
    eng.timing_enable("all", False)
    n = 30 * len(srcs)
    print(f"cluster_decode={cd}: " + ", ".join(f"{k} {1000 * v[0] / n:.2f}us x{v[1] / n:.0f}" for k, v in sorted(rep.items()) if k.startswith("s1")), flush=True)
