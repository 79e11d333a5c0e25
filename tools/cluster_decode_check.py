"""Cluster decode kernel vs the per-kernel Stage-I path: batch-1..4 latency and token agreement."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W

spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=8, max_beam=1)
srcs = W.make_sources(16, 1001, spec["lengths"])
caps = W.stage1_caps(srcs, 2)
res = {}
for mode in (0, 1):
    eng.set_option("cluster_decode", mode)
    for B in (1, 3):
        tot = {"encoder": 0.0, "stage1": 0.0, "stage2": 0.0}
        steps = 0
        toks = []
        for rep in range(2):
            for i in range(0, len(srcs), B):
                ss, cc = srcs[i:i + B], caps[i:i + B]
                out = eng.translate_batch(ss, 2, max_steps=cc)
                if rep == 1:
                    toks += [t.tokens for t in out]
                    for kk, vv in eng.phase_times().items():
                        tot[kk] += vv
                    steps += max(cc)
        res[(mode, B)] = toks
        n = len(srcs) / B
        print(f"cluster_decode={mode} B={B}: stage1 {1000 * tot['stage1'] / steps:.1f} us/step, "
              f"{sum(tot.values()) / n:.3f} ms/call (enc {tot['encoder'] / n:.3f})", flush=True)
for B in (1, 3):
    a, b = res[(0, B)], res[(1, B)]
    agree = sum(sum(x == y for x, y in zip(p, q)) for p, q in zip(a, b)) / sum(max(len(p), len(q)) for p, q in zip(a, b))
    print(f"B={B} token agreement cluster vs per-kernel path: {agree:.4f}")
