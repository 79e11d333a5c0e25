"""Encoder cluster kernel vs the per-kernel chain by source length (batch 1), and the
phase times of the cluster kernel (globaltimer stamps, CTA 0): python tools/ec_trace.py [trace]"""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=8, max_beam=1)
base = W.make_sources(1, 1001, spec["lengths"])[0]
for L in (4, 8, 12, 16, 24, 32, 40, 48, 64):
    s = np.asarray(((base[:-1] * 8)[: L - 1]) + [2], np.int32)
    res = []
    for mode in (1, 0):
        eng.set_option("enc_cluster", mode)
        t = []
        for _ in range(6):
            eng.translate_arrays(s, [L], k=2, max_steps=[3])
            t.append(eng.phase_times()["encoder"])
        res.append(1000 * min(t[2:]))
    print(f"M={L:3d}: encoder cluster {res[0]:7.1f} us  per-kernel {res[1]:7.1f} us")
if len(sys.argv) > 1:
    eng.set_option("enc_cluster", 1)
    eng.set_option("ec_trace", 1)
    eng.translate_batch([base], 2, max_steps=[5])
    eng.synchronize()
