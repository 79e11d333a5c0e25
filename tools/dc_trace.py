import os, sys
sys.path.insert(0, "/root/repo")
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=8, max_beam=1)
srcs = W.make_sources(3, 1001, spec["lengths"])
eng.set_option("cluster_decode", 1)
eng.set_option("dc_dbg", 8)
for g in (0, 1):
    eng.set_option("graphs", g)
    for s in srcs:
        eng.translate_batch([s], 2, max_steps=[30])
    eng.synchronize()
