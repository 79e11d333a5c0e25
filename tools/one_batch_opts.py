"""One C2 batch with engine options (for ncu captures): python tools/one_batch_opts.py B opt=v[,opt=v]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W

B = int(sys.argv[1])
spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=B, max_beam=1)
for kv in filter(None, (sys.argv[2] if len(sys.argv) > 2 else "").split(",")):
    k, v = kv.split("=")
    eng.set_option(k, int(v))
srcs = W.make_sources(B, spec["seed"] + 1000, spec["lengths"])
caps = W.stage1_caps(srcs, 2)
ids = np.concatenate([np.asarray(s, np.int32) for s in srcs])
out = eng.translate_arrays(ids, [len(s) for s in srcs], k=2, max_steps=caps)
eng.synchronize()
print("ok", int(out["lens"].sum()))
