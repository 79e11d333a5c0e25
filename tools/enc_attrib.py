"""Encoder phase time with kernel groups dropped (debug attribution):
python tools/enc_attrib.py [batch]  -- enc_skip 1 LN, 2 attention, 4 projections."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=B, max_beam=1)
srcs = W.make_sources(B, 1001, spec["lengths"])
ids = np.concatenate([np.asarray(s, np.int32) for s in srcs])
lens = [len(s) for s in srcs]
for mask, name in ((0, "full"), (1, "-LN"), (2, "-attn"), (4, "-proj"), (5, "-LN-proj")):
    eng.set_option("enc_skip", mask)
    t = []
    for _ in range(4):
        eng.translate_arrays(ids, lens, k=2, max_steps=[2] * B)
        t.append(eng.phase_times()["encoder"])
    print(f"B={B} tokens={sum(lens)} {name:10s} encoder {min(t[1:]):.3f} ms", flush=True)
eng.set_option("enc_skip", 0)
