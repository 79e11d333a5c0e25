import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=32, max_beam=1)
srcs = W.make_sources(1, 1001, spec["lengths"])
ids = np.concatenate([np.asarray(s, np.int32) for s in srcs]); lens = [len(s) for s in srcs]
eng.set_option("mega_trace", 1)
for _ in range(3):
    eng.translate_arrays(ids, lens, k=2, max_steps=[30])
tr = eng.debug_trace()
print("fine (cycles): wait", tr[49] - tr[48], "proj->first epi", tr[50] - tr[49], "epi", tr[51] - tr[50], "rest", tr[52] - tr[51])
print("tile (cycles): issue direct", tr[41] - tr[40], "slot part", tr[42] - tr[41], "direct part", tr[43] - tr[42])
