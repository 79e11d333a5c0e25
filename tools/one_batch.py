"""One fused batch (config $HRT_CFG, default c2) for profiling."""
import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = W.CONFIGS[os.environ.get("HRT_CFG", "c2")]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]),
                 dtype="float32" if spec["dtype"] == "f32" else "bfloat16", max_sentences=B, max_beam=1)
srcs = W.make_sources(B, 1001, spec["lengths"])
caps = W.stage1_caps(srcs, 2)
ids = np.concatenate([np.asarray(s, np.int32) for s in srcs]); lens = [len(s) for s in srcs]
if os.environ.get("HRT_GRAPHS") == "0":
    eng.set_option("graphs", 0)
for _ in range(n):
    eng.translate_arrays(ids, lens, k=2, max_steps=caps)
print(eng.phase_times())
