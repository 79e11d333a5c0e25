import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
B = 1024
spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=B, max_beam=1)
srcs = W.make_sources(B, 1001, spec["lengths"])
ids = np.concatenate([np.asarray(s, np.int32) for s in srcs]); lens = [len(s) for s in srcs]
for lnep in (0, 1):
    eng.set_option("ln_epi", lnep)
    for _ in range(2):
        eng.translate_arrays(ids, lens, k=2, max_steps=[2] * B)
    for cls in ("gemm", "all"):
        eng.timing_enable(cls, True)
        eng.translate_arrays(ids, lens, k=2, max_steps=[2] * B)
        r = eng.timing_read(); rep = eng.timing_report()
        eng.timing_enable(cls, False)
        print(lnep, cls, f"{r['ms']:.3f} ms {r['launches']} launches", {k: (round(v[0], 3), v[1]) for k, v in rep.items()})
