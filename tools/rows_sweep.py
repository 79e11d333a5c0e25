"""Stage-I per-step cost at uniform live rows under option variants."""
import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
spec = W.CONFIGS["c2"]
rows = [int(x) for x in sys.argv[1].split(",")]
variants = sys.argv[2:] or ["base"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=max(rows), max_beam=1)
for v in variants:
    if v != "base":
        for kv in v.split(","):
            k, val = kv.split("=")
            eng.set_option(k, int(val))
    out = []
    for B in rows:
        srcs = W.make_sources(B, 1001, spec["lengths"])
        ids = np.concatenate([np.asarray(s, np.int32) for s in srcs]); lens = [len(s) for s in srcs]
        t = []
        for _ in range(4):
            eng.translate_arrays(ids, lens, k=2, max_steps=[30] * B)
            t.append(eng.phase_times()["stage1"])
        out.append(f"R={B}: {1000 * min(t[1:]) / 30:.1f}")
    print(f"{v:24s} us/step  " + "  ".join(out), flush=True)
