"""Batch-1 latency under engine option variants: python tools/b1_opts.py opt=val,opt=val ..."""
import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=8, max_beam=1)
srcs = W.make_sources(16, 1001, spec["lengths"])
caps = W.stage1_caps(srcs, 2)
for variant in sys.argv[1:] or ["base"]:
    if variant != "base":
        for kv in variant.split(","):
            k, v = kv.split("=")
            eng.set_option(k, int(v))
    for rep in range(2):
        tot = {"encoder": 0.0, "stage1": 0.0, "stage2": 0.0}
        steps = 0
        for s, c in zip(srcs, caps):
            eng.translate_arrays(np.asarray(s, np.int32), [len(s)], k=2, max_steps=[c])
            for kk, vv in eng.phase_times().items():
                tot[kk] += vv
            steps += c
    n = len(srcs)
    print(f"{variant:28s} total {sum(tot.values()) / n:.3f} ms/sentence  encoder {tot['encoder'] / n:.3f}  "
          f"stage1 {tot['stage1'] / n:.3f} ({1000 * tot['stage1'] / steps:.1f} us/step)  stage2 {tot['stage2'] / n:.3f}")
