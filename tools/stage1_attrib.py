"""Graph-mode Stage-I time with kernel groups dropped (debug attribution)."""
import argparse, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--batches", default="1,64,1024")
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--opts", default="", help="engine options name=value,...")
a = ap.parse_args()
spec = W.CONFIGS[a.config]
Bs = [int(x) for x in a.batches.split(",")]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=max(Bs),
                 max_beam=spec["beam"])
for kv in [x for x in a.opts.split(",") if x]:
    kk, vv = kv.split("=")
    eng.set_option(kk, int(vv))
names = ((0, "full"),) if os.environ.get("FULL_ONLY") else ((0, "full"), (1, "-LN"), (4, "-gemm"), (8, "-vocab"), (16, "-select/rowstat"),
         (32, "-embed/beam_sel"), (2, "-attn"), (64, "-self-attn"), (128, "-cross-attn"))
for B in Bs:
    srcs = W.make_sources(B, 1001, spec["lengths"])
    caps = [a.steps] * B
    ids = np.concatenate([np.asarray(s, np.int32) for s in srcs])
    lens = [len(s) for s in srcs]
    for mask, name in names:
        eng.set_option("stage1_skip", mask)
        t = []
        try:
            for _ in range(4):
                eng.translate_arrays(ids, lens, k=spec["k"], b_at=spec["beam"], max_steps=caps)
                t.append(eng.phase_times()["stage1"])
        except Exception as ex:  # skipped kernels can leave garbage state
            print(f"B={B:5d} {name:16s} failed: {type(ex).__name__}", flush=True)
            break
        print(f"B={B:5d} {name:16s} stage1 {min(t[1:]):8.3f} ms  per step {1000*min(t[1:])/a.steps:7.1f} us",
              flush=True)
eng.set_option("stage1_skip", 0)
