"""Timing attribution of the persistent Stage-I kernel: skip phases (results meaningless)."""
import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
spec = W.CONFIGS["c2"]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=32, max_beam=1)
srcs = W.make_sources(B, 1001, spec["lengths"])
ids = np.concatenate([np.asarray(s, np.int32) for s in srcs]); lens = [len(s) for s in srcs]
steps = 40
names = "A:qkv B:self C:wo D:qc E:cross F:woc G:w1 H:w2 I:vocab".split()
def run(skip):
    eng.set_option("mega_skip", skip)
    ts = []
    for _ in range(4):
        eng.translate_arrays(ids, lens, k=2, max_steps=[steps] * B)
        ts.append(eng.phase_times()["stage1"])
    return min(ts) * 1000 / steps
full = run(0)
allskip = run(511)
print(f"B={B}: full {full:.1f} us/step; barriers only {allskip:.1f} us/step")
for i, n in enumerate(names):
    only = run(511 & ~(1 << i))
    print(f"  {n:8s} alone: +{only - allskip:.1f} us   removing it: -{full - run(1 << i):.1f} us")
