"""Per-call-site device time of one C2 batch (eager launches, CUDA events per launch)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=B, max_beam=1)
srcs = W.make_sources(B, 1001, spec["lengths"])
caps = W.stage1_caps(srcs, 2)
ids = np.concatenate([np.asarray(s, np.int32) for s in srcs]); lens = [len(s) for s in srcs]
for kv in filter(None, os.environ.get("OPTS", "").split(",")):
    k, v = kv.split("=")
    eng.set_option(k, int(v))
for _ in range(2):
    eng.translate_arrays(ids, lens, k=2, max_steps=caps)
eng.timing_enable("all", True)
eng.translate_arrays(ids, lens, k=2, max_steps=caps)
rep = eng.timing_report()
eng.timing_enable("all", False)
tot = sum(v[0] for v in rep.values())
print(f"B={B}: {tot:.3f} ms in {sum(v[1] for v in rep.values())} launches (per-launch events)")
for k, (ms, n, fl) in sorted(rep.items(), key=lambda x: -x[1][0]):
    print(f"  {k:22s} {ms:8.3f} ms {n:6d} x {1000 * ms / n:8.2f} us  {fl / (ms * 1e-3) / 1e12 if ms and fl else 0:8.1f} TFLOP/s")
