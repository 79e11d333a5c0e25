import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
import torch
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=8, max_beam=1)
srcs = W.make_sources(32, 1001, spec["lengths"])
caps = W.stage1_caps(srcs, 2)
ids1 = [np.asarray(s, np.int32) for s in srcs]
out1 = eng.alloc_outputs(1)
for rep in range(3):
    for i in range(32):
        eng.translate_arrays(ids1[i], [len(ids1[i])], k=2, max_steps=[caps[i]], out=out1)
# per-call wall vs device phases
wall, dev = [], []
for i in range(32):
    t0 = time.perf_counter()
    eng.translate_arrays(ids1[i], [len(ids1[i])], k=2, max_steps=[caps[i]], out=out1)
    wall.append(time.perf_counter() - t0)
    dev.append(sum(eng.phase_times().values()) / 1000)
wall, dev = np.array(wall) * 1e6, np.array(dev) * 1e6
print(f"per call: wall {wall.mean():.1f} us, device phases {dev.mean():.1f} us, host overhead {np.mean(wall - dev):.1f} us (min {np.min(wall-dev):.1f})")
# python-side cost of the call path without the engine (ctypes marshalling only)
t0 = time.perf_counter()
for i in range(1000):
    lens = np.asarray([len(ids1[0])], np.int32)
t1 = time.perf_counter()
print(f"python asarray: {(t1 - t0) * 1e3:.2f} us/iter")
