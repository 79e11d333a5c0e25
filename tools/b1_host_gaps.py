"""Batch-1 phases with and without host-launch gaps: the same translate call is issued
(a) as usual, and (b) behind a ~3 ms spin kernel on the engine stream, so every launch of
the call is queued before the GPU reaches it and the device phase times are pure GPU
execution. The difference is the time the GPU waited for the host to launch."""
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_2212_01543_b200 as hrt  # noqa: E402
from paper_2212_01543_b200 import workload as W  # noqa: E402

spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=8, max_beam=1)
srcs = W.make_sources(32, 1001, spec["lengths"])
caps = W.stage1_caps(srcs, 2)
ids1 = [np.asarray(s, np.int32) for s in srcs]
out1 = eng.alloc_outputs(1)
st = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", 0))
for rep in range(3):
    for i in range(32):
        eng.translate_arrays(ids1[i], [len(ids1[i])], k=2, max_steps=[caps[i]], out=out1)
for mode in ("eager", "queued"):
    ph = {"encoder": [], "stage1": [], "stage2": []}
    for i in range(32):
        if mode == "queued":
            with torch.cuda.stream(st):
                torch.cuda._sleep(6_000_000)  # ~3 ms at 1.9 GHz
        eng.translate_arrays(ids1[i], [len(ids1[i])], k=2, max_steps=[caps[i]], out=out1)
        for kk, v in eng.phase_times().items():
            ph[kk].append(v)
    print(mode, {kk: round(float(np.mean(v)), 4) for kk, v in ph.items()}, "ms per sentence (device phases)", flush=True)
