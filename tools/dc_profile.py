"""Batch-1 decodes with the cluster decode kernel, bracketed for ncu --profile-from-start off."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=8, max_beam=1)
srcs = W.make_sources(3, 1001, spec["lengths"])
eng.set_option("cluster_decode", int(os.environ.get("CD", "1")))
for s in srcs:
    eng.translate_batch([s], 2, max_steps=[30])
torch.cuda.synchronize()
torch.cuda.profiler.start()
eng.translate_batch([srcs[0]], 2, max_steps=[30])
eng.synchronize()
torch.cuda.profiler.stop()
