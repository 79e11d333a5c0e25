"""One profiled HRT batch (for ncu --profile-from-start off).

    python tools/profile_step.py [--batch 1024] [--config c2]

Warms the engine up, then brackets exactly one hrt_translate_batch with
cudaProfilerStart/Stop so `ncu --profile-from-start off` captures one step.
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--uniform-cap", type=int, default=0)
    a = ap.parse_args()
    import torch

    import paper_2212_01543_b200 as hrt
    from paper_2212_01543_b200 import workload as W

    spec = W.CONFIGS[a.config]
    srcs = W.make_sources(a.batch, spec["seed"] + 1000, spec["lengths"])
    caps = W.stage1_caps(srcs, spec["k"])
    if a.uniform_cap:
        caps = [a.uniform_cap] * len(caps)
    eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]),
                     dtype="bfloat16" if spec["dtype"] == "bf16" else "float32", max_sentences=a.batch,
                     max_beam=spec["beam"])
    if a.no_graph:
        eng.set_option("graphs", 0)
    ids = np.concatenate([np.asarray(s, np.int32) for s in srcs])
    lens = [len(s) for s in srcs]
    for _ in range(2):
        out = eng.translate_arrays(ids, lens, k=spec["k"], b_at=spec["beam"], max_steps=caps)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(a.repeat):
        out = eng.translate_arrays(ids, lens, k=spec["k"], b_at=spec["beam"], max_steps=caps)
    eng.synchronize()
    torch.cuda.profiler.stop()
    print("words", int(out["lens"].sum()), "launches", eng.stats()["kernel_launches"])


if __name__ == "__main__":
    main()
