"""Per-kernel-class device time of one fused batch (eager launches, CUDA events per launch)."""
import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=B, max_beam=1)
srcs = W.make_sources(B, 1001, spec["lengths"])
caps = W.stage1_caps(srcs, 2)
ids = np.concatenate([np.asarray(s, np.int32) for s in srcs]); lens = [len(s) for s in srcs]
for _ in range(2):
    eng.translate_arrays(ids, lens, k=2, max_steps=caps)
for cls in ("gemm", "vocab", "attn", "all"):
    eng.timing_enable(cls, True)
    eng.translate_arrays(ids, lens, k=2, max_steps=caps)
    r = eng.timing_read()
    rep = eng.timing_report()
    eng.timing_enable(cls, False)
    print(f"{cls:6s} {r['ms']:8.3f} ms {r['launches']:6d} launches  flops {r['flops']/1e9:9.1f} G  -> {r['flops']/(r['ms']*1e-3)/1e12 if r['ms'] else 0:7.1f} TFLOP/s")
    for k, (ms, n, _f) in sorted(rep.items(), key=lambda x: -x[1][0])[:8]:
        print(f"     {k:18s} {ms:8.3f} ms {n:6d}")
