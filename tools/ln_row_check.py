"""Full-row residual+LayerNorm epilogue (option ln_row): token agreement of each variant with
the fp32 engine and with the unfused bf16 path, at C2 shape.
python tools/ln_row_check.py [B]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
spec = W.CONFIGS["c2"]
model = hrt.HRTModel.random(spec["shape"], spec["seed"])
srcs = W.make_sources(B, 77, spec["lengths"])
caps = W.stage1_caps(srcs, 2)


def agree(a, b):
    same = sum(p == q for x, y in zip(a, b) for p, q in zip(x.tokens, y.tokens))
    return same / sum(max(len(x.tokens), len(y.tokens)) for x, y in zip(a, b))


f32 = hrt.Engine(model, dtype="float32", max_sentences=B, max_beam=1)
ref = f32.translate_batch(srcs, 2, max_steps=caps)
del f32
eng = hrt.Engine(model, dtype="bfloat16", max_sentences=B, max_beam=1)
outs = {}
for v in (0, 1, 2, 3, 4, 0):
    eng.set_option("ln_row", v)
    outs[v] = eng.translate_batch(srcs, 2, max_steps=caps)
    print(f"ln_row={v}: vs fp32 {agree(outs[v], ref):.4f}  vs unfused bf16 {agree(outs[v], outs[0]):.4f}", flush=True)
