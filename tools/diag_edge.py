import json, numpy as np, sys
sys.path.insert(0, "/root/repo")
from oracle import hrt_oracle as O
import paper_2212_01543_b200 as hrt
g = json.load(open("/root/repo/tests/golden/toy.json"))
cfg = hrt.ModelConfig.from_any(g["config"])
params = {k: np.asarray(v, np.float64) for k, v in g["params"].items()} if "params" in g else hrt.init_params(cfg, g["seed"])
model = hrt.HRTModel(cfg, params)
c = g["config"]
ocfg = O.Config(**{k: (tuple(v) if k == "chunk_sizes" else v) for k, v in c.items()})
orc = O.Oracle(ocfg, model.params, dtype=np.float64)
sess = hrt.CudaSession(model, dtype=np.float32, max_sentences=8)
ref = O.hrt_translate(orc, [9, 2], 2)
one = hrt.hrt_translate(sess, [9, 2], 2)
print("oracle", ref.tokens[:6], "engine single", one.tokens[:6], one.score, ref.score)
ids, pos = O.build_stage2_input(ref.anchors, 2)
ol = np.array(orc.parallel_logits(np.asarray([ids]), np.asarray([pos]), "full")[0], np.float64)
sess.encode([9, 2])
el = np.array(sess.parallel_logits([ids], np.asarray([pos]), "full")[0], np.float64)
print("protocol parallel_logits max abs diff", np.abs(el - ol).max(), "max |ref|", np.abs(ol).max())
print("row0 top", ol[0, [87, 62]], el[0, [87, 62]])
mem_o = np.array(orc.encode([9, 2]), np.float64) if hasattr(orc, "encode") else None
rng = np.random.default_rng(11)
L, V = c["max_len"], c["vocab_size"]
def body(n):
    return [int(x) for x in rng.integers(7, V, n)]
srcs = [[2], body(L - 1) + [2], body(L + 6) + [2], body(3) + [2], [9, 2]]
for combo in ([4], [0, 4], [1, 4], [2, 4], [3, 4], [0, 1, 2, 3, 4], [2, 3], [1, 3]):
    out = hrt.hrt_translate_batch(sess, [srcs[i] for i in combo], 2)
    oks = []
    for i, tr in zip(combo, out):
        r = O.hrt_translate(orc, srcs[i], 2)
        oks.append(tr.tokens == r.tokens)
    print(combo, oks)
