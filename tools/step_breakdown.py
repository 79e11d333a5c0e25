"""Live per-call-site device-time breakdown of one fused batch (eager launches,
CUDA events around every launch; numbers are per batch)."""
import argparse, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--uniform-cap", type=int, default=0, help="force every Stage-I cap (uniform live rows)")
    a = ap.parse_args()
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
    ids = np.concatenate([np.asarray(s, np.int32) for s in srcs])
    lens = [len(s) for s in srcs]
    for _ in range(2):
        eng.translate_arrays(ids, lens, k=spec["k"], b_at=spec["beam"], max_steps=caps)
    eng.timing_enable("all", True)
    eng.translate_arrays(ids, lens, k=spec["k"], b_at=spec["beam"], max_steps=caps)
    rep = eng.timing_report()
    eng.timing_enable("all", False)
    tot = sum(v[0] for v in rep.values())
    steps = max(caps)
    print(f"batch {a.batch}: {tot:.3f} ms in timed launches, Stage-I steps {steps}")
    for k, (ms, n, _f) in sorted(rep.items(), key=lambda x: -x[1][0]):
        print(f"  {k:18s} {ms:8.3f} ms {n:6d} launches {1000*ms/n:8.2f} us/launch")
    eng.translate_arrays(ids, lens, k=spec["k"], b_at=spec["beam"], max_steps=caps)
    print("graph-mode phases (ms):", eng.phase_times())


if __name__ == "__main__":
    main()
