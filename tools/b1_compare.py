"""Batch-1 / small-batch latency: regular graph path vs the tail megakernel."""
import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2212_01543_b200 as hrt
from paper_2212_01543_b200 import workload as W
spec = W.CONFIGS["c2"]
eng = hrt.Engine(hrt.HRTModel.random(spec["shape"], spec["seed"]), dtype="bfloat16", max_sentences=32, max_beam=1)
import threading, pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0); clk = []; stop = threading.Event()
def samp():
    while not stop.is_set():
        clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)); stop.wait(0.002)
th = threading.Thread(target=samp, daemon=True); th.start()
for B in (1, 8, 16):
    srcs = W.make_sources(B * 16, 1001, spec["lengths"])
    caps = W.stage1_caps(srcs, 2)
    for mega in (0, 1):
        eng.set_option("mega", mega)
        res = []
        for rep in range(2):
            tot = 0.0
            steps = 0
            for i in range(0, len(srcs), B):
                s = srcs[i:i + B]
                ids = np.concatenate([np.asarray(x, np.int32) for x in s]); lens = [len(x) for x in s]
                eng.translate_arrays(ids, lens, k=2, max_steps=caps[i:i + B])
                ph = eng.phase_times()
                tot += sum(ph.values())
                steps += max(caps[i:i + B])
            res.append((tot, steps, ph))
        tot, steps, ph = res[-1]
        print(f"B={B} mega={mega}: {tot / 16:.3f} ms/call, stage1 {ph['stage1']:.3f} ms last call; "
              f"mean Stage-I steps {steps / 16:.1f}; phases {ph}; sm clock median {np.median(clk[-200:]) if clk else None}")
        clk.clear()
