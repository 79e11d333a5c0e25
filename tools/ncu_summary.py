"""Summarise an ncu CSV launch list (gpu__time_duration.sum + dram bytes per
launch) into per-kernel-class totals; optionally write the GEMM-class DRAM
traffic per launch to a JSON that bench.py uses for roofline.traffic.

    python tools/ncu_summary.py launches.csv [--traffic-json profiles/gemm_traffic.json]
"""
import argparse
import collections
import csv
import json
import re


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    per = collections.OrderedDict()
    for r in csv.DictReader(lines):
        k = r["ID"]
        d = per.setdefault(k, {"name": r["Kernel Name"], "grid": r.get("Grid Size", "")})
        v = float(r["Metric Value"].replace(",", "")) if r["Metric Value"] not in ("", "n/a") else 0.0
        u = r.get("Metric Unit", "")
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["us"] = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1e-3)
        elif r["Metric Name"].startswith("dram__bytes"):
            d[r["Metric Name"]] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return per


def klass(name):
    name = re.sub(r"hrt(_bf16|_f32)?::", "", name).replace("(int)", "")
    base = re.sub(r"\(.*", "", name)
    m = re.search(r"tc_gemm_kernel<(\d+), (\d+), (\w+)", name)
    if m:
        return f"tc_gemm[{m.group(3)}]BN{m.group(1)}"
    return re.sub(r"^void ", "", re.sub(r"<.*", "", base)).replace("hrt::", "")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--traffic-json", default=None)
    a = ap.parse_args()
    per = load(a.csv)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in per.values():
        k = klass(d["name"])
        g = agg[k]
        g[0] += 1
        g[1] += d.get("us", 0.0)
        g[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(g[1] for g in agg.values())
    print(f"{len(per)} launches, {tot / 1000:.3f} ms device time (ncu: serialised, cold caches)")
    print(f"{'class':34s} {'launches':>8s} {'ms':>9s} {'share':>6s} {'us/launch':>10s} {'DRAM MB/launch':>15s}")
    for k, (n, us, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:34s} {n:8d} {us / 1000:9.3f} {100 * us / tot:5.1f}% {us / n:10.2f} {b / n / 1e6:15.3f}")
    if a.traffic_json:
        # every tcgen05 GEMM launch (plain + the fused residual + LayerNorm kernels), as bench.py's GEMM class
        gem = [d for d in per.values() if "tc_gemm" in d["name"]]
        tb = sum(d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0) for d in gem)
        out = {"source": a.csv, "gemm_launches": len(gem), "gemm_dram_bytes_total": tb,
               "gemm_dram_bytes_per_launch": tb / max(1, len(gem)),
               "gemm_share_of_ncu_time": sum(d.get("us", 0) for d in gem) / tot if tot else None}
        json.dump(out, open(a.traffic_json, "w"), indent=1)
        print("wrote", a.traffic_json, out)


if __name__ == "__main__":
    main()
