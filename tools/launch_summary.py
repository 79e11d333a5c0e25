"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)."""
import csv, sys, collections, re

def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        rows.append((r["Kernel Name"], v))
    return rows

def short(name):
    name = re.sub(r"\(.*", "", name)
    m = re.match(r"(?:void )?(?:hrt(?:_bf16|_f32)?::)?([\w:]+)(<.*>)?", name)
    base = m.group(1) if m else name
    tmpl = m.group(2) or ""
    for tag in ("VocabEpi", "EpiBiasT<[^>]*true>", "EpiBiasT", "EpiResidual", "EpiStoreF32"):
        if re.search(tag, tmpl):
            base += "[" + tag.split("<")[0] + ("+relu" if "true" in tag else "") + "]"
            break
    bn = re.match(r"<(\d+), (\d+)", tmpl)
    if bn and "tc_gemm" in base:
        base += f"BN{bn.group(1)}"
    return base

if __name__ == "__main__":
    rows = load(sys.argv[1])
    tot = sum(v for _, v in rows)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v in rows:
        a = agg[short(n)]; a[0] += 1; a[1] += v
    print(f"{len(rows)} launches, {tot/1000:.3f} ms total device time")
    for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v/1000:9.3f} ms {100*v/tot:5.1f}%  {c:5d} x {v/c:8.2f} us  {n}")
