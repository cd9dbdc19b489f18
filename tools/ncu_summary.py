"""Per-kernel summary of an ncu --csv launch list (gpu__time_duration.sum and,
when captured, dram__bytes_read.sum / dram__bytes_write.sum).

    python tools/ncu_summary.py LAUNCHES.csv [--skip N] [--json OUT.json]

--skip drops the first N launches of every kernel (warm-up runs).  Prints a
markdown table (launches, mean time, share, DRAM bytes per launch) and writes
the per-kernel means as JSON for bench.py's roofline `traffic` fields.
"""
import csv
import json
import re
import sys
from collections import OrderedDict, defaultdict


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"maya::(\(anonymous namespace\)::)?", "", name)
    return name.strip()


def load(path: str):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if not ln.startswith("==")]
    for r in csv.DictReader(lines):
        if "Kernel Name" not in r or not r.get("Metric Name"):
            continue
        rows.append(r)
    per = OrderedDict()
    for r in rows:
        key = (r["ID"], short(r["Kernel Name"]))
        unit = r.get("Metric Unit", "")
        v = float(r["Metric Value"].replace(",", ""))
        name = r["Metric Name"]
        if name == "gpu__time_duration.sum":
            v = v * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0,
                     "ms": 1.0, "second": 1e3, "s": 1e3}.get(unit, 1.0)
            name = "ms"
        elif name.startswith("dram__bytes"):
            v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
        per.setdefault(key, {})[name] = v
    return per


def summarise(per, skip: int = 0):
    by = defaultdict(list)
    for (_, k), m in per.items():
        by[k].append(m)
    out = OrderedDict()
    total = 0.0
    for k, ms in by.items():
        ms = ms[skip:] or ms
        n = len(ms)
        t = sum(m.get("ms", 0.0) for m in ms) / n
        rd = sum(m.get("dram__bytes_read.sum", 0.0) for m in ms) / n
        wr = sum(m.get("dram__bytes_write.sum", 0.0) for m in ms) / n
        out[k] = {"launches": n, "mean_ms": t, "dram_read_bytes": rd, "dram_write_bytes": wr}
        total += t * n
    for k, v in out.items():
        v["share"] = v["mean_ms"] * v["launches"] / total if total else 0.0
    return out


def main():
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    s = summarise(load(path), skip)
    print("| kernel | launches | mean ms | share | DRAM read MB | DRAM write MB | GB/s |")
    print("|---|---|---|---|---|---|---|")
    for k, v in sorted(s.items(), key=lambda kv: -kv[1]["share"]):
        gbs = (v["dram_read_bytes"] + v["dram_write_bytes"]) / (v["mean_ms"] * 1e6) if v["mean_ms"] else 0
        print(f"| {k} | {v['launches']} | {v['mean_ms']:.4f} | {100 * v['share']:.1f}% | "
              f"{v['dram_read_bytes'] / 1e6:.1f} | {v['dram_write_bytes'] / 1e6:.1f} | {gbs:.0f} |")
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump({"source": path, "skip": skip, "kernels": s}, f, indent=1)


if __name__ == "__main__":
    main()
