"""Summarise an ncu --csv launch list: per kernel (name + grid), launches, total / mean device
time, dram bytes per launch and achieved GB/s.  Usage: python scripts/ncu_summary.py launches.csv"""
import csv
import io
import sys
from collections import OrderedDict


def load(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    out = OrderedDict()
    for r in rows:
        key = (r["Kernel Name"].split("(")[0].replace("void ", "")[:60], r.get("Grid Size", ""))
        lid = r["ID"]
        d = out.setdefault(key, {})
        e = d.setdefault(lid, {})
        v = r["Metric Value"].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        unit = r["Metric Unit"]
        scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
                 "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        e[r["Metric Name"]] = v * scale
    return out


def main(path):
    data = load(path)
    tot = sum(e.get("gpu__time_duration.sum", 0.0) for d in data.values() for e in d.values())
    print(f"{'kernel':60s} {'grid':>14s} {'n':>5s} {'ms tot':>8s} {'share':>6s} {'us/launch':>10s} {'MB/launch':>10s} {'GB/s':>8s}")
    for (name, grid), d in sorted(data.items(), key=lambda kv: -sum(e.get("gpu__time_duration.sum", 0) for e in kv[1].values())):
        t = sum(e.get("gpu__time_duration.sum", 0.0) for e in d.values())
        b = sum(e.get("dram__bytes_read.sum", 0.0) + e.get("dram__bytes_write.sum", 0.0) for e in d.values())
        n = len(d)
        print(f"{name:60s} {grid:>14s} {n:5d} {t*1e3:8.3f} {t/tot:6.1%} {t/n*1e6:10.1f} {b/n/1e6:10.2f} {b/t/1e9 if t else 0:8.0f}")
    print(f"total {tot*1e3:.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
