"""Summarise an ncu launch-list CSV (gpu__time_duration.sum [+ dram bytes]) by kernel.

    python tools/launch_table.py gpurun_out/launches.csv [--last-frac 0.5] [--only ck]
"""
import collections
import csv
import io
import sys


def load(path):
    text = open(path).read()
    i = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[i:])))
    per = collections.OrderedDict()
    for r in rows:
        k = (int(r["ID"]), r["Kernel Name"], r["Grid Size"])
        unit = r["Metric Unit"]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                 "Gbyte": 1e9}.get(unit, 1.0)
        per.setdefault(k, {})[r["Metric Name"]] = v * scale
    return per


def short(name):
    base = name.split("(")[0]
    return base.replace("void ", "").replace("ck::", "").replace("<unnamed>::", "")[:48]


def main():
    path = sys.argv[1]
    frac = 0.5
    if "--last-frac" in sys.argv:
        frac = float(sys.argv[sys.argv.index("--last-frac") + 1])
    per = load(path)
    items = list(per.items())
    items = items[int(len(items) * (1 - frac)):]
    agg = collections.OrderedDict()
    for (i, name, grid), m in items:
        a = agg.setdefault(short(name), {"n": 0, "us": 0.0, "rd": 0.0, "wr": 0.0})
        a["n"] += 1
        a["us"] += m.get("gpu__time_duration.sum", 0)
        a["rd"] += m.get("dram__bytes_read.sum", 0)
        a["wr"] += m.get("dram__bytes_write.sum", 0)
    tot = sum(a["us"] for a in agg.values())
    print(f"{'kernel':48s} {'n':>4s} {'us':>9s} {'share':>6s} {'dram GB/s':>9s}")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        bw = (a["rd"] + a["wr"]) / (a["us"] * 1e3) if a["us"] else 0
        print(f"{k:48s} {a['n']:4d} {a['us']:9.1f} {a['us'] / tot:6.3f} {bw:9.1f}")
    print(f"{'total':48s} {'':4s} {tot:9.1f}")


if __name__ == "__main__":
    main()
