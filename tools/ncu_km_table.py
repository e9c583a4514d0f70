"""Print the per-launch metrics of gpurun_out/ncu_km<V>.csv (ncu --csv --metrics ... of the keymult launches)."""
import csv
import io
import sys

for km in sys.argv[1:]:
    txt = open(f"gpurun_out/ncu_km{km}.csv").read()
    txt = txt[txt.index('"ID"'):]
    by = {}
    for r in csv.DictReader(io.StringIO(txt)):
        by.setdefault(r["ID"], {})[r["Metric Name"]] = r["Metric Value"]
    for i, m in list(by.items())[:4]:
        print(km, i, {k.split(".")[0][-28:]: v for k, v in m.items()})
