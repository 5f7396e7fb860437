"""Summarise an ncu --csv launch list: python tools/ncu_csv.py file.csv [last_n_launches]"""
import csv
import io
import sys

txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
rows = list(csv.DictReader(io.StringIO(txt)))
by = {}
for r in rows:
    by.setdefault(r["ID"], {"name": r["Kernel Name"], "grid": r["Grid Size"]})[r["Metric Name"]] = r["Metric Value"]
ids = sorted(by, key=int)
if len(sys.argv) > 2:
    ids = ids[-int(sys.argv[2]):]
for i in ids:
    d = by[i]
    name = d.pop("name").split("(")[0][:48]
    grid = d.pop("grid")
    print(f"{i:>4} {name:<48} {grid:<14} " + "  ".join(f"{k.split('__')[1] if '__' in k else k}={v}" for k, v in d.items()))
