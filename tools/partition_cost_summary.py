"""Reduce an ncu launch list (gpu__time_duration.sum csv) of
tools/partition_cost.py to mean per-kernel microseconds over the saturated
steps: python tools/partition_cost_summary.py launches.csv G [skip_steps]"""
import csv
import sys
from collections import defaultdict

path, G = sys.argv[1], int(sys.argv[2])
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 10
rows = []
with open(path) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        rows.append((r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", ""), float(r["Metric Value"].replace(",", ""))))
# per step: G x k_neuron, then G x (k_hist, sweep)
per = defaultdict(list)
for name, v in rows:
    per[name].append(v)
unit = "ns"
for name, vals in per.items():
    steady = vals[skip * G:] if len(vals) > skip * G else vals
    print(f"{name:28s} launches {len(vals):5d}  mean(steady) {sum(steady) / max(1, len(steady)) / 1000:8.2f} us")
