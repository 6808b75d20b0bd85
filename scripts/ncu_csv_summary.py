"""Summarise an ncu --metrics gpu__time_duration.sum --csv log: per kernel, launches and last time (us)."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    lines = [l for l in open(path) if l.startswith('"')]
    seen = collections.OrderedDict()
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            seen.setdefault(r["Kernel Name"].split("(")[0][:70], []).append(float(r["Metric Value"]) / 1e3)
    print(path)
    for k, v in seen.items():
        print(f"  {len(v):3d} x  last {v[-1]:8.1f} us  {k}")
