"""Summarise a gpurun_out/<dir> round profile into profiles/<round>/ (launch shares, ncu key metrics).

Usage: python scripts/summarize_profiles.py gpurun_out/round profiles/r01
"""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) > vi:
            agg[r[ki][:90]][0] += 1
            agg[r[ki][:90]][1] += float(r[vi].replace(",", ""))
    tot = sum(v for _, v in agg.values())
    with open(dst, "w") as fh:
        fh.write("# ncu --metrics gpu__time_duration.sum --clock-control none, python bench.py --steps 1 --warmup 3\n")
        fh.write("# (cold-cache, serialised launches of the whole process: compare SHARES, not absolute times)\n")
        fh.write("# launches  total_us  avg_us  share  kernel\n")
        for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
            fh.write(f"{n:6d} {v / 1e3:11.1f} {v / n / 1e3:9.1f} {100 * v / tot:5.1f}%  {k}\n")


def ncu_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:120]}
        for k in KEYS:
            if k in h:
                d[k] = f"{r[h.index(k)]} {u[h.index(k)]}".strip()
        res.append(d)
    return res


def main():
    src, dst = sys.argv[1], sys.argv[2]
    os.makedirs(dst, exist_ok=True)
    for f in os.listdir(src):
        if f.endswith(".json") or f.endswith(".jsonl") or f in ("smi.txt",):
            shutil.copy(os.path.join(src, f), os.path.join(dst, f))
    if os.path.exists(os.path.join(src, "launches.csv")):
        launches(os.path.join(src, "launches.csv"), os.path.join(dst, "launches_summary.txt"))
    summary = {}
    for f in sorted(os.listdir(src)):
        if f.endswith(".ncu-rep"):
            summary[f[:-8]] = ncu_metrics(os.path.join(src, f))
            det = subprocess.run(["ncu", "-i", os.path.join(src, f), "--page", "details", "--csv"],
                                 capture_output=True, text=True).stdout
            with open(os.path.join(dst, f[:-8] + "_ncu_details.csv"), "w") as fh:
                fh.write(det)
    with open(os.path.join(dst, "ncu_summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary, indent=1)[:4000])


if __name__ == "__main__":
    main()
