"""C4 attention sweep alone (bench.attention_sweep), one JSON line per point.
SWEEP_TC_ONLY=1: only the tcgen05-regime windows (64, 256, inf, full) at d=64 and d=32."""
import json, math, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_2312_17649_b200 as P

hbm, tf, _, _ = bench.peaks()
tc_only = os.environ.get("SWEEP_TC_ONLY") == "1"
wins = ((("sparse", 64), ("sparse", 256), ("sparse", math.inf), ("full", math.inf)) if tc_only else
        (("sparse", 1), ("sparse", 4), ("sparse", 16), ("sparse", 64), ("sparse", 256), ("sparse", math.inf),
         ("full", math.inf)))
res = bench.attention_sweep(P, torch.device("cuda"), (hbm, tf), windows=wins)
for pt in res["points"]:
    print(json.dumps(pt))
wins32 = (("sparse", 64), ("sparse", 256)) if tc_only else (("sparse", 4), ("sparse", 64), ("sparse", 256))
res = bench.attention_sweep(P, torch.device("cuda"), (hbm, tf), d=32, windows=wins32)
for pt in res["points"]:
    print(json.dumps(dict(pt, d=32)))
