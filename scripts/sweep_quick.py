"""C4 attention sweep alone (bench.attention_sweep), one JSON line per point."""
import json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_2312_17649_b200 as P

hbm, tf, _, _ = bench.peaks()
res = bench.attention_sweep(P, torch.device("cuda"), (hbm, tf))
for pt in res["points"]:
    print(json.dumps(pt))
res = bench.attention_sweep(P, torch.device("cuda"), (hbm, tf), d=32,
                            windows=(("sparse", 4), ("sparse", 64), ("sparse", 256)))
for pt in res["points"]:
    print(json.dumps(dict(pt, d=32)))
