"""bench.fp32_variant alone: the ranking-exact fp32 modes at 32 x s=4099 (pairs/s + parity)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
import paper_2312_17649_b200 as P
res = bench.fp32_variant(P, torch.device("cuda"), int(sys.argv[1]) if len(sys.argv) > 1 else 5)
for m in ("f16x3", "bf16x6", "sgemm"):
    print(m, round(res[m]["value"], 1), res[m]["parity"])
