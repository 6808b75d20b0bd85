"""fp32 modes at the headline documents: time per 32-pair step and parity vs the reference golden."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
import paper_2312_17649_b200 as P
print(json.dumps(bench.fp32_variant(P, torch.device("cuda"), 3), indent=1))
