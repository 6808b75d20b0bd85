"""Top CUDA kernels of one fine-tuning step (torch.profiler), ELECTRA dims, bf16.

    python scripts/train_profile.py [--nseq 8 --doc-len 4086]   (passages: --nseq 64 --doc-len 164)
"""
import argparse, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_17649_b200 as P
from paper_2312_17649_b200 import training as TR

ap = argparse.ArgumentParser()
ap.add_argument("--nseq", type=int, default=8)
ap.add_argument("--doc-len", type=int, default=4086)
a = ap.parse_args()
s = a.doc_len + 13
cfg = P.EncoderConfig(layers=12, embed_dim=768, heads=12, ff_dim=3072, max_positions=s, vocab_size=30522,
                      pattern="sparse", window=4, precision="bf16")
model = TR.TrainableCrossEncoder(cfg, seed=0)
opt = TR.AdamW(1e-5)
rng = np.random.default_rng(0)
ids = rng.integers(3, cfg.vocab_size, size=(a.nseq, s))
part = P.SubsequencePartition((0, 1), (1, 12), (12, s))
batch = P.PackedBatch.from_ids(ids, part)
layout = model.make_layout(batch)
ids_dev = torch.from_numpy(batch.ids).cuda()
names = sorted(model.weights)


def step():
    sc = model.score_packed(ids_dev, layout, check_finite=False)
    loss = ((sc[:a.nseq // 2] - sc[a.nseq // 2:]) ** 2).mean()
    with model.gemm_mode():
        gr = torch.autograd.grad(loss, [model.weights[n] for n in names])
    opt.step(model.weights, dict(zip(names, gr)))


for _ in range(3):
    step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=70))
if os.environ.get("CAT_SHAPES"):
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], record_shapes=True) as prof2:
        step()
        torch.cuda.synchronize()
    print(prof2.key_averages(group_by_input_shape=True).table(sort_by="cuda_time_total", row_limit=25,
                                                               max_name_column_width=30, max_shapes_column_width=120))
