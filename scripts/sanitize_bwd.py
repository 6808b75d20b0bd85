"""Small fine-tuning-path workload for compute-sanitizer (memcheck / racecheck / synccheck).

Runs the attention adjoint on the tiled path (bf16, d=64, sparse/longformer, both paddings), the
generic path (fp32, QDS, d=32), the LayerNorm / GELU / colsum kernels and two fused AdamW steps.
"""
import math, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_17649_b200 as P
from paper_2312_17649_b200 import training as TR

rng = np.random.default_rng(0)
for pattern, w, pad, dt, d, qds in [("sparse", 4, "exclude", torch.bfloat16, 64, 0),
                                    ("longformer", 16, "zero-logit", torch.bfloat16, 64, 0),
                                    ("sparse", 2, "zero-logit", torch.float32, 32, 0),
                                    ("qds", 4, "exclude", torch.float32, 32, 7)]:
    m = rng.integers(1, 12, size=3)
    n = rng.integers(1, 150, size=3)
    if qds == 0 and pad == "exclude":
        n = np.array([1200, 900, 40])  # long rows: 2-warp head-row CTAs with the key split, scalar partial reduce
    lay = P.PackedLayout.from_lengths(m + n + 3, m + 1, device="cuda", qds_every=qds)
    pat = P.make_pattern(pattern, w)
    H = 2
    T = lay.total_tokens
    qkv = torch.randn(T, 3 * H * d, device="cuda").to(dt).requires_grad_(True)
    out = TR.PatternAttention.apply(qkv, lay, pat, H, math.sqrt(d), pad, True)
    out.backward(torch.randn_like(out))
x = torch.randn(300, 96, device="cuda").requires_grad_(True)
b = torch.randn(300, 96, device="cuda").bfloat16().requires_grad_(True)
g = torch.ones(96, device="cuda", requires_grad=True)
be = torch.zeros(96, device="cuda", requires_grad=True)
y, y16 = TR.ResidualLayerNorm.apply(x, b, g, be, True)
(y.sum() + y16.float().sum()).backward()
w1 = torch.randn(96, 128, device="cuda", requires_grad=True)
b1 = torch.zeros(128, device="cuda", requires_grad=True)
TR.LinearGelu.apply(x.detach().bfloat16(), w1, None, b1, None, torch.bfloat16).float().sum().backward()
TR.column_sum(torch.randn(77, 40, device="cuda"))
cfg = P.EncoderConfig(layers=1, embed_dim=64, heads=1, ff_dim=128, max_positions=64, vocab_size=50,
                      pattern="sparse", window=2, precision="bf16")
model = TR.TrainableCrossEncoder(cfg, seed=0)
opt = TR.AdamW(1e-3)
task = TR.SyntheticTask(vocab_words=12, query_terms=2, doc_len=6)
for _ in range(2):
    TR.train_step(model, opt, [task.sample_triple(rng) for _ in range(2)])
torch.cuda.synchronize()
print("sanitize_bwd workload done")
