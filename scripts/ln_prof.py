"""ResidualLayerNorm fwd+bwd at the fine-tuning shape (32,792 x 768, a fp32 + b bf16) for ncu."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_17649_b200.training import ResidualLayerNorm, column_sum

rows, cols = 32792, 768
a = torch.randn(rows, cols, device="cuda").requires_grad_(True)
b = torch.randn(rows, cols, device="cuda").bfloat16().requires_grad_(True)
g = torch.ones(cols, device="cuda", requires_grad=True)
be = torch.zeros(cols, device="cuda", requires_grad=True)
dy = torch.randn(rows, cols, device="cuda")
x16 = torch.randn(rows, 3072, device="cuda").bfloat16()
for _ in range(3):
    ResidualLayerNorm.apply(a, b, g, be).backward(dy)
    column_sum(x16)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
e[0].record()
y = ResidualLayerNorm.apply(a, b, g, be)
e[1].record()
y.backward(dy)
e[2].record()
column_sum(x16)
e[3].record()
torch.cuda.synchronize()
print("fwd %.1f us, bwd %.1f us, colsum(32792x3072 bf16) %.1f us" % tuple(1000 * e[i].elapsed_time(e[i + 1]) for i in range(3)))
