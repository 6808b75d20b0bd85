"""One attention-adjoint call at ELECTRA-base dims for ncu (pairs x s=4099, sparse w=4, bf16)."""
import argparse, math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_17649_b200 as P
from paper_2312_17649_b200 import training as TR

ap = argparse.ArgumentParser()
ap.add_argument("--nseq", type=int, default=8)
ap.add_argument("--doc-len", type=int, default=4086)
ap.add_argument("--window", type=int, default=4)
ap.add_argument("--pattern", default="sparse")
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
s = 10 + a.doc_len + 3
lay = P.PackedLayout.from_lengths([s] * a.nseq, [11] * a.nseq, device="cuda")
pat = P.make_pattern(a.pattern, a.window)
T, hd, H = lay.total_tokens, 768, 12
qkv = torch.randn(T, 3 * hd, device="cuda").bfloat16()
out = P.attend_packed(qkv[:, :hd], qkv[:, hd:2 * hd], qkv[:, 2 * hd:], lay, pat, H)
dout = torch.randn(T, hd, device="cuda").bfloat16()
g = torch.empty(T, 3 * hd, device="cuda")
for _ in range(a.iters):
    TR.attention_backward(qkv, out, dout, g, lay, pat, H, 8.0, "exclude")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
TR.attention_backward(qkv, out, dout, g, lay, pat, H, 8.0, "exclude")
e1.record(); torch.cuda.synchronize()
print("attn bwd ms", e0.elapsed_time(e1))
