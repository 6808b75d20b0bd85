"""One sc_attn_fwd configuration, for ncu launch lists / full captures (C4 shapes)."""
import argparse, math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_17649_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--nseq", type=int, default=64)
ap.add_argument("--doc", type=int, default=4086)
ap.add_argument("--w", default="4")
ap.add_argument("--pattern", default="sparse")
ap.add_argument("--heads", type=int, default=12)
ap.add_argument("--d", type=int, default=64)
ap.add_argument("--qlen", type=int, default=10)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--algo", default="auto")
a = ap.parse_args()
w = math.inf if a.w == "inf" else int(a.w)
s = a.qlen + a.doc + 3
T = s * a.nseq
H, d = a.heads, a.d
lay = P.PackedLayout.from_lengths([s] * a.nseq, [a.qlen + 1] * a.nseq)
g = torch.Generator(device="cuda").manual_seed(0)
qkv = torch.randn((T, 3 * H * d), device="cuda", generator=g).to(torch.bfloat16)
out = torch.empty((T, H * d), device="cuda", dtype=torch.bfloat16)
pat = P.make_pattern(a.pattern, w)
for _ in range(a.iters):
    P.attend_packed(qkv[:, :H * d], qkv[:, H * d:2 * H * d], qkv[:, 2 * H * d:], lay, pat, H, out=out,
                    algo=a.algo, check=False)
torch.cuda.synchronize()
