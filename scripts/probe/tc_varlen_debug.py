"""Debug: which (head, row) of the packed varlen w=64 case differ between the tc kernel and the oracle."""
import math, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import paper_2312_17649_b200 as P
from oracle import sparsecross_oracle as O
from golden import cases
rng = np.random.default_rng(11)
H, d = 3, 64
shapes = [(10, 164), (1, 1), (7, 530), (10, 4), (25, 97), (10, 64)]
if len(sys.argv) > 1: shapes = eval(sys.argv[1])
seq = [m + n + 3 for m, n in shapes]
lay = P.PackedLayout.from_lengths(seq, [m + 1 for m, _ in shapes], device="cuda")
T = sum(seq)
x = torch.from_numpy(rng.standard_normal((T, 3 * H * d)).astype(np.float32)).cuda().to(torch.bfloat16)
pat = P.make_pattern("sparse", 64)
out = P.attend_packed(x[:, :H * d], x[:, H * d:2 * H * d], x[:, 2 * H * d:], lay, pat, H, algo=os.environ.get("ALGO", "auto")).double().cpu().numpy()
xin = x.double().cpu().numpy().reshape(T, 3, H, d)
r = 0
for (m, n), s in zip(shapes, seq):
    blk = xin[r:r + s].transpose(1, 2, 0, 3)
    spans = cases.attn_spans(m, n)
    ref = np.concatenate(O.apply_pattern(spans, O.split_groups(spans, *blk), O.make_pattern("sparse", 64), math.sqrt(d)), axis=-2)
    got = out[r:r + s].reshape(s, H, d).transpose(1, 0, 2)
    err = np.abs(got - ref).max(-1)  # (H, s)
    bad = np.argwhere(err > 0.02)
    print(f"seq m={m} n={n} s={s}: bad rows {len(bad)}", "first:", bad[:10].tolist(), "rows with bad by head:",
          [np.flatnonzero(err[h] > 0.02)[[0, -1]].tolist() if (err[h] > 0.02).any() else None for h in range(H)])
    r += s
