"""sc_attn_fwd at s=4099 x 64 sequences, H=12, d=64: forced band vs tcgen05 kernel per window (us per sequence-layer)."""
import json, math, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2312_17649_b200 as P

nseq, doc, H, d = 64, 4086, 12, 64
s = 10 + doc + 3
T = s * nseq
lay = P.PackedLayout.from_lengths([s] * nseq, [11] * nseq, device="cuda")
g = torch.Generator(device="cuda").manual_seed(0)
qkv = torch.randn((T, 3 * H * d), device="cuda", generator=g).to(torch.bfloat16)
out = torch.empty((T, H * d), device="cuda", dtype=torch.bfloat16)
for w in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "16,32,40,48,64,80,96").split(",")]:
    pat = P.make_pattern("sparse", w)
    row = {"w": w}
    for algo in ("band", "tc"):
        f = lambda: P.attend_packed(qkv[:, :H * d], qkv[:, H * d:2 * H * d], qkv[:, 2 * H * d:], lay, pat, H,
                                    out=out, algo=algo, check=False)
        try:
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                f()
            e1.record()
            torch.cuda.synchronize()
            row[algo] = round(e0.elapsed_time(e1) / 10 * 1e3 / nseq, 2)
        except Exception as ex:
            row[algo] = str(ex)[:60]
    print(json.dumps(row), flush=True)
