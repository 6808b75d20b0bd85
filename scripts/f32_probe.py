"""fp32 parity-path throughput probe: ELECTRA-base f32 encoder forward + the generic attention alone."""
import math, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_17649_b200 as P

s = 4099
cfg = P.EncoderConfig(layers=12, embed_dim=768, heads=12, ff_dim=3072, max_positions=s, vocab_size=30522,
                      pattern="sparse", window=4, precision="f32")
model = P.CrossEncoder(cfg, seed=0)
rng = np.random.default_rng(0)
ids = rng.integers(3, cfg.vocab_size, size=(8, s))
part = P.SubsequencePartition((0, 1), (1, 12), (12, s))
batch = P.PackedBatch.from_ids(ids, part)
lay = model.make_layout(batch)
idd = torch.from_numpy(batch.ids).cuda()
for _ in range(2):
    model.encode_packed(idd, lay, check_finite=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    model.encode_packed(idd, lay, check_finite=False)
e1.record(); torch.cuda.synchronize()
print("f32 encoder ms/step (8 x 4099):", e0.elapsed_time(e1) / 3)
T, hd = lay.total_tokens, 768
qkv = torch.randn(T, 3 * hd, device="cuda")
pat = P.sparse_pattern(4)
out = torch.empty(T, hd, device="cuda")
for _ in range(2):
    P.attend_packed(qkv[:, :hd], qkv[:, hd:2 * hd], qkv[:, 2 * hd:], lay, pat, 12, out=out, check=False)
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    P.attend_packed(qkv[:, :hd], qkv[:, hd:2 * hd], qkv[:, 2 * hd:], lay, pat, 12, out=out, check=False)
e1.record(); torch.cuda.synchronize()
print("f32 generic attention ms/layer:", e0.elapsed_time(e1) / 5)
