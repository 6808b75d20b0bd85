"""Probe: fp32 bf16x6 headline scores vs the reference golden at several main-product K-chunks."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import cases
import paper_2312_17649_b200 as P
from paper_2312_17649_b200 import encoder as E

ref = np.load(os.path.join(ROOT, "tests/golden/ranking.npz"))["scores"]
cfg = P.EncoderConfig(**cases.ELECTRA_DOC, precision="f32")
seqs = []
for j in range(len(ref)):
    q = np.random.default_rng((0, 0)).integers(3, cfg.vocab_size, size=10)
    d = np.random.default_rng((0, 0, j)).integers(3, cfg.vocab_size, size=4086)
    seqs.append(P.assemble_input(q, d, cfg.max_positions))
batch = P.PackedBatch.from_sequences(seqs)
order = sorted(range(len(ref)), key=lambda j: (-ref[j], j))
for mode, chunk in (("sgemm", 0), ("bf16x6", 768), ("bf16x6", 384), ("bf16x6", 256), ("bf16x6", 128)):
    E.X6_CHUNK = chunk or 768
    m = P.CrossEncoder(cfg, seed=0, fp32_gemm=mode)
    sc = m.score_packed(batch).cpu().numpy()
    o = sorted(range(len(sc)), key=lambda j: (-sc[j], j))
    lay = m.make_layout(batch); ids = torch.from_numpy(batch.ids).cuda()
    fn = lambda: m.scores_from_hidden(m.encode_packed(ids, lay), lay)
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); fn(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 2
    print(f"{mode} chunk {chunk}: max |d| {np.abs(sc - ref).max():.3e} mean {np.abs(sc-ref).mean():.3e} "
          f"ranking identical {o == order}; {ms:.1f} ms / {len(ref)} pairs = {len(ref) / ms * 1e3:.1f} pairs/s", flush=True)
    del m; torch.cuda.empty_cache()
