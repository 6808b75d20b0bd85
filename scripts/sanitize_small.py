"""Small packed batches through every attention kernel + the encoder loop, for compute-sanitizer runs."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_17649_b200 as P  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    H, d = 4, 64
    shapes = [(10, 300), (1, 1), (7, 130), (14, 127), (3, 65)]
    seq = [m + n + 3 for m, n in shapes]
    T = sum(seq)
    x = torch.from_numpy(rng.standard_normal((T, 3 * H * d)).astype(np.float32)).cuda()
    for name, w, algo, dt, qds in [("sparse", 4, "band", torch.bfloat16, 0), ("longformer", 16, "band", torch.bfloat16, 0),
                                   ("sparse", 64, "tc", torch.bfloat16, 0), ("full", math.inf, "tc", torch.bfloat16, 0),
                                   ("qds", 4, "tc", torch.bfloat16, 30), ("sparse", 4, "generic", torch.float32, 0),
                                   ("qds", 4, "generic", torch.float32, 30)]:
        lay = P.PackedLayout.from_lengths(seq, [m + 1 for m, _ in shapes], qds_every=qds)
        xx = x.to(dt)
        P.attend_packed(xx[:, :H * d], xx[:, H * d:2 * H * d], xx[:, 2 * H * d:], lay, P.make_pattern(name, w), H, algo=algo)
        P.attend_packed(xx[:, :H * d], xx[:, H * d:2 * H * d], xx[:, 2 * H * d:], lay, P.make_pattern(name, w), H,
                        algo=algo, rows="head")
        torch.cuda.synchronize()
        print("ok", name, w, algo, flush=True)
    # head_dim 32 (MiniLM heads): band kernel head pairs, tcgen05 zero-padded operands
    x32 = x[:, :3 * H * 32].contiguous()
    for name, w, algo in [("sparse", 4, "band"), ("longformer", 4, "band"), ("sparse", 64, "tc")]:
        lay = P.PackedLayout.from_lengths(seq, [m + 1 for m, _ in shapes])
        xx = x32.to(torch.bfloat16)
        P.attend_packed(xx[:, :H * 32], xx[:, H * 32:2 * H * 32], xx[:, 2 * H * 32:], lay, P.make_pattern(name, w), H,
                        algo=algo)
        torch.cuda.synchronize()
        print("ok d=32", name, w, algo, flush=True)
    # fp32 ranking-exact mode (f16x3 split GEMMs, LayerNorm writing the next GEMM's planes)
    cfg32 = P.EncoderConfig(layers=2, embed_dim=128, heads=2, ff_dim=256, max_positions=400, vocab_size=500,
                            precision="f32")
    m32 = P.CrossEncoder(cfg32, seed=0, fp32_gemm="f16x3")
    m32.score_pairs([(rng.integers(3, 500, size=10), rng.integers(3, 500, size=int(n))) for n in (5, 100, 300)])
    torch.cuda.synchronize()
    print("ok encoder f16x3", flush=True)
    cfg = P.EncoderConfig(layers=2, embed_dim=128, heads=2, ff_dim=256, max_positions=400, vocab_size=500, precision="bf16")
    model = P.CrossEncoder(cfg, seed=0, prune_last_layer=True)
    model.score_pairs([(rng.integers(3, 500, size=10), rng.integers(3, 500, size=int(n))) for n in (5, 100, 300)])
    torch.cuda.synchronize()
    print("ok encoder", flush=True)


if __name__ == "__main__":
    main()
