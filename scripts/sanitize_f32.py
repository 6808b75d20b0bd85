"""fp32 parity-path attention (band_f32_kernel + generic head rows with records) for compute-sanitizer."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_17649_b200 as P

rng = np.random.default_rng(1)
for pattern, w, pad in [("sparse", 4, "exclude"), ("longformer", 8, "zero-logit"), ("sparse", 0, "zero-logit"),
                        ("sparse", 32, "exclude")]:
    m = rng.integers(1, 20, size=4)
    n = np.concatenate([rng.integers(1, 200, size=3), [130]])
    lay = P.PackedLayout.from_lengths(m + n + 3, m + 1, device="cuda")
    H, d = 2, 64
    T = lay.total_tokens
    x = torch.randn(T, 3 * H * d, device="cuda")
    P.attend_packed(x[:, :H * d], x[:, H * d:2 * H * d], x[:, 2 * H * d:], lay, P.make_pattern(pattern, w), H,
                    padding=pad)
torch.cuda.synchronize()
print("sanitize_f32 workload done")
