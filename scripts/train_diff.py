"""Per-weight differences of a short train_toy run vs the reference trainer fixture."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests", "golden")]
import cases
import paper_2312_17649_b200 as P
G = np.load(os.path.join(ROOT, "tests", "golden", "training.npz"))
for pattern, window in (("full", 4), ("sparse", 1)):
    cfg = P.EncoderConfig(**cases.task_config_kw(pattern, window), precision="f32")
    res = P.train_toy(cfg, P.SyntheticTask(**cases.TASK), steps=3, lr=1e-3, seed=0, batch_pairs=4)
    key = f"toy_{pattern}_{window}"
    print(key, [r.loss for r in res.trace], G[key + "_loss"])
    init = P.init_weights(cfg, 0)
    for wn, t in sorted(res.model.weights.items()):
        a = t.detach().cpu().numpy(); b = G[f"{key}|{wn}"]
        print(f"{wn:10s} maxdiff {np.abs(a-b).max():.3e}  moved ours {np.abs(a-init[wn]).max():.2e} ref {np.abs(b-init[wn]).max():.2e}")
