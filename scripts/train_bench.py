"""Fine-tuning step timing: ELECTRA-base dims, packed pairs, bf16 autocast.

Times (CUDA events, after warm-up) the forward with autograd, the backward,
the AdamW step, and the attention adjoint alone at the same shapes, and
prints one JSON line.

    python scripts/train_bench.py --doc-len 4086 --pairs 4 --steps 5
"""

import argparse
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_17649_b200 as P  # noqa: E402
from paper_2312_17649_b200 import training as TR  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--doc-len", type=int, default=4086)
    ap.add_argument("--query-len", type=int, default=10)
    ap.add_argument("--pairs", type=int, default=4)
    ap.add_argument("--window", type=float, default=4)
    ap.add_argument("--pattern", default="sparse")
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--graph", action="store_true", help="CUDA-graph forward+backward (GraphedTrainStep)")
    a = ap.parse_args()
    w = math.inf if a.window == math.inf else int(a.window)
    s = a.query_len + a.doc_len + 3
    cfg = P.EncoderConfig(layers=a.layers, embed_dim=768, heads=12, ff_dim=3072, max_positions=s,
                          vocab_size=30522, pattern=a.pattern, window=w, precision=a.precision)
    model = TR.TrainableCrossEncoder(cfg, seed=0)
    opt = TR.AdamW(1e-5, moment_dtype=torch.float32)
    rng = np.random.default_rng(0)
    n = 2 * a.pairs
    ids = rng.integers(3, cfg.vocab_size, size=(n, s))
    ids[:, 0] = 1
    ids[:, a.query_len + 1] = 2
    ids[:, -1] = 2
    part = P.SubsequencePartition((0, 1), (1, a.query_len + 2), (a.query_len + 2, s))
    batch = P.PackedBatch.from_ids(ids, part)
    layout = model.make_layout(batch)
    ids_dev = torch.from_numpy(batch.ids).cuda()
    teacher = torch.randn(n, device="cuda", dtype=torch.float64)
    names = sorted(model.weights)

    graphed = None
    if a.graph:
        graphed = TR.GraphedTrainStep(model, opt, batch)
        gap = (teacher[:a.pairs] - teacher[a.pairs:]).cpu().numpy()

    def step(times=None):
        e = [ev() for _ in range(4)]
        if graphed is not None:
            e[0].record()
            graphed.graph.replay()
            e[1].record()
            e[2].record()
            W = model.weights
            grads, off = TR.GradDict(graphed.grad_flat), 0
            for n in names:
                k = W[n].numel()
                grads[n] = graphed.grad_flat[off:off + k].view(W[n].shape)
                off += k
            opt.step(W, grads)
            e[3].record()
            if times is not None:
                times.append(e)
            return
        e[0].record()
        scores = model.score_packed(ids_dev, layout, check_finite=False)
        gap = (scores[:a.pairs].double() - scores[a.pairs:].double()) - (teacher[:a.pairs] - teacher[a.pairs:])
        loss = torch.mean(gap * gap)
        e[1].record()
        with model.gemm_mode():
            grads = torch.autograd.grad(loss, [model.weights[k] for k in names], allow_unused=True)
        e[2].record()
        opt.step(model.weights, {k: (torch.zeros_like(model.weights[k]) if g is None else g)
                                 for k, g in zip(names, grads)})
        e[3].record()
        if times is not None:
            times.append(e)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    times = []
    for _ in range(a.steps):
        step(times)
    torch.cuda.synchronize()
    fwd = float(np.median([t[0].elapsed_time(t[1]) for t in times]))
    bwd = float(np.median([t[1].elapsed_time(t[2]) for t in times]))
    optm = float(np.median([t[2].elapsed_time(t[3]) for t in times]))
    total = float(np.median([t[0].elapsed_time(t[3]) for t in times]))

    # attention adjoint alone at the same shapes (one layer)
    T, hd = layout.total_tokens, cfg.embed_dim
    dt = torch.bfloat16 if a.precision == "bf16" else torch.float32
    qkv = torch.randn(T, 3 * hd, device="cuda").to(dt)
    out = P.attend_packed(qkv[:, :hd], qkv[:, hd:2 * hd], qkv[:, 2 * hd:], layout, model.pattern, cfg.heads)
    dout = torch.randn(T, hd, device="cuda").to(dt)
    g = torch.empty(T, 3 * hd, device="cuda")
    for _ in range(3):
        TR.attention_backward(qkv, out, dout, g, layout, model.pattern, cfg.heads, 8.0, cfg.padding)
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(10):
        TR.attention_backward(qkv, out, dout, g, layout, model.pattern, cfg.heads, 8.0, cfg.padding)
    e1.record()
    torch.cuda.synchronize()
    attn_bwd = e0.elapsed_time(e1) / 10
    e0.record()
    for _ in range(10):
        P.attend_packed(qkv[:, :hd], qkv[:, hd:2 * hd], qkv[:, 2 * hd:], layout, model.pattern, cfg.heads,
                        out=out, check=False)
    e1.record()
    torch.cuda.synchronize()
    attn_fwd = e0.elapsed_time(e1) / 10
    es = qkv.element_size()
    bytes_bwd = T * hd * (5 * es + 3 * 4) + T * cfg.heads * 8  # q,k,v,o,dO in; dq,dk,dv fp32 out; stats
    print(json.dumps({
        "metric": "finetune_step", "graph": a.graph, "tokens": T, "pairs": a.pairs, "seq_len": s, "pattern": a.pattern,
        "window": a.window, "precision": a.precision, "layers": a.layers,
        "ms_step": total, "ms_forward": fwd, "ms_backward": bwd, "ms_adamw": optm,
        "tokens_per_s": T / total * 1e3, "pairs_per_s": n / total * 1e3,
        "attn_bwd_ms_per_layer": attn_bwd, "attn_fwd_ms_per_layer": attn_fwd,
        "attn_bwd_share_of_backward": attn_bwd * a.layers / bwd,
        "attn_bwd_GBps_algorithmic": bytes_bwd / attn_bwd / 1e6,
    }))


if __name__ == "__main__":
    main()
