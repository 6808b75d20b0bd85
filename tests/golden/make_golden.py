"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py            # all fixtures
    python tests/golden/make_golden.py --skip-long # skip the s=4099 ELECTRA case

It imports ``sparsecross`` from /root/reference/pkg/src read-only and writes
``tests/golden/*.npz`` (reference outputs only; inputs are regenerated from
the seeds in ``cases.py``).  Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import argparse
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import cases  # noqa: E402
from sparsecross import attention as A  # noqa: E402
from sparsecross import band as B  # noqa: E402
from sparsecross import bench as BE  # noqa: E402
from sparsecross import encoder as E  # noqa: E402
from sparsecross import reference as R  # noqa: E402


def part(m, n):
    return E.SubsequencePartition((0, 1), (1, m + 2), (m + 2, m + n + 3))


def gen_band():
    out = {}
    for i, case in enumerate(cases.BAND_CASES):
        s, t, w, d = case
        q, k, p, v = cases.band_inputs(i, case)
        out[f"scores_{i}"] = B.band_scores(q, k, w)
        out[f"apply_{i}"] = B.band_apply(p, v, w)
        out[f"valid_{i}"] = B.band_validity(s, w, t)
    np.savez_compressed(os.path.join(HERE, "band.npz"), **out)


def gen_masks():
    out = {}
    for i, (name, w, (m, n)) in enumerate(cases.MASK_CASES):
        pat = A.make_pattern(name, w, cases.mask_globals(name, n))
        out[f"mask_{i}"] = np.packbits(R.pattern_mask(pat, part(m, n)))
    np.savez_compressed(os.path.join(HERE, "masks.npz"), **out)


def gen_attention():
    out = {}
    for i, case in enumerate(cases.ATTN_CASES):
        name, w, pad, m, n, heads, d, dt = case
        x = cases.attn_inputs(i, case)
        pt = part(m, n)
        qkv = {g: tuple(a[:, lo:hi, :] for a in x) for g, (lo, hi) in zip(A.GROUPS, cases.attn_spans(m, n))}
        pat = A.make_pattern(name, w, cases.attn_globals(name, m, n))
        outs = A.apply_pattern(pt, qkv, pat, math.sqrt(d), pad)
        out[f"out_{i}"] = np.concatenate(outs, axis=-2)
    np.savez_compressed(os.path.join(HERE, "attention.npz"), **out)


def rerank_ids(seed, qid, j, query_len, doc_len, vocab, max_positions):
    q = np.random.default_rng((seed, qid)).integers(3, vocab, size=query_len)
    d = np.random.default_rng((seed, qid, j)).integers(3, vocab, size=doc_len)
    return E.assemble_input(q, d, max_positions)


def gen_encoders(skip_long):
    out = {}
    # C1 exactly as BASELINE.json configs[0]: reference bench defaults, f32, batch 8.
    spec = BE.BenchSpec("sparse", 4, doc_lens=(164,), batch_size=8, precision="f32")
    cfg = E.EncoderConfig(**cases.C1, precision="f32")
    model = E.CrossEncoder(cfg, seed=0)
    batch = BE.gen_random_batch(spec, 164, cfg)
    out["c1_ids"] = batch.ids
    out["c1_hidden"] = model.forward(batch.ids, batch.partition)
    out["c1_scores"] = model.score(batch.ids, batch.partition)
    fc = BE.flop_count(batch.pattern, (1, 11, 165), 32, 2, 2, 64)
    out["c1_flops"] = np.array([fc.attention, fc.projections, fc.feed_forward, fc.total])
    fc = BE.flop_count(A.sparse_pattern(4), (1, 11, 4087), 768, 12, 12, 3072)
    out["c3_flops"] = np.array([fc.attention, fc.projections, fc.feed_forward, fc.total])
    # Tiny test configs of T/test_encoder.py:199-208, every pattern, both paddings, f64.
    for name in ("full", "longformer", "qds", "sparse"):
        for pad in ("exclude", "zero-logit"):
            cfg = E.EncoderConfig(**cases.TINY, pattern=name, padding=pad, precision="f64")
            model = E.CrossEncoder(cfg, seed=15)
            qy, dc = cases.tiny_sequence(16, 4, 13, cfg.vocab_size)
            seq = E.assemble_input(qy, dc, cfg.max_positions)
            key = f"tiny_{name}_{pad}"
            out[key + "_hidden"] = model.forward(seq.ids, seq.partition)[0]
            out[key + "_score"] = model.score(seq.ids, seq.partition)
            if pad == "exclude":
                resolved = E.resolve_pattern(cfg, seq.partition)
                out[key + "_dense"] = R.reference_encoder_forward(seq.ids, seq.partition, resolved, cfg, model.weights)
    # ELECTRA-base dims, passages (s = 177): one query x 100 candidates, f32.
    cfg = E.EncoderConfig(**cases.ELECTRA_PASSAGE, precision="f32")
    model = E.CrossEncoder(cfg, seed=0)
    seqs = [rerank_ids(0, 0, j, 10, 164, cfg.vocab_size, cfg.max_positions) for j in range(100)]
    ids = np.stack([s.ids for s in seqs])
    t0 = time.time()
    scores = np.concatenate([model.score(ids[i:i + 10], seqs[0].partition) for i in range(0, 100, 10)])
    print(f"electra passage x100: {time.time() - t0:.1f}s", flush=True)
    out["electra_passage_scores"] = scores
    out["electra_passage_cls"] = model.forward(ids[:2], seqs[0].partition)[:, 0, :]
    if not skip_long:
        cfg = E.EncoderConfig(**cases.ELECTRA_DOC, precision="f32")
        model = E.CrossEncoder(cfg, seed=0)
        seqs = [rerank_ids(0, 0, j, 10, 4086, cfg.vocab_size, cfg.max_positions) for j in range(2)]
        ids = np.stack([s.ids for s in seqs])
        t0 = time.time()
        x = model.forward(ids, seqs[0].partition)
        print(f"electra doc x2: {time.time() - t0:.1f}s", flush=True)
        out["electra_doc_cls"] = x[:, 0, :]
        out["electra_doc_scores"] = x[:, 0, :] @ model.weights["head_w"] + model.weights["head_b"]
        out["electra_doc_rowsum"] = x.sum(axis=-1)
    np.savez_compressed(os.path.join(HERE, "encoder.npz"), **out)


def gen_serialize():
    """Model directories written by the reference's save_model (R/serialize.py:50-76)."""
    import math as _m

    from sparsecross import serialize as S

    scores = {}
    for tag, prec, window in (("f64", "f64", 2), ("f32", "f32", 2), ("inf", "f64", _m.inf)):
        cfg = E.EncoderConfig(layers=1, embed_dim=8, heads=2, ff_dim=16, max_positions=32, vocab_size=20,
                              pattern="sparse", window=window, precision=prec)
        model = E.CrossEncoder(cfg, seed=42)
        S.save_model(model, os.path.join(HERE, f"ref_model_{tag}"))
        seq = E.assemble_input([3, 4, 5], [6, 7, 8, 9])
        scores[f"score_{tag}"] = model.score(seq.ids, seq.partition)
    np.savez_compressed(os.path.join(HERE, "serialize.npz"), **scores)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-long", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    steps = {"band": gen_band, "masks": gen_masks, "attention": gen_attention,
             "encoder": lambda: gen_encoders(args.skip_long), "serialize": gen_serialize}
    for name, fn in steps.items():
        if args.only and name not in args.only.split(","):
            continue
        t0 = time.time()
        fn()
        print(f"{name}: {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
