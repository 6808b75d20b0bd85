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


def gen_ranking():
    """1 query x RANK_DOCS candidates at s=4099, f32 reference scores (ranking.npz).  Candidates 0
    and 1 are encoder.npz's electra_doc_scores pairs (the bench's first two pairs)."""
    cfg = E.EncoderConfig(**cases.ELECTRA_DOC, precision="f32")
    model = E.CrossEncoder(cfg, seed=0)
    seqs = [rerank_ids(0, 0, j, 10, 4086, cfg.vocab_size, cfg.max_positions) for j in range(cases.RANK_DOCS)]
    ids = np.stack([s.ids for s in seqs])
    scores = []
    for i in range(0, len(seqs), 4):
        t0 = time.time()
        scores.append(model.score(ids[i:i + 4], seqs[0].partition))
        print(f"  ranking docs {i}..{i + 3}: {time.time() - t0:.1f}s", flush=True)
    scores = np.concatenate(scores)
    from sparsecross import evaluation as EV
    order = [int(e.doc_id[1:]) for e in EV.rerank(lambda _q, j: scores[j], None,
                                                   [(f"d{j}", j) for j in range(len(scores))])]
    np.savez_compressed(os.path.join(HERE, "ranking.npz"), scores=scores, order=np.array(order))


def gen_rerank():
    """The reference's own re-rank driver (R/evaluation.py:176-205 with R/encoder.py:535-538 as the
    scorer, driven per query like R/cli.py:224-238) over cases.rerank_workload: TREC run + scores."""
    from sparsecross import evaluation as EV

    cfg = E.EncoderConfig(**cases.ELECTRA_PASSAGE, precision="f32")
    model = E.CrossEncoder(cfg, seed=0)
    entries, raw = [], []
    for qid, qids, cands, top_k in cases.rerank_workload(cfg.vocab_size, cfg.max_positions):
        t0 = time.time()
        got = []

        def scorer(query, doc):
            got.append(-np.inf)  # replaced below unless score_pair raises (the reference's -inf)
            got[-1] = model.score_pair(query, doc)
            return got[-1]

        entries += EV.rerank(scorer, qids, cands, top_k=top_k, query_id=qid)
        raw += got
        print(f"  rerank {qid}: {time.time() - t0:.1f}s", flush=True)
    run = EV.format_run(entries)
    np.savez_compressed(os.path.join(HERE, "rerank.npz"), run=np.array(run), scores=np.array(raw, np.float64))


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


def _group_backward_full(pt, qkv, pat, scale, pad, grad_out):
    """dq/dk/dv (heads, s, d) through the reference's group adjoints, assembled like
    layer_backward (R/encoder.py:421-435)."""
    spans = {g: pt.span(g) for g in A.GROUPS}
    caches = {g: A.group_attention(qkv, g, pat, scale, pad, want_cache=True)[1] for g in A.GROUPS}
    shape = grad_out.shape
    dq, dk, dv = np.zeros(shape, grad_out.dtype), np.zeros(shape, grad_out.dtype), np.zeros(shape, grad_out.dtype)
    for g in A.GROUPS:
        lo, hi = spans[g]
        gq, contribs = A.group_attention_backward(caches[g], grad_out[..., lo:hi, :], g, pat)
        dq[..., lo:hi, :] += gq
        for target, idx, gk, gv in contribs:
            t0, t1 = spans[target]
            if idx is None:
                dk[..., t0:t1, :] += gk
                dv[..., t0:t1, :] += gv
            else:
                dk[..., t0 + idx, :] += gk
                dv[..., t0 + idx, :] += gv
    return dq, dk, dv


def gen_training():
    """Backward / training fixtures from the reference's own adjoints and trainer."""
    from sparsecross import training as TR

    out = {}
    # band adjoints (R/band.py:239-274)
    for i, case in enumerate(cases.BAND_CASES):
        s, t, w, d = case
        q, k, p, v = cases.band_inputs(i, case)
        gb, go = cases.band_grad_inputs(i, case)
        out[f"band_gq_{i}"], out[f"band_gk_{i}"] = B.band_scores_backward(gb, q, k, w)
        out[f"band_gp_{i}"], out[f"band_gv_{i}"] = B.band_apply_backward(go, p, v, w)
    # attention adjoints over every ATTN_CASE (R/attention.py:260-269, :348-378, :476-507)
    for i, case in enumerate(cases.ATTN_CASES):
        name, w, pad, m, n, heads, d, dt = case
        x = cases.attn_inputs(i, case)
        go = cases.attn_grad_out(i, case)
        pt = part(m, n)
        qkv = {g: tuple(a[:, lo:hi, :] for a in x) for g, (lo, hi) in zip(A.GROUPS, cases.attn_spans(m, n))}
        pat = A.make_pattern(name, w, cases.attn_globals(name, m, n))
        dq, dk, dv = _group_backward_full(pt, qkv, pat, math.sqrt(d), pad, go)
        big = dq.size > 8000  # large cases: 4 random projections per row (cases.grad_projection)
        for tag, g in (("dq", dq), ("dk", dk), ("dv", dv)):
            out[f"attn_{tag}_{i}"] = g @ cases.grad_projection(i, d) if big else g
    # encoder weight gradients (R/encoder.py:511-533), tiny configs, every pattern x padding, f64
    for name in ("full", "longformer", "qds", "sparse"):
        for pad in ("exclude", "zero-logit"):
            cfg = E.EncoderConfig(**cases.TINY, pattern=name, padding=pad, precision="f64")
            model = E.CrossEncoder(cfg, seed=15)
            seqs = [E.assemble_input(*cases.tiny_sequence(16 + j, 4, 13, cfg.vocab_size), cfg.max_positions)
                    for j in range(2)]
            ids = np.stack([sq.ids for sq in seqs])
            scores, cache = model.score(ids, seqs[0].partition, want_cache=True)
            grads = model.backward(cache, cases.TRAIN_GRAD_SCORES)
            key = f"grad_{name}_{pad}"
            out[key + "_scores"] = scores
            for wn, g in grads.items():
                out[f"{key}|{wn}"] = np.asarray(g)
    # trainer: task sampling, AdamW, a short train_toy run (R/training.py:79-357)
    task = TR.SyntheticTask(**cases.TASK)
    rng = np.random.default_rng(3)
    trip = [task.sample_triple(rng) for _ in range(5)]
    out["task_triples"] = np.array([list(t.query) + list(t.positive) + list(t.negative) for t in trip])
    val = task.sample_validation(np.random.default_rng(4), 2, per_level=2)
    out["task_val"] = np.array([[int(dj[1:]) for dj, _ in vq.candidates] for vq in val])
    out["task_val_docs"] = np.array([[list(doc) for _, doc in vq.candidates] for vq in val])
    ws, gs = cases.adamw_inputs()
    opt = TR.AdamW(lr=0.05, weight_decay=0.1, warmup_steps=2, total_steps=6)
    for step in range(5):
        opt.step(ws, gs[step])
    for n, a in ws.items():
        out[f"adamw|{n}"] = a
    for pattern, window in (("full", 4), ("sparse", 1), ("qds", 4)):
        cfg = E.EncoderConfig(**cases.task_config_kw(pattern, window), precision="f32")
        res = TR.train_toy(cfg, task, steps=3, lr=1e-3, seed=0, batch_pairs=4)
        key = f"toy_{pattern}_{window}"
        out[key + "_loss"] = np.array([r.loss for r in res.trace])
        for wn, a in res.model.weights.items():
            out[f"{key}|{wn}"] = a
    np.savez_compressed(os.path.join(HERE, "training.npz"), **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-long", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    steps = {"band": gen_band, "masks": gen_masks, "attention": gen_attention,
             "encoder": lambda: gen_encoders(args.skip_long), "serialize": gen_serialize,
             "training": gen_training, "ranking": gen_ranking, "rerank": gen_rerank}
    for name, fn in steps.items():
        if args.only and name not in args.only.split(","):
            continue
        t0 = time.time()
        fn()
        print(f"{name}: {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
