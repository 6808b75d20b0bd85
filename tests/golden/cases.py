"""Seeded case definitions shared by the golden generator and the tests.

Inputs are regenerated from seeds (numpy PCG64 is deterministic for a fixed
numpy version), so fixtures store only the reference OUTPUTS.
"""

from __future__ import annotations

import math

import numpy as np

INF = math.inf

# (s, t, w, d) band-kernel cases; w >= 16 with s >= 2w+1 exercises the
# reference's blocked path (R/band.py:136, :167-168).
BAND_CASES = [
    (1, 1, 0, 3), (5, 5, 0, 4), (7, 5, 2, 3), (6, 9, 1, 5), (12, 12, 4, 8),
    (9, 4, 3, 2), (40, 40, 16, 8), (70, 60, 17, 16), (33, 33, 20, 4), (3, 12, 5, 6),
]

# (pattern, window, (m, n)) -> brute-force mask cases (R/reference.py:30-57).
MASK_CASES = [
    (name, w, mn)
    for name in ("full", "longformer", "qds", "sparse")
    for w in (0, 1, 4, 16, INF)
    for mn in ((1, 4), (3, 9), (4, 11), (10, 95))
]


def mask_globals(name, n):
    return (2, 7) if (name == "qds" and n >= 8) else ()


# Attention cases: (pattern, window, padding, m, n, heads, d, dtype-name).
# m/n are the query/doc token counts: group lengths are 1, m+1, n+1.
ATTN_CASES = []
for _name in ("sparse", "longformer", "full", "qds"):
    for _w in (0, 1, 4):
        for _pad in ("exclude", "zero-logit"):
            ATTN_CASES.append((_name, _w, _pad, 3, 9, 2, 8, "f64"))
for _w in (1, 4, 16, 64, INF):
    ATTN_CASES.append(("sparse", _w, "exclude", 10, 164, 2, 64, "f32"))
ATTN_CASES += [
    ("sparse", 4, "zero-logit", 10, 164, 2, 64, "f32"),
    ("longformer", 4, "exclude", 10, 164, 2, 64, "f32"),
    ("longformer", 64, "zero-logit", 10, 164, 2, 64, "f32"),
    ("full", INF, "exclude", 10, 164, 2, 16, "f32"),
    ("sparse", 4, "exclude", 10, 587, 3, 64, "f32"),
    ("sparse", 256, "exclude", 10, 587, 1, 64, "f32"),
    ("sparse", 2, "exclude", 1, 2, 2, 16, "f64"),
    ("sparse", 0, "zero-logit", 2, 1, 1, 8, "f64"),
    ("longformer", 3, "exclude", 40, 30, 2, 32, "f32"),
    ("sparse", 8, "exclude", 17, 77, 4, 128, "f32"),
]


def attn_spans(m, n):
    return ((0, 1), (1, m + 2), (m + 2, m + n + 3))


def attn_inputs(idx, case):
    """Random (q, k, v) of shape (heads, s, d) for attention case ``idx``."""
    _name, _w, _pad, m, n, heads, d, dt = case
    s = m + n + 3
    rng = np.random.default_rng((1234, idx))
    x = rng.standard_normal((3, heads, s, d))
    return x.astype(np.float32 if dt == "f32" else np.float64)


def attn_globals(name, m, n):
    if name != "qds":
        return ()
    return tuple(p for p in (2, 7, 29) if p < n)


def band_inputs(idx, case):
    s, t, w, d = case
    rng = np.random.default_rng((99, idx))
    q = rng.standard_normal((s, d))
    k = rng.standard_normal((t, d))
    p = rng.standard_normal((s, 2 * w + 1))
    v = rng.standard_normal((t, d))
    return q, k, p, v


# Encoder configs (EncoderConfig field order: layers, embed_dim, heads,
# ff_dim, max_positions, vocab_size, pattern, window, ...).
C1 = dict(layers=2, embed_dim=32, heads=2, ff_dim=64, max_positions=177, vocab_size=1024,
          pattern="sparse", window=4)
TINY = dict(layers=2, embed_dim=16, heads=2, ff_dim=32, max_positions=64, vocab_size=40,
            window=2, qds_global_every=4)
ELECTRA_PASSAGE = dict(layers=12, embed_dim=768, heads=12, ff_dim=3072, max_positions=512,
                       vocab_size=30522, pattern="sparse", window=4)
ELECTRA_DOC = dict(ELECTRA_PASSAGE, max_positions=4099)


def tiny_sequence(seed, m, n, vocab):
    rng = np.random.default_rng(seed)
    return rng.integers(3, vocab, size=m), rng.integers(3, vocab, size=n)


# ---- backward / training fixtures -------------------------

def band_grad_inputs(idx, case):
    """Upstream gradients (grad_band (s, 2w+1), grad_out (s, d)) for band case ``idx``."""
    s, t, w, d = case
    rng = np.random.default_rng((77, idx))
    return rng.standard_normal((s, 2 * w + 1)), rng.standard_normal((s, d))


def attn_grad_out(idx, case):
    """Output gradient (heads, s, d) for attention case ``idx``."""
    _name, _w, _pad, m, n, heads, d, dt = case
    rng = np.random.default_rng((4321, idx))
    g = rng.standard_normal((heads, m + n + 3, d))
    return g.astype(np.float32 if dt == "f32" else np.float64)


def grad_projection(idx, d):
    """(d, 4) projection the large attention-gradient fixtures are stored through."""
    return np.random.default_rng((999, idx)).standard_normal((d, 4))


TRAIN_GRAD_SCORES = np.array([0.7, -1.3])

TASK = dict(vocab_words=12, query_terms=2, doc_len=6)   # T/test_training.py:28


def task_config_kw(pattern, window):
    """T/test_training.py:31-43 (vocab = 3 special + 12 words)."""
    return dict(layers=2, embed_dim=32, heads=4, ff_dim=64, max_positions=16, vocab_size=15,
                pattern=pattern, window=window)


def adamw_inputs():
    rng = np.random.default_rng(55)
    ws = {"a": rng.standard_normal((3, 4)), "b": rng.standard_normal(5), "c": np.array(0.25)}
    gs = [{n: rng.standard_normal(np.shape(a)) * (0.0 if step == 2 and n == "b" else 1.0)
           for n, a in ws.items()} for step in range(5)]
    return ws, gs


# ---- headline ranking + re-rank driver fixtures (round 2) -------------------

# 1 query x RANK_DOCS candidates at s=4099 (q10 + d4086): the C3/C5 headline pairs, ids from
# default_rng((0, 0, j)) exactly as bench.py and rerank.synthetic_queries draw them.
RANK_DOCS = 32

# Re-rank driver (R/evaluation.py:176-205 driven like R/cli.py:224-238) at ELECTRA-base dims,
# max_positions 512: (query length, #candidates, top_k).  Query 3 is too long for max_positions
# (assemble_input raises -> every pair scores -inf in the reference).
RERANK_QUERIES = [(10, 20, 100), (31, 24, 15), (4, 20, 100), (520, 5, 100)]


def rerank_workload(vocab, maxpos=512):
    """[(qid, query_ids, [(doc_id, doc_ids), ...], top_k)]: mixed doc lengths 0..700 (those above
    maxpos - m - 3 are truncated by assemble_input), one empty document and, in query 0, a
    duplicate of candidate 3 at position 7 (a score tie that the stable sort must keep in
    candidate order)."""
    out = []
    for q, (qlen, ncand, top_k) in enumerate(RERANK_QUERIES):
        rng = np.random.default_rng((7, q))
        qids = rng.integers(3, vocab, size=qlen)
        lens = rng.integers(0, 700, size=ncand)
        lens[min(2, ncand - 1)] = 0
        cands = [(f"d{q}_{j}", np.random.default_rng((7, q, j)).integers(3, vocab, size=int(n)))
                 for j, n in enumerate(lens)]
        if q == 0:
            cands[7] = ("d0_7", cands[3][1].copy())
        out.append((f"q{q}", qids, cands, top_k))
    return out
