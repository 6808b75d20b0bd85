"""CPU oracle for the sparse cross-encoder hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in vectorised numpy, the algorithm of the reference
package ``sparsecross`` 0.1.0 (arXiv 2312.17649) along the inference hot
path: band kernels, joint segment softmax, grouped pattern attention, the
dense brute-force mask, and the post-LN encoder forward.  Every function
cites the reference ``file:line`` it follows (``R/`` =
``/root/reference/pkg/src/sparsecross/``).

Status: **parity pinned**.  ``tests/test_oracle_golden.py`` checks this
module against golden vectors produced by importing the reference itself
(``tests/golden/make_golden.py``, committed with the fixtures).

Use restrictions: only ``tests/``, ``__graft_entry__.smoke``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import
this module, and only as the checker or the timed CPU baseline.  The
product package ``paper_2312_17649_b200`` never imports it; its GPU path
fails loudly when the CUDA library is missing.
"""

from __future__ import annotations

import math

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view
from scipy.special import erf

FULL = math.inf
GROUPS = ("cls", "query", "doc")
CLS_ID, SEP_ID, NUM_SPECIAL = 0, 1, 3          # R/tokenizer.py:11-14
LN_EPS = 1e-12                                 # R/encoder.py:41


class OracleError(ValueError):
    """Any condition on which the reference raises a ValueError subclass."""


def _finite(w) -> bool:
    return not (isinstance(w, float) and math.isinf(w))


# ---------------------------------------------------------------------------
# Band kernels  (R/band.py)
# ---------------------------------------------------------------------------

def band_validity(rows: int, w: int, target_len: int) -> np.ndarray:
    """R/band.py:48-52 -- slot (i, j) valid iff 0 <= i + j - w < target_len."""
    tgt = np.arange(rows)[:, None] - w + np.arange(2 * w + 1)[None, :]
    return (tgt >= 0) & (tgt < target_len)


def _padded_windows(m: np.ndarray, w: int, rows: int) -> np.ndarray:
    """View (..., rows, feat, 2w+1): window j of row i is target row i+j-w (0 if absent).

    Restates the zero padding of R/band.py:139-151 with a sliding window.
    """
    t = m.shape[-2]
    pad = np.zeros(m.shape[:-2] + (rows + 2 * w, m.shape[-1]), dtype=m.dtype)
    take = min(t, rows + w)
    pad[..., w:w + take, :] = m[..., :take, :]
    return sliding_window_view(pad, 2 * w + 1, axis=-2)


def band_scores(q: np.ndarray, k: np.ndarray, w: int) -> np.ndarray:
    """R/band.py:154-194 (⊡_w): out[..., i, j] = q_i . k_{i+j-w}; 0 where out of range."""
    if q.shape[-1] != k.shape[-1]:
        raise OracleError("feature dims differ")
    win = _padded_windows(k, w, q.shape[-2])          # (..., s, d, 2w+1)
    return np.einsum("...sd,...sdj->...sj", q, win)


def band_apply(p: np.ndarray, v: np.ndarray, w: int) -> np.ndarray:
    """R/band.py:197-236 (⊙_w): out_i = sum_j p_ij v_{i+j-w}; invalid slots never contribute."""
    if p.shape[-1] != 2 * w + 1:
        raise OracleError("band width inconsistent with window")
    ok = band_validity(p.shape[-2], w, v.shape[-2])
    p = np.where(ok, p, 0.0).astype(np.result_type(p, v), copy=False)
    win = _padded_windows(v, w, p.shape[-2])          # (..., s, d, 2w+1)
    return np.einsum("...sj,...sdj->...sd", p, win)


def dense_band_oracle(q, k, w):
    """R/band.py:369-388 -- full q k^T masked where |t - i| > w (masked array)."""
    full = q @ k.T
    off = np.arange(k.shape[0])[None, :] - np.arange(q.shape[0])[:, None]
    return np.ma.MaskedArray(full, mask=np.abs(off) > w)


# ---------------------------------------------------------------------------
# Patterns  (R/attention.py:55-157)
# ---------------------------------------------------------------------------

def make_pattern(name: str, window, global_positions=()) -> dict:
    """R/attention.py:92-157 -- pattern as {'name', 'targets': {src: ((tgt, w), ...)}, 'globals'}."""
    every = (("cls", FULL), ("query", FULL), ("doc", FULL))
    local = (("cls", FULL), ("query", FULL), ("doc", window))
    if name == "full":
        t = {g: every for g in GROUPS}
    elif name in ("longformer", "qds"):
        t = {"cls": every, "query": every, "doc": local}
    elif name == "sparse":
        t = {"cls": every, "query": (("query", FULL),), "doc": local}
    else:
        raise OracleError(f"unknown pattern {name!r}")
    g = tuple(int(p) for p in global_positions) if name == "qds" else ()
    return {"name": name, "targets": t, "globals": g}


def qds_global_positions(doc_tokens: int, every: int = 30) -> tuple:
    """R/encoder.py:180-184."""
    return tuple(range(every - 1, doc_tokens, every))


# ---------------------------------------------------------------------------
# Joint segment softmax and segment attention  (R/attention.py:228-345)
# ---------------------------------------------------------------------------

def masked_segment_softmax(values, valids, scale, padding="exclude"):
    """R/attention.py:228-257 -- one softmax over the union of all segments' valid slots."""
    fill = 0.0 if padding == "zero-logit" else -np.inf
    ys = [v / scale if ok is None else np.where(ok, v / scale, fill) for v, ok in zip(values, valids)]
    m = np.max(np.stack([y.max(axis=-1) for y in ys]), axis=0)
    if np.isneginf(m).any():
        raise OracleError("a row has zero valid entries across all segments")
    es = [np.exp(y - m[..., None]) for y in ys]
    z = sum(e.sum(axis=-1, keepdims=True) for e in es)
    return [e / z for e in es]


def attend_segments(q, segments, scale, padding="exclude"):
    """R/attention.py:290-345 -- segments = [(k, v, w, extra_invalid)], output summed in tuple order."""
    if not segments:
        raise OracleError("segment tuple must be nonempty")
    s = q.shape[-2]
    vals, oks = [], []
    for k, v, w, extra in segments:
        if not _finite(w):
            vals.append(q @ np.swapaxes(k, -1, -2))
            oks.append(None)
            continue
        sc = band_scores(q, k, int(w))
        ok = band_validity(s, int(w), k.shape[-2])
        if extra is not None:
            if padding == "zero-logit":
                sc = np.where(extra, -np.inf, sc)
            else:
                ok = ok & ~extra
        vals.append(sc)
        oks.append(ok)
    probs = masked_segment_softmax(vals, oks, scale, padding)
    out = None
    for p, (k, v, w, _e) in zip(probs, segments):
        part = p @ v if not _finite(w) else band_apply(p, v, int(w))
        out = part if out is None else out + part
    return out


def _qds_exclusions(doc_len, w, globals_):
    """R/attention.py:403-413 -- doc-doc band slots that hit a global token."""
    if not globals_:
        return None
    tgt = np.arange(doc_len)[:, None] - w + np.arange(2 * w + 1)[None, :]
    hit = np.zeros(doc_len + 1, dtype=bool)
    hit[list(globals_)] = True
    return hit[np.clip(tgt, 0, doc_len)] & band_validity(doc_len, w, doc_len)


def group_attention(qkv: dict, source: str, pattern: dict, scale: float, padding="exclude"):
    """R/attention.py:416-473 -- attention of one source group (with the QDS global-token rules)."""
    q = qkv[source][0]
    gl = pattern["globals"]
    segs = []
    for tgt, w in pattern["targets"][source]:
        k, v = qkv[tgt][1], qkv[tgt][2]
        extra = None
        if gl and source == "doc" and tgt == "doc" and _finite(w):
            extra = _qds_exclusions(qkv["doc"][1].shape[-2], int(w), gl)
        segs.append((k, v, w, extra))
    if gl and source == "doc":
        idx = np.asarray(gl)
        segs.append((qkv["doc"][1][..., idx, :], qkv["doc"][2][..., idx, :], FULL, None))
    out = attend_segments(q, segs, scale, padding)
    if gl and source == "doc":
        idx = np.asarray(gl)
        gsegs = [(qkv[g][1], qkv[g][2], FULL, None) for g in GROUPS]
        out = np.array(out)
        out[..., idx, :] = attend_segments(q[..., idx, :], gsegs, scale, padding)
    return out


def apply_pattern(spans, qkv, pattern, scale=None, padding="exclude"):
    """R/attention.py:510-537 -- (O_cls, O_query, O_doc)."""
    if scale is None:
        scale = math.sqrt(qkv["cls"][0].shape[-1])
    return tuple(group_attention(qkv, g, pattern, scale, padding) for g in GROUPS)


def split_groups(spans, q, k, v) -> dict:
    """R/encoder.py:299-303 -- group views of (..., s, d) arrays; spans = ((0,1),(1,a),(a,s))."""
    return {g: (q[..., lo:hi, :], k[..., lo:hi, :], v[..., lo:hi, :]) for g, (lo, hi) in zip(GROUPS, spans)}


# ---------------------------------------------------------------------------
# Dense brute-force route  (R/reference.py)
# ---------------------------------------------------------------------------

def token_groups(spans):
    """R/reference.py:22-27 (_locate), vectorised: per-position (group id, group-relative index)."""
    s = spans[2][1]
    gid = np.empty(s, dtype=np.int64)
    rel = np.empty(s, dtype=np.int64)
    for g, (lo, hi) in enumerate(spans):
        gid[lo:hi] = g
        rel[lo:hi] = np.arange(hi - lo)
    return gid, rel


def pattern_mask(pattern: dict, spans) -> np.ndarray:
    """R/reference.py:30-57 -- (s, s) bool mask, position i may attend to t."""
    gid, rel = token_groups(spans)
    s = gid.shape[0]
    mask = np.zeros((s, s), dtype=bool)
    dr = np.abs(rel[None, :] - rel[:, None])
    for si, src in enumerate(GROUPS):
        rows = gid == si
        for tgt, w in pattern["targets"].get(src, ()):
            ti = GROUPS.index(tgt)
            ok = (gid[None, :] == ti) & (True if not _finite(w) else dr <= w)
            mask |= rows[:, None] & ok
    gl = pattern["globals"]
    if gl:
        isg = np.zeros(s, dtype=bool)
        d = gid == 2
        isg[d] = np.isin(rel[d], gl)
        mask[isg & d, :] = True
        mask |= d[:, None] & (isg & d)[None, :]
    return mask


def masked_attention(q, k, v, mask, scale):
    """R/reference.py:60-70 -- dense softmax with a {0, -inf} additive mask."""
    if (~mask.any(axis=1)).any():
        raise OracleError("mask leaves a row with no attendable position")
    y = np.where(mask, (q @ k.T) / scale, -np.inf)
    e = np.exp(y - y.max(axis=1, keepdims=True))
    return (e / e.sum(axis=1, keepdims=True)) @ v


# ---------------------------------------------------------------------------
# Inputs, weights, encoder  (R/encoder.py, R/bench.py)
# ---------------------------------------------------------------------------

def assemble_input(query_ids, doc_ids, max_positions=None):
    """R/encoder.py:154-177 -- ([CLS] q [SEP] d [SEP], spans); doc tail truncated, query never."""
    q, d = list(query_ids), list(doc_ids)
    if not q:
        raise OracleError("query must contain at least one token")
    if max_positions is not None:
        if len(q) + 3 > max_positions:
            raise OracleError("query cannot fit")
        d = d[:max_positions - len(q) - 3]
    ids = np.asarray([CLS_ID] + q + [SEP_ID] + d + [SEP_ID], dtype=np.int64)
    m, n = len(q), len(d)
    return ids, ((0, 1), (1, m + 2), (m + 2, m + n + 3))


def gen_random_ids(seed, query_len, doc_len, batch, vocab):
    """R/bench.py:128-140 -- seeded uniform ids; rng keyed on (seed, doc_len)."""
    rng = np.random.default_rng((seed, doc_len))
    rows = []
    for _ in range(batch):
        qy = rng.integers(NUM_SPECIAL, vocab, size=query_len)
        dc = rng.integers(NUM_SPECIAL, vocab, size=doc_len)
        rows.append(np.concatenate([[CLS_ID], qy, [SEP_ID], dc, [SEP_ID]]))
    spans = ((0, 1), (1, query_len + 2), (query_len + 2, query_len + doc_len + 3))
    return np.stack(rows).astype(np.int64), spans


def init_weights(cfg: dict, seed: int = 0, dtype=np.float32) -> dict:
    """R/encoder.py:217-247 -- U(+-1/sqrt(fan_in)) in draw order tok, pos, per layer q,k,v,o,w1,w2, head."""
    rng = np.random.default_rng(seed)
    h, ff = cfg["embed_dim"], cfg["ff_dim"]

    def u(shape, fan_in):
        b = 1.0 / math.sqrt(fan_in)
        return rng.uniform(-b, b, size=shape).astype(dtype)

    wt = {"tok_emb": u((cfg["vocab_size"], h), 1), "pos_emb": u((cfg["max_positions"], h), 1)}
    for i in range(cfg["layers"]):
        p = f"L{i}."
        for nm in ("q", "k", "v", "o"):
            wt[p + "w" + nm] = u((h, h), h)
            wt[p + "b" + nm] = np.zeros(h, dtype)
        wt[p + "ln1_g"], wt[p + "ln1_b"] = np.ones(h, dtype), np.zeros(h, dtype)
        wt[p + "w1"], wt[p + "b1"] = u((h, ff), h), np.zeros(ff, dtype)
        wt[p + "w2"], wt[p + "b2"] = u((ff, h), ff), np.zeros(h, dtype)
        wt[p + "ln2_g"], wt[p + "ln2_b"] = np.ones(h, dtype), np.zeros(h, dtype)
    wt["head_w"] = u((h,), h)
    wt["head_b"] = np.zeros((), dtype)
    return wt


def gelu(x):
    """R/encoder.py:258-259 -- exact erf GELU."""
    return 0.5 * x * (1.0 + erf(x / np.sqrt(2.0).astype(x.dtype)))


def layer_norm(x, g, b):
    """R/encoder.py:267-273 -- biased variance, eps 1e-12."""
    xc = x - x.mean(axis=-1, keepdims=True)
    var = (xc * xc).mean(axis=-1, keepdims=True)
    return g * (xc * (1.0 / np.sqrt(var + LN_EPS))) + b


def resolve_pattern(cfg: dict, spans) -> dict:
    """R/encoder.py:187-193."""
    gl = ()
    if cfg["pattern"] == "qds":
        gl = qds_global_positions(spans[2][1] - spans[2][0] - 1, cfg.get("qds_global_every", 30))
    return make_pattern(cfg["pattern"], cfg["window"], gl)


def layer_forward(x, spans, pattern, wt, i, cfg):
    """R/encoder.py:306-371 -- QKV -> grouped attention -> Wo -> LN -> erf-GELU FFN -> LN (post-LN)."""
    p = f"L{i}."
    b, s, h = x.shape
    H = cfg["heads"]
    d = h // H

    def heads(t):
        return t.reshape(b, s, H, d).transpose(0, 2, 1, 3)

    q = heads(x @ wt[p + "wq"] + wt[p + "bq"])
    k = heads(x @ wt[p + "wk"] + wt[p + "bk"])
    v = heads(x @ wt[p + "wv"] + wt[p + "bv"])
    qkv = split_groups(spans, q, k, v)
    outs = [group_attention(qkv, g, pattern, math.sqrt(d), cfg.get("padding", "exclude")) for g in GROUPS]
    o = np.concatenate(outs, axis=-2).transpose(0, 2, 1, 3).reshape(b, s, h)
    x1 = layer_norm(x + (o @ wt[p + "wo"] + wt[p + "bo"]), wt[p + "ln1_g"], wt[p + "ln1_b"])
    f = gelu(x1 @ wt[p + "w1"] + wt[p + "b1"]) @ wt[p + "w2"] + wt[p + "b2"]
    out = layer_norm(x1 + f, wt[p + "ln2_g"], wt[p + "ln2_b"])
    if not np.isfinite(out).all():
        raise FloatingPointError(f"non-finite activations in layer {i}")
    return out


def embed(ids, wt, dtype):
    """R/encoder.py:483 -- tok_emb[ids] + pos_emb[:s] (no embedding LN, no token types)."""
    return (wt["tok_emb"][ids] + wt["pos_emb"][: ids.shape[1]]).astype(dtype, copy=False)


def encoder_forward(ids, spans, cfg, wt, dtype=np.float32):
    """R/encoder.py:475-500 -- final-layer (B, s, h) activations for equal-length sequences."""
    ids = np.atleast_2d(np.asarray(ids, dtype=np.int64))
    pattern = resolve_pattern(cfg, spans)
    x = embed(ids, wt, dtype)
    for i in range(cfg["layers"]):
        x = layer_forward(x, spans, pattern, wt, i, cfg)
    return x


def score(ids, spans, cfg, wt, dtype=np.float32):
    """R/encoder.py:502-509 -- x[:, 0] . head_w + head_b."""
    x = encoder_forward(ids, spans, cfg, wt, dtype)
    return x[:, 0, :] @ wt["head_w"] + wt["head_b"]


def rank_order(scores) -> list:
    """R/evaluation.py:194-201 -- stable sort by (-score, candidate position)."""
    return sorted(range(len(scores)), key=lambda j: (-float(scores[j]), j))


def flop_count(pattern, group_lens, h, layers, ff_dim):
    """R/bench.py:167-219 -- multiply-add model (padded band slots counted)."""
    lens = dict(zip(GROUPS, group_lens))
    s = sum(group_lens)
    att = 0
    for src in GROUPS:
        for tgt, w in pattern["targets"][src]:
            att += lens[src] * (lens[tgt] if not _finite(w) else 2 * int(w) + 1) * h
    if pattern["globals"]:
        g = len(pattern["globals"])
        att += lens["doc"] * g * h + g * s * h
    return {"attention": 2 * att * layers, "projections": 4 * s * h * h * layers,
            "feed_forward": 2 * s * h * ff_dim * layers}


# ---------------------------------------------------------------------------
# Adjoints  (R/band.py:239-274, R/attention.py:260-269, :348-378, :476-507)
# -- the checker for the fine-tuning path
# ---------------------------------------------------------------------------

def _band_scatter(g: np.ndarray, x: np.ndarray, w: int, t: int) -> np.ndarray:
    """out[..., r, :] = sum over valid slots (i, j) with i+j-w == r of g[..., i, j] x[..., i, :]."""
    s = g.shape[-2]
    out = np.zeros(g.shape[:-2] + (t, x.shape[-1]), dtype=np.result_type(g, x))
    for j in range(2 * w + 1):
        lo, hi = max(0, w - j), min(s, t + w - j)      # rows whose slot j lands in [0, t)
        if lo < hi:
            out[..., lo + j - w:hi + j - w, :] += g[..., lo:hi, j:j + 1] * x[..., lo:hi, :]
    return out


def band_scores_backward(grad_band, q, k, w):
    """R/band.py:239-253 -- (grad_q, grad_k) of band_scores; invalid slots never read."""
    return band_apply(grad_band, k, w), _band_scatter(
        np.where(band_validity(q.shape[-2], w, k.shape[-2]), grad_band, 0.0), q, w, k.shape[-2])


def band_apply_backward(grad_out, p, v, w):
    """R/band.py:256-274 -- (grad_p, grad_v) of band_apply; grad_p is 0 at invalid slots."""
    ok = band_validity(p.shape[-2], w, v.shape[-2])
    return band_scores(grad_out, v, w), _band_scatter(np.where(ok, p, 0.0), grad_out, w, v.shape[-2])


def attend_segments_backward(q, segments, scale, grad_out, padding="exclude"):
    """R/attention.py:348-378 (+ the softmax adjoint :260-269), recomputing the probabilities.

    Returns (grad_q, [(grad_k, grad_v) per segment]).  Zero-logit padding
    slots carry probability but a constant logit, so only valid slots reach q/k.
    """
    s = q.shape[-2]
    vals, oks = [], []
    for k, v, w, extra in segments:
        if not _finite(w):
            vals.append(q @ np.swapaxes(k, -1, -2))
            oks.append(None)
            continue
        sc = band_scores(q, k, int(w))
        ok = band_validity(s, int(w), k.shape[-2])
        if extra is not None:
            if padding == "zero-logit":
                sc = np.where(extra, -np.inf, sc)
            else:
                ok = ok & ~extra
        vals.append(sc)
        oks.append(ok)
    probs = masked_segment_softmax(vals, oks, scale, padding)
    gps, gvs = [], []
    for p, (k, v, w, _e) in zip(probs, segments):
        if not _finite(w):
            gps.append(grad_out @ np.swapaxes(v, -1, -2))
            gvs.append(np.swapaxes(p, -1, -2) @ grad_out)
        else:
            gp, gv = band_apply_backward(grad_out, p, v, int(w))
            gps.append(gp)
            gvs.append(gv)
    dot = sum(np.sum(p * gp, axis=-1, keepdims=True) for p, gp in zip(probs, gps))
    gq = np.zeros_like(q)
    kv = []
    for p, gp, gv, (k, v, w, _e) in zip(probs, gps, gvs, segments):
        ga = p * (gp - dot) / scale
        if not _finite(w):
            gq = gq + ga @ k
            gk = np.swapaxes(ga, -1, -2) @ q
        else:
            dq_part, gk = band_scores_backward(ga, q, k, int(w))
            gq = gq + dq_part
        kv.append((gk, gv))
    return gq, kv


def _group_segments(qkv, source, pattern):
    gl = pattern["globals"]
    segs, where = [], []
    for tgt, w in pattern["targets"][source]:
        extra = None
        if gl and source == "doc" and tgt == "doc" and _finite(w):
            extra = _qds_exclusions(qkv["doc"][1].shape[-2], int(w), gl)
        segs.append((qkv[tgt][1], qkv[tgt][2], w, extra))
        where.append((tgt, None))
    if gl and source == "doc":
        idx = np.asarray(gl)
        segs.append((qkv["doc"][1][..., idx, :], qkv["doc"][2][..., idx, :], FULL, None))
        where.append(("doc", idx))
    return segs, where


def apply_pattern_backward(spans, qkv, pattern, grad_out, scale=None, padding="exclude"):
    """R/attention.py:476-507 assembled like R/encoder.py:421-435: (dq, dk, dv) over the whole
    sequence for grad_out (..., s, d).  QDS global doc rows: windowed result discarded, dense
    recompute over every group."""
    if scale is None:
        scale = math.sqrt(qkv["cls"][0].shape[-1])
    span = dict(zip(GROUPS, spans))
    dq = np.zeros_like(grad_out)
    dk = np.zeros_like(grad_out)
    dv = np.zeros_like(grad_out)
    gl = pattern["globals"]
    for src in GROUPS:
        lo, hi = span[src]
        q = qkv[src][0]
        go = grad_out[..., lo:hi, :]
        segs, where = _group_segments(qkv, src, pattern)
        if gl and src == "doc":
            idx = np.asarray(gl)
            go_local = np.array(go)
            go_local[..., idx, :] = 0.0
            gq, kv = attend_segments_backward(q, segs, scale, go_local, padding)
            gsegs = [(qkv[g][1], qkv[g][2], FULL, None) for g in GROUPS]
            gq_g, kv_g = attend_segments_backward(q[..., idx, :], gsegs, scale, go[..., idx, :], padding)
            gq[..., idx, :] += gq_g
            kv += kv_g
            where += [(g, None) for g in GROUPS]
        else:
            gq, kv = attend_segments_backward(q, segs, scale, go, padding)
        dq[..., lo:hi, :] += gq
        for (tgt, idx), (gk, gv) in zip(where, kv):
            t0, t1 = span[tgt]
            if idx is None:
                dk[..., t0:t1, :] += gk
                dv[..., t0:t1, :] += gv
            else:
                dk[..., t0 + idx, :] += gk
                dv[..., t0 + idx, :] += gv
    return dq, dk, dv
