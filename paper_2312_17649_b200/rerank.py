"""Batched, multi-GPU re-ranking driver and TREC run IO.

Replaces the reference's one-pair-per-forward loop (R/cli.py:206-247 ->
R/evaluation.py:176-205 -> CrossEncoder.score_pair): every candidate of a
query is packed into varlen batches and scored on the GPU; queries are
sharded contiguously over ranks (one process per GPU) and the fp32 scores are
gathered with one collective (NCCL over NVLink on B200, gloo on CPU tests).
Ranking uses the reference order: stable sort by (-score, candidate
position); a candidate that cannot be scored gets -inf (R/evaluation.py:194-201).
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from .encoder import CrossEncoder, EncoderError, PackedBatch
from .tokenizer import CLS_ID, SEP_ID


class EvaluationError(ValueError):
    pass


@dataclass(frozen=True)
class RunEntry:
    """One TREC run line (R/evaluation.py:23-29)."""

    query_id: str
    doc_id: str
    rank: int
    score: float
    tag: str = "sparsecross"


def format_run(entries) -> str:
    """``qid Q0 docid rank score tag`` lines (R/evaluation.py:52-55)."""
    return "".join(f"{e.query_id} Q0 {e.doc_id} {e.rank} {e.score:.6f} {e.tag}\n" for e in entries)


def parse_run(lines) -> list:
    """Inverse of format_run (R/evaluation.py:38-49)."""
    out = []
    for n, line in enumerate(lines, 1):
        line = line.strip()
        if not line:
            continue
        parts = line.split()
        if len(parts) != 6:
            raise EvaluationError(f"run line {n}: expected 6 fields, got {len(parts)}")
        qid, _q0, did, rank, score, tag = parts
        out.append(RunEntry(qid, did, int(rank), float(score), tag))
    return out


def write_run(entries, path) -> None:
    """R/evaluation.py:63-65 (same argument order)."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(format_run(entries))


def read_run(path) -> list:
    with open(path, encoding="utf-8") as fh:
        return parse_run(fh)


def parse_qrels(lines) -> dict:
    """TREC qrels ``qid iter docid rel`` -> {qid: {docid: rel}} (R/evaluation.py:68-82)."""
    qrels: dict = {}
    for n, line in enumerate(lines, 1):
        line = line.strip()
        if not line:
            continue
        parts = line.split()
        if len(parts) != 4:
            raise EvaluationError(f"qrels line {n}: expected 4 fields, got {len(parts)}")
        qid, _iter, did, rel = parts
        rel = int(rel)
        if rel < 0:
            raise EvaluationError(f"qrels line {n}: negative relevance")
        qrels.setdefault(qid, {})[did] = rel
    return qrels


def read_qrels(path) -> dict:
    with open(path, encoding="utf-8") as fh:
        return parse_qrels(fh)


def _dcg(gains) -> float:
    """sum (2^g - 1) / log2(rank + 1) (R/evaluation.py:94-95)."""
    return sum((2.0 ** g - 1.0) / math.log2(r + 1) for r, g in enumerate(gains, 1))


def ndcg_at_k(run, qrels, k: int = 10):
    """(per-query nDCG@k, mean over the run's queries) (R/evaluation.py:98-123): documents in rank
    order, the ideal from all judged documents; queries missing from qrels score 0 (with a warning)."""
    if k < 1:
        raise EvaluationError("k must be >= 1")
    by_query: dict = {}
    for e in run:
        by_query.setdefault(e.query_id, []).append(e)
    per_query = {}
    for qid, entries in by_query.items():
        entries = sorted(entries, key=lambda e: e.rank)
        judged = qrels.get(qid)
        if judged is None:
            warnings.warn(f"query {qid} missing from qrels; scoring 0", stacklevel=2)
            per_query[qid] = 0.0
            continue
        gains = [judged.get(e.doc_id, 0) for e in entries[:k]]
        idcg = _dcg(sorted(judged.values(), reverse=True)[:k])
        per_query[qid] = _dcg(gains) / idcg if idcg > 0 else 0.0
    mean = sum(per_query.values()) / len(per_query) if per_query else 0.0
    return per_query, mean


def rank_entries(query_id: str, doc_ids, scores, top_k: int = 100, tag: str = "sparsecross") -> list:
    """Stable (-score, position) order, top_k cut, 1-based ranks (R/evaluation.py:194-205)."""
    order = sorted(range(len(scores)), key=lambda j: (-float(scores[j]), j))
    return [RunEntry(query_id, doc_ids[j], r, float(scores[j]), tag) for r, j in enumerate(order[:top_k], 1)]


def rerank(scorer, query, candidates, top_k: int = 100, query_id: str = "q", tag: str = "sparsecross"):
    """Reference-signature re-rank with a per-pair scorer (R/evaluation.py:176-205)."""
    candidates = list(candidates)
    if not candidates:
        raise EvaluationError("candidate list must be nonempty")
    scores = []
    for _doc_id, doc in candidates:
        try:
            scores.append(float(scorer(query, doc)))
        except Exception:
            scores.append(-math.inf)
    return rank_entries(query_id, [c[0] for c in candidates], scores, top_k, tag)


def pack_pairs(query_ids, candidate_ids, max_positions: int | None = None) -> PackedBatch:
    """Vectorised ``assemble_input`` for one query and many documents (R/encoder.py:154-177):
    [CLS] q [SEP] d [SEP] per pair, the doc tail truncated to max_positions - m - 3, the
    query never truncated; returns the packed varlen batch."""
    q = np.asarray(query_ids, dtype=np.int32).reshape(-1)
    m = int(q.shape[0])
    if m < 1:
        raise EncoderError("query must contain at least one token")
    if max_positions is not None and m + 3 > max_positions:
        raise EncoderError(f"query of {m} tokens cannot fit in {max_positions} positions")
    keep = None if max_positions is None else max_positions - m - 3
    docs = [np.asarray(d, dtype=np.int32).reshape(-1)[:keep] for d in candidate_ids]
    if not docs:
        raise EncoderError("empty batch")
    seq = np.array([m + 3 + d.shape[0] for d in docs], dtype=np.int64)
    off = np.zeros(len(docs) + 1, dtype=np.int64)
    np.cumsum(seq, out=off[1:])
    ids = np.empty(int(off[-1]), dtype=np.int32)
    for o, d in zip(off[:-1], docs):
        ids[o] = CLS_ID
        ids[o + 1: o + 1 + m] = q
        ids[o + 1 + m] = SEP_ID
        ids[o + 2 + m: o + 2 + m + d.shape[0]] = d
        ids[o + 2 + m + d.shape[0]] = SEP_ID
    return PackedBatch(ids, seq, np.full(len(docs), m + 1, dtype=np.int64))


def _launch_candidates(model: CrossEncoder, query_ids, candidate_ids, max_tokens: int):
    """Launch the packed chunks of one query's candidates back to back (no host sync: the next
    chunk is packed on the host while the GPU runs).  Returns (device scores, [(candidate indices, bad)]),
    ``bad`` being each chunk's per-layer non-finite counts (encode_packed's fused check)."""
    maxpos, vocab = model.config.max_positions, model.config.vocab_size
    q = np.asarray(query_ids).reshape(-1)
    m = len(q)
    ninf = torch.full((len(candidate_ids),), -math.inf, dtype=torch.float32, device=model.device)
    if m < 1 or m + 3 > maxpos or q.min() < 0 or q.max() >= vocab:
        return ninf, []  # assemble_input / _check_ids raise for every pair: the reference scores -inf
    keep = maxpos - m - 3

    def in_vocab(d):  # _check_ids after assemble_input's truncation (R/encoder.py:154-177, :475-487)
        d = np.asarray(d).reshape(-1)[:keep]
        return d.size == 0 or (d.min() >= 0 and d.max() < vocab)

    ok = [j for j, d in enumerate(candidate_ids) if in_vocab(d)]
    if len(ok) < len(candidate_ids):  # score the rest; their slots stay -inf
        if not ok:
            return ninf, []
        vals, chunks = _launch_candidates(model, query_ids, [candidate_ids[j] for j in ok], max_tokens)
        idx = torch.tensor(ok, dtype=torch.int64, device=model.device)
        ninf.index_copy_(0, idx, vals)
        return ninf, [([ok[j] for j in js], bad) for js, bad in chunks]
    got, chunks, lo = [], [], 0
    lens = [min(len(d) + m + 3, maxpos) for d in candidate_ids]
    while lo < len(candidate_ids):
        hi, tok = lo, 0
        while hi < len(candidate_ids) and (hi == lo or tok + lens[hi] <= max_tokens):
            tok += lens[hi]
            hi += 1
        got.append(model.score_packed(pack_pairs(query_ids, candidate_ids[lo:hi], maxpos)))
        chunks.append((list(range(lo, hi)), model._last_bad))
        lo = hi
    return torch.cat(got), chunks


def _rescore_nonfinite(model: CrossEncoder, pending) -> None:
    """The reference's per-pair error rule (R/evaluation.py:194-197 over R/encoder.py:356-357): a
    pair whose activations turn non-finite raises in ``score_pair`` and scores -inf.  ``pending`` =
    [(vals, query_ids, candidate_ids, chunks)]; one host sync reads every chunk's flag, and only
    the pairs of a flagged chunk are scored again one by one (in place in ``vals``)."""
    flagged = [(v, q, c, js, bad) for v, q, c, chunks in pending for js, bad in chunks if bad is not None]
    if not flagged:
        return
    counts = torch.stack([bad.sum() for *_, bad in flagged]).cpu().numpy()
    maxpos = model.config.max_positions
    for (vals, q, cands, js, _bad), n in zip(flagged, counts):
        if n == 0:
            continue
        for j in js:
            sc = model.score_packed(pack_pairs(q, [cands[j]], maxpos))
            ok = int(model._last_bad.sum()) == 0 and bool(torch.isfinite(sc).all())
            vals[j] = sc[0] if ok else -math.inf


def score_candidates(model: CrossEncoder, query_ids, candidate_ids, max_tokens: int = 1 << 18,
                     as_tensor: bool = False):
    """fp32 scores of every (query, candidate) pair, packed varlen on the GPU; a pair the reference
    could not score (query too long, non-finite activations) gets -inf, as R/evaluation.py:194-197.
    With ``as_tensor`` the device tensor is returned (no D2H copy of the scores)."""
    vals, chunks = _launch_candidates(model, query_ids, candidate_ids, max_tokens)
    _rescore_nonfinite(model, [(vals, query_ids, candidate_ids, chunks)])
    return vals if as_tensor else vals.cpu().numpy()


def shard_range(n: int, world: int, rank: int) -> tuple:
    """Contiguous block [lo, hi) of n items owned by `rank` (queries are never split)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_scores(local: torch.Tensor, counts, group=None) -> torch.Tensor:
    """All-gather variable-length fp32 score vectors (one collective; pad to the max count)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    mx = max(counts)
    buf = torch.full((mx,), float("nan"), dtype=torch.float32, device=local.device)
    buf[: local.numel()] = local
    out = torch.empty((world * mx,), dtype=torch.float32, device=local.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    return torch.cat([out[r * mx: r * mx + c] for r, c in enumerate(counts)])


def rerank_distributed(model: CrossEncoder | None, queries, top_k: int = 100, tag: str = "sparsecross",
                       rank: int = 0, world: int = 1, group=None, score_fn=None) -> list | None:
    """Re-rank ``queries`` = [(qid, query_ids, [(doc_id, doc_ids), ...][, top_k]), ...] over `world`
    ranks (a 4th element overrides ``top_k`` for that query).

    Each rank scores a contiguous block of queries; scores are gathered with
    one all-gather; rank 0 returns the ranked run entries (others return None).
    ``score_fn(query_ids, candidate_ids) -> float32 array`` overrides the GPU
    scorer (used by the CPU multi-process tests).
    """
    lo, hi = shard_range(len(queries), world, rank)
    if score_fn is None:
        # GPU path: every query's chunks are launched back to back (host packing of the
        # next chunk overlaps the GPU); scores stay on the device until the gather
        pending = []
        for q in queries[lo:hi]:
            cands = [c[1] for c in q[2]]
            pending.append((*_launch_candidates(model, q[1], cands, 1 << 18), q[1], cands))
        _rescore_nonfinite(model, [(v, qi, c, ch) for v, ch, qi, c in pending])
        parts = [p[0] for p in pending]
        flat_t = torch.cat(parts) if parts else torch.zeros(0, dtype=torch.float32, device=model.device)
    else:
        local = [np.asarray(score_fn(q[1], [c[1] for c in q[2]]), np.float32) for q in queries[lo:hi]]
        flat_t = torch.from_numpy(np.concatenate(local) if local else np.zeros(0, np.float32))
    if world > 1:
        per_q = [len(q[2]) for q in queries]
        counts = [sum(per_q[slice(*shard_range(len(queries), world, r))]) for r in range(world)]
        nccl = torch.distributed.get_backend(group) == "nccl"
        dev = (model.device if model is not None else torch.device("cuda")) if nccl else torch.device("cpu")
        allv = gather_scores(flat_t.to(dev), counts, group).cpu().numpy()
    else:
        allv = flat_t.cpu().numpy()
    if rank != 0:
        return None
    entries, off = [], 0
    for qid, _q, cands, *k in queries:
        sc = allv[off: off + len(cands)]
        off += len(cands)
        entries += rank_entries(qid, [c[0] for c in cands], sc, k[0] if k else top_k, tag)
    return entries


def synthetic_queries(n_queries: int, docs_per_query: int, doc_len: int, vocab: int, seed: int = 0,
                      query_len: int = 10, qid_offset: int = 0):
    """TREC-DL-style synthetic workload (C5): pair (q, i) ids from default_rng((seed, q, i))."""
    out = []
    for q in range(qid_offset, qid_offset + n_queries):
        qids = np.random.default_rng((seed, q)).integers(3, vocab, size=query_len)
        cands = [(f"d{q}_{i}", np.random.default_rng((seed, q, i)).integers(3, vocab, size=doc_len))
                 for i in range(docs_per_query)]
        out.append((f"q{q}", qids, cands))
    return out
