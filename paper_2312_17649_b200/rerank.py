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
from dataclasses import dataclass

import numpy as np
import torch

from .encoder import CrossEncoder, EncoderError, PackedBatch, assemble_input


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


def write_run(path, entries) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(format_run(entries))


def read_run(path) -> list:
    with open(path, encoding="utf-8") as fh:
        return parse_run(fh)


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


def score_candidates(model: CrossEncoder, query_ids, candidate_ids, max_tokens: int = 1 << 18) -> np.ndarray:
    """fp32 scores of every (query, candidate) pair, packed varlen on the GPU; unscorable -> -inf."""
    seqs, ok = [], []
    for doc in candidate_ids:
        try:
            seqs.append(assemble_input(query_ids, doc, model.config.max_positions))
            ok.append(True)
        except EncoderError:
            ok.append(False)
    scores = np.full(len(candidate_ids), -np.inf, dtype=np.float32)
    if seqs:
        got, chunk, tok = [], [], 0
        for s in seqs:
            if chunk and tok + s.partition.seq_len > max_tokens:
                got.append(model.score_packed(PackedBatch.from_sequences(chunk)))
                chunk, tok = [], 0
            chunk.append(s)
            tok += s.partition.seq_len
        got.append(model.score_packed(PackedBatch.from_sequences(chunk)))
        vals = torch.cat(got).cpu().numpy()
        model._raise_if_nonfinite()
        scores[np.asarray(ok)] = vals
    return scores


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
    """Re-rank ``queries`` = [(qid, query_ids, [(doc_id, doc_ids), ...]), ...] over `world` ranks.

    Each rank scores a contiguous block of queries; scores are gathered with
    one all-gather; rank 0 returns the ranked run entries (others return None).
    ``score_fn(query_ids, candidate_ids) -> float32 array`` overrides the GPU
    scorer (used by the CPU multi-process tests).
    """
    if score_fn is None:
        def score_fn(qids, cands):
            return score_candidates(model, qids, cands)
    lo, hi = shard_range(len(queries), world, rank)
    local = [np.asarray(score_fn(q[1], [c[1] for c in q[2]]), np.float32) for q in queries[lo:hi]]
    flat = np.concatenate(local) if local else np.zeros(0, np.float32)
    if world > 1:
        per_q = [len(q[2]) for q in queries]
        counts = [sum(per_q[slice(*shard_range(len(queries), world, r))]) for r in range(world)]
        nccl = torch.distributed.get_backend(group) == "nccl"
        dev = (model.device if model is not None else torch.device("cuda")) if nccl else torch.device("cpu")
        allv = gather_scores(torch.from_numpy(flat).to(dev), counts, group).cpu().numpy()
    else:
        allv = flat
    if rank != 0:
        return None
    entries, off = [], 0
    for qid, _q, cands in queries:
        sc = allv[off: off + len(cands)]
        off += len(cands)
        entries += rank_entries(qid, [c[0] for c in cands], sc, top_k, tag)
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
