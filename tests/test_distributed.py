"""Multi-process (world size 2, gloo on CPU) checks of the re-rank sharding and score gather.

The GPU path uses the same code with the NCCL backend; here a deterministic
CPU scorer stands in for the encoder so the collective logic is exercised
without a device.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def fake_score(qids, cands):
    """Deterministic stand-in scorer (ties on purpose: every 7th candidate repeats a score)."""
    q = int(np.sum(qids)) % 97
    return np.array([((int(np.sum(c)) + q) % 13) / 13.0 for c in cands], np.float32)


def _worker(rank, world, port, queries, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2312_17649_b200.rerank import gather_scores, rerank_distributed

    # variable-length gather
    local = torch.arange(rank + 2, dtype=torch.float32) + 10 * rank
    allv = gather_scores(local, [2, 3])
    assert allv.tolist() == [0.0, 1.0, 10.0, 11.0, 12.0]
    entries = rerank_distributed(None, queries, top_k=5, rank=rank, world=world, score_fn=fake_score)
    if rank == 0:
        from paper_2312_17649_b200.rerank import write_run

        write_run(entries, out_path)
    else:
        assert entries is None
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_covers_everything():
    from paper_2312_17649_b200.rerank import shard_range

    for n in (0, 1, 7, 100, 1000):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_rank_entries_reference_tie_break():
    from paper_2312_17649_b200.rerank import rank_entries

    e = rank_entries("q", ["a", "b", "c", "d"], [0.5, 0.7, 0.5, -np.inf], top_k=3)
    assert [x.doc_id for x in e] == ["b", "a", "c"] and [x.rank for x in e] == [1, 2, 3]


def test_world2_gloo_matches_single_process(tmp_path):
    from paper_2312_17649_b200.rerank import read_run, rerank_distributed, synthetic_queries

    queries = synthetic_queries(5, 9, 20, vocab=1000, seed=3)
    single = rerank_distributed(None, queries, top_k=5, score_fn=fake_score)
    out = tmp_path / "run.txt"
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, queries, str(out)), nprocs=2, join=True, start_method="spawn")
    got = read_run(out)
    assert [(e.query_id, e.doc_id, e.rank) for e in got] == [(e.query_id, e.doc_id, e.rank) for e in single]
    np.testing.assert_allclose([e.score for e in got], [e.score for e in single], atol=1e-6)


def test_trec_run_roundtrip(tmp_path):
    from paper_2312_17649_b200.rerank import RunEntry, format_run, parse_run

    entries = [RunEntry("q1", "d3", 1, 0.5), RunEntry("q1", "d1", 2, -0.25, "x")]
    assert parse_run(format_run(entries).splitlines()) == entries
    with pytest.raises(ValueError):
        parse_run(["q1 Q0 d1 1 0.5"])


def _dp_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2312_17649_b200.training import AdamW, GradDict, allreduce_gradients

    # every rank: the same weights, its own gradients; after the all-reduce every rank holds the
    # mean and applies the same AdamW update
    w = {"a": torch.arange(6, dtype=torch.float64).reshape(2, 3) / 10, "b": torch.ones(4, dtype=torch.float64)}
    opt = AdamW(0.1, weight_decay=0.01, moment_dtype=torch.float64)
    for step in range(3):
        gen = torch.Generator().manual_seed(100 * step + rank)
        flat = torch.randn(10, dtype=torch.float64, generator=gen)
        g = GradDict(flat)
        g["a"], g["b"] = flat[:6].view(2, 3), flat[6:]
        allreduce_gradients(g)
        opt.step(w, g)
    torch.save({k: v.clone() for k, v in w.items()}, f"{out_path}.{rank}")
    dist.barrier()
    dist.destroy_process_group()


def test_data_parallel_gradient_average_gloo(tmp_path):
    from paper_2312_17649_b200.training import AdamW

    world, port = 2, _free_port()
    out = str(tmp_path / "w")
    mp.spawn(_dp_worker, args=(world, port, out), nprocs=world, join=True)
    got = [torch.load(f"{out}.{r}") for r in range(world)]
    # single-process reference on the mean gradient
    w = {"a": torch.arange(6, dtype=torch.float64).reshape(2, 3) / 10, "b": torch.ones(4, dtype=torch.float64)}
    opt = AdamW(0.1, weight_decay=0.01, moment_dtype=torch.float64)
    for step in range(3):
        fl = sum(torch.randn(10, dtype=torch.float64, generator=torch.Generator().manual_seed(100 * step + r))
                 for r in range(world)) / world
        opt.step(w, {"a": fl[:6].view(2, 3), "b": fl[6:]})
    for r in range(world):
        for k in w:
            assert torch.equal(got[r][k], got[0][k])
            torch.testing.assert_close(got[r][k], w[k], rtol=1e-12, atol=1e-12)
