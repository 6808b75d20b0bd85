"""GPU parity of the batched re-rank driver against the reference's own run.

``tests/golden/rerank.npz`` holds the TREC run the reference produces with
``rerank(model.score_pair, ...)`` per query (R/evaluation.py:176-205, driven like
R/cli.py:224-238) at ELECTRA-base dims, f32, over ``cases.rerank_workload``:
queries of 4-31 tokens plus one too long for max_positions (every pair -inf),
documents of 0-700 tokens (those past max_positions truncated), an empty
document and a duplicated candidate (a tie kept in candidate order), and a
per-query top_k cut.
"""

import math
import os
import socket

import numpy as np
import pytest
import torch

import cases

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def P():
    import paper_2312_17649_b200 as pkg

    return pkg


@pytest.fixture(scope="module")
def gold():
    g = np.load(os.path.join(GOLD, "rerank.npz"))
    from paper_2312_17649_b200.rerank import parse_run

    return parse_run(str(g["run"]).splitlines()), g["scores"]


@pytest.fixture(scope="module")
def model(P):
    return P.CrossEncoder(P.EncoderConfig(**cases.ELECTRA_PASSAGE, precision="f32"), seed=0)


def workload(vocab=30522):
    return [(qid, q, cands, k) for qid, q, cands, k in cases.rerank_workload(vocab)]


def assert_same_run(got, ref, atol=1e-4):
    assert [(e.query_id, e.doc_id, e.rank, e.tag) for e in got] == \
        [(e.query_id, e.doc_id, e.rank, e.tag) for e in ref]
    for a, b in zip(got, ref):
        if math.isinf(b.score):
            assert a.score == b.score
        else:
            assert abs(a.score - b.score) < atol, (a, b)


def test_score_candidates_match_reference_scores(P, gold, model):
    from paper_2312_17649_b200.rerank import score_candidates

    _run, ref = gold
    got = np.concatenate([score_candidates(model, q, [c[1] for c in cands]) for _qid, q, cands, _k in workload()])
    assert got.shape == ref.shape
    assert np.array_equal(np.isinf(got), np.isinf(ref))
    fin = np.isfinite(ref)
    err = np.abs(got[fin] - ref[fin]).max()
    print(f"re-rank fp32 max |dscore| = {err:.3e} over {fin.sum()} pairs")
    assert err < 1e-4


def test_rerank_distributed_matches_reference_run(P, gold, model):
    from paper_2312_17649_b200.rerank import rerank_distributed

    run, _ = gold
    got = rerank_distributed(model, workload())
    assert_same_run(got, run)


def test_rerank_reference_signature_matches(P, gold, model):
    """The reference-signature per-pair ``rerank`` with the device ``score_pair`` as scorer."""
    from paper_2312_17649_b200.rerank import rerank

    run, _ = gold
    got = []
    for qid, q, cands, k in workload():
        got += rerank(model.score_pair, q, cands, top_k=k, query_id=qid)
    assert_same_run(got, run)


def test_nonfinite_and_out_of_vocab_pairs_score_minus_inf(P):
    """A pair whose activations turn non-finite (R/encoder.py:356-357) or whose ids fail _check_ids
    raises in the reference's score_pair and scores -inf in rerank (R/evaluation.py:194-197); the
    other pairs of the same packed chunk keep their own scores."""
    from paper_2312_17649_b200.rerank import rerank, rerank_distributed, score_candidates

    cfg = P.EncoderConfig(**cases.TINY, pattern="sparse", precision="f32")
    w = P.init_weights(cfg, 20)
    w["tok_emb"][37] = np.inf
    model = P.CrossEncoder(cfg, weights=w)
    q = [3, 4, 5]
    cands = [[6, 7, 8], [6, 37, 8], [9, 10], [40, 6], [11] * 70 + [99]]  # 37 poisons; 40 out of vocab
    got = score_candidates(model, q, cands)
    single = []
    for d in cands:
        try:
            single.append(model.score_pair(q, d))
        except (P.EncoderError, P.NonFiniteActivationError):
            single.append(-math.inf)
    assert np.isinf(got[1]) and np.isinf(got[3]) and np.isinf(single[1]) and np.isinf(single[3])
    np.testing.assert_allclose(got, single, atol=1e-6)  # cands[4]: out-of-vocab id truncated away
    ents = rerank_distributed(model, [("q", q, [(f"d{j}", d) for j, d in enumerate(cands)])])
    ref = rerank(model.score_pair, q, [(f"d{j}", d) for j, d in enumerate(cands)], query_id="q")
    assert [e.doc_id for e in ents] == [e.doc_id for e in ref]
    assert [e.doc_id for e in ents][-2:] == ["d1", "d3"]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, out_path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2312_17649_b200 as P
    from paper_2312_17649_b200.rerank import rerank_distributed

    torch.cuda.set_device(0)  # both ranks share the one GPU; gloo gathers on the host
    model = P.CrossEncoder(P.EncoderConfig(**cases.ELECTRA_PASSAGE, precision="f32"), seed=0)
    entries = rerank_distributed(model, workload(), rank=rank, world=world)
    if rank == 0:
        with open(out_path, "w") as fh:
            fh.write("".join(f"{e.query_id} {e.doc_id} {e.rank} {e.score!r}\n" for e in entries))
    else:
        assert entries is None
    dist.barrier()
    dist.destroy_process_group()


def test_world2_gloo_real_model_equals_single_process(P, model, tmp_path):
    """world size 2 over the real model on one GPU (each rank scores its own query block) gives the
    single-process run bit for bit (sharded scores == 1-GPU scores, bitwise)."""
    import torch.multiprocessing as mp

    from paper_2312_17649_b200.rerank import rerank_distributed

    single = rerank_distributed(model, workload())
    out = tmp_path / "run.txt"
    mp.start_processes(_gloo_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True, start_method="spawn")
    lines = out.read_text().splitlines()
    assert lines == [f"{e.query_id} {e.doc_id} {e.rank} {e.score!r}" for e in single]
