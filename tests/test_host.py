"""CPU-only checks: C-ABI library loads and exports the header's symbols; host-side API logic."""

import math
import os
import re

import numpy as np
import pytest

import cases
from oracle import sparsecross_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "sparsecross_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:SC_API\s+)?(?:const\s+)?\w+\*?\s+\*?(sc_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_header_symbol():
    from paper_2312_17649_b200 import _lib

    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 14
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_lib.SIGNATURES)
    assert lib.sc_version() >= 10000


def test_library_is_sm100a():
    import subprocess

    from paper_2312_17649_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_invalid_arguments_map_to_reference_errors():
    import paper_2312_17649_b200 as P
    from paper_2312_17649_b200 import _lib

    with pytest.raises(P.BandShapeError):
        _lib.call("sc_band_validity", 3, -1, 3, None, None, exc=P.BandShapeError)
    assert "window" in _lib.last_error()


def test_patterns_and_links():
    import paper_2312_17649_b200 as P

    sp = P.sparse_pattern(4)
    np.testing.assert_array_equal(sp.links().reshape(3, 3),
                                  [[-1, -1, -1], [-2, -1, -2], [-1, -1, 4]])
    np.testing.assert_array_equal(P.longformer_pattern(2).links().reshape(3, 3)[1], [-1, -1, -1])
    with pytest.raises(P.AttentionError):
        P.make_pattern("strided", 3)
    with pytest.raises(P.AttentionError):
        P.AttentionPattern("sparse", {"doc": (("doc", -1),)})
    with pytest.raises(P.AttentionError):
        P.AttentionPattern("sparse", {"doc": (("doc", 1),)}, global_positions=(2,))
    lens = np.array([[1, 2, 5]])
    bad = P.AttentionPattern("x", {"cls": (("cls", math.inf),), "query": (("query", math.inf),),
                                   "doc": (("query", 0),)})
    with pytest.raises(P.AttentionError):
        P.attention.check_rows_have_keys(bad, lens, "exclude")
    P.attention.check_rows_have_keys(bad, lens, "zero-logit")


def test_partition_and_assembly_match_reference_rules():
    import paper_2312_17649_b200 as P

    seq = P.assemble_input(range(3, 13), range(3, 4088), max_positions=4096)
    assert seq.ids.shape[0] == 4096 and seq.partition.group_len("doc") == 4084
    ids, spans = O.assemble_input(list(range(3, 13)), list(range(3, 4088)), 4096)
    np.testing.assert_array_equal(seq.ids, ids)
    assert (seq.partition.cls_span, seq.partition.query_span, seq.partition.doc_span) == spans
    with pytest.raises(P.EncoderError):
        P.assemble_input(range(3, 20), [5], max_positions=12)
    with pytest.raises(P.EncoderError):
        P.SubsequencePartition((0, 1), (2, 4), (4, 6))
    assert P.qds_global_positions(4086, 30)[-1] == 4079 and len(P.qds_global_positions(4086, 30)) == 136


def test_init_weights_identical_to_oracle():
    import paper_2312_17649_b200 as P

    cfg = P.EncoderConfig(**cases.C1, precision="f32")
    a = P.init_weights(cfg, 0)
    b = O.init_weights(cases.C1, 0, np.float32)
    assert a.keys() == b.keys()
    for k in a:
        np.testing.assert_array_equal(a[k], b[k])


def test_packed_batch_layout():
    import paper_2312_17649_b200 as P

    seqs = [P.assemble_input([5, 6], [7, 8, 9]), P.assemble_input([4], [])]
    pb = P.PackedBatch.from_sequences(seqs)
    assert pb.total_tokens == 8 + 4 and pb.nseq == 2
    np.testing.assert_array_equal(pb.seq_lens, [8, 4])
    np.testing.assert_array_equal(pb.qgroup_lens, [3, 2])


def test_interpolate_positions():
    import paper_2312_17649_b200 as P

    pos = np.array([[0.0, 0.0], [2.0, 4.0], [6.0, 8.0]])
    out = P.interpolate_positions(pos, 5)
    np.testing.assert_allclose(out[1], 0.5 * pos[0] + 0.5 * pos[1])
    np.testing.assert_array_equal(out[-1], pos[-1])


def test_pack_pairs_matches_assemble_input():
    """Vectorised candidate packing == per-pair assemble_input (R/encoder.py:154-177), incl. truncation."""
    from paper_2312_17649_b200.encoder import PackedBatch, assemble_input
    from paper_2312_17649_b200.rerank import pack_pairs

    rng = np.random.default_rng(4)
    for m, maxpos in [(10, 4099), (7, 200), (1, 20)]:
        q = rng.integers(3, 1000, size=m)
        docs = [rng.integers(3, 1000, size=int(n)) for n in [0, 1, 5, 150, 4086, 5000]]
        a = pack_pairs(q, docs, maxpos)
        b = PackedBatch.from_sequences([assemble_input(q, d, maxpos) for d in docs])
        np.testing.assert_array_equal(a.ids, b.ids)
        np.testing.assert_array_equal(a.seq_lens, b.seq_lens)
        np.testing.assert_array_equal(a.qgroup_lens, b.qgroup_lens)
    with pytest.raises(ValueError):
        pack_pairs(rng.integers(3, 9, size=30), docs, 20)


class TestTrecEvaluation:
    """TREC qrels IO and nDCG@k (R/evaluation.py:68-123; hand values from T/test_evaluation.py:29-62)."""

    @staticmethod
    def run_for(qid, docs_scores):
        from paper_2312_17649_b200.rerank import RunEntry

        return [RunEntry(qid, did, rank, score) for rank, (did, score) in enumerate(docs_scores, 1)]

    def test_ideal_and_worked_example(self):
        from paper_2312_17649_b200.rerank import ndcg_at_k

        qrels = {"q1": {"a": 3, "b": 2, "c": 1, "d": 0}}
        per_query, mean = ndcg_at_k(self.run_for("q1", [("a", 4.0), ("b", 3.0), ("c", 2.0), ("d", 1.0)]), qrels, 4)
        assert per_query["q1"] == pytest.approx(1.0) and mean == pytest.approx(1.0)
        qrels = {"q": {"d1": 0, "d2": 2, "d3": 1}}
        per_query, _ = ndcg_at_k(self.run_for("q", [("d1", 3.0), ("d2", 2.0), ("d3", 1.0)]), qrels, 3)
        assert per_query["q"] == pytest.approx(0.6590018048024133, abs=1e-10)
        per_query, _ = ndcg_at_k(self.run_for("q1", [("a", 2.0), ("b", 1.0)]), {"q1": {"x": 2}}, 2)
        assert per_query["q1"] == 0.0

    def test_missing_query_and_bad_k(self):
        from paper_2312_17649_b200.rerank import EvaluationError, ndcg_at_k

        with pytest.warns(UserWarning):
            per_query, mean = ndcg_at_k(self.run_for("ghost", [("a", 1.0)]), {}, 10)
        assert per_query["ghost"] == 0.0 and mean == 0.0
        with pytest.raises(EvaluationError):
            ndcg_at_k([], {}, 0)

    def test_qrels_and_run_round_trip(self, tmp_path):
        from paper_2312_17649_b200.rerank import (EvaluationError, parse_qrels, read_qrels, read_run, write_run)

        p = tmp_path / "qrels.txt"
        p.write_text("q1 0 d1 2\n\nq1 0 d2 0\nq2 0 d9 1\n")
        assert read_qrels(p) == {"q1": {"d1": 2, "d2": 0}, "q2": {"d9": 1}}
        with pytest.raises(EvaluationError):
            parse_qrels(["q1 0 d1"])
        with pytest.raises(EvaluationError):
            parse_qrels(["q1 0 d1 -1"])
        entries = self.run_for("q1", [("d1", 0.5), ("d2", 0.25)])
        write_run(entries, tmp_path / "run.txt")  # the reference's argument order
        assert read_run(tmp_path / "run.txt") == entries


class TestSegmentScoresHost:
    """SegmentScores / segment_softmax argument checks (R/attention.py:164-210), no device needed."""

    def test_rejects_empty_and_mismatched(self):
        from paper_2312_17649_b200 import AttentionError, SegmentScores
        with pytest.raises(AttentionError):
            SegmentScores([])
        with pytest.raises(AttentionError):
            SegmentScores([np.zeros((2, 2)), np.zeros((3, 2))])
        assert SegmentScores([np.zeros((3, 2)), np.zeros((3, 5))]).rows == 3

    def test_rejects_bad_scale_and_padding(self):
        from paper_2312_17649_b200 import AttentionError, segment_softmax
        with pytest.raises(AttentionError):
            segment_softmax([np.zeros((2, 2))], scale=0.0)
        with pytest.raises(AttentionError):
            segment_softmax([np.zeros((2, 2))], scale=1.0, padding="bogus")


class TestBenchHarness:
    """benchmark.py (R/bench.py:43-408): spec checks, bit-identical inputs, FLOP model, reports."""

    @staticmethod
    def spec(**kw):
        from paper_2312_17649_b200 import BenchSpec
        d = dict(pattern="sparse", window=4, query_len=10, doc_lens=(16,), batch_size=2, repetitions=3,
                 warmup=1, precision="f32", seed=0)
        d.update(kw)
        return BenchSpec(**d)

    def test_spec_rejections(self):
        from paper_2312_17649_b200 import BenchConfigError
        for bad in (dict(batch_size=101), dict(repetitions=2), dict(pattern="strided"), dict(doc_lens=()),
                    dict(window=1.5), dict(warmup=-1)):
            with pytest.raises(BenchConfigError):
                self.spec(**bad)

    def test_ids_match_reference_golden(self):
        from paper_2312_17649_b200 import default_model_config, gen_random_batch
        g = np.load(os.path.join(os.path.dirname(__file__), "golden", "encoder.npz"))
        s = self.spec(doc_lens=(164,), batch_size=8)
        cfg = default_model_config(s, vocab_size=cases.C1["vocab_size"])
        b = gen_random_batch(s, 164, cfg)
        np.testing.assert_array_equal(b.ids, g["c1_ids"])
        assert b.partition.seq_len == 177
        q = self.spec(pattern="qds", doc_lens=(120,))
        assert len(gen_random_batch(q, 120, default_model_config(q)).pattern.global_positions) == 4

    def test_flop_model_matches_reference_golden(self):
        from paper_2312_17649_b200 import flop_count, make_pattern
        g = np.load(os.path.join(os.path.dirname(__file__), "golden", "encoder.npz"))
        c1 = flop_count(make_pattern("sparse", 4), (1, 11, 165), 32, 2, 2, 64)
        assert c1.total == g["c1_flops"][3]
        c3 = flop_count(make_pattern("sparse", 4), (1, 11, 4087), 768, 12, 12, 3072)
        assert [c3.attention, c3.projections, c3.feed_forward] == list(g["c3_flops"][:3])
        for name, w, gl in (("full", math.inf, ()), ("longformer", 8, ()), ("qds", 4, (29, 59, 89, 119)),
                            ("sparse", 2, ())):
            mine = flop_count(make_pattern(name, w, gl), (1, 11, 120), 8, 2, ff_dim=16)
            ref = O.flop_count(O.make_pattern(name, w, gl), (1, 11, 120), 8, 2, 16)
            assert (mine.attention, mine.projections, mine.feed_forward) == \
                (ref["attention"], ref["projections"], ref["feed_forward"])
        s = sum((1, 11, 20))
        assert flop_count(make_pattern("full", math.inf), (1, 11, 20), 8, 1, ff_dim=16).attention_qk == s * s * 8
        assert flop_count(make_pattern("sparse", 9), (1, 5, 10), 4, 1, ff_dim=8).window_exceeds_dense
        assert not flop_count(make_pattern("sparse", 2), (1, 5, 10), 4, 1, ff_dim=8).window_exceeds_dense

    def test_emit_report(self):
        from paper_2312_17649_b200 import BenchConfigError, BenchRecord, emit_report

        def rec(pattern="sparse", window=4, t=1e-3, peak=1000, oom=False):
            return BenchRecord(pattern, window, 10, 16, 2, None if oom else t, None if oom else 0.0,
                               None if oom else peak, None if oom else 0, 1234, 1, oom)
        lines = emit_report([rec()], "csv").strip().split("\n")
        assert lines[0] == "pattern,w,query_len,doc_len,batch,time_per_doc_s,peak_bytes,flops"
        assert lines[1].startswith("sparse,4,10,16,2,")
        assert "OOM" in emit_report([rec(oom=True)], "csv")
        md = emit_report([rec(), rec("full", math.inf, 2e-3, 2000)], "md", baseline=("sparse", 4))
        assert "(+100%)" in md and "| full " in md and "inf" in md
        with pytest.raises(BenchConfigError):
            emit_report([], "csv")
        with pytest.raises(BenchConfigError):
            emit_report([rec()], "md", baseline=("full", 3))
        with pytest.raises(BenchConfigError):
            emit_report([rec()], "html")


def test_bench_batch_prefix_is_the_ranking_golden():
    """bench.py's synthetic batch starts with exactly these candidates (its parity field relies on it)."""
    import bench
    import paper_2312_17649_b200 as P

    def doc_batch(n, cfg):
        seqs = []
        for j in range(n):
            q = np.random.default_rng((0, 0)).integers(3, cfg.vocab_size, size=10)
            d = np.random.default_rng((0, 0, j)).integers(3, cfg.vocab_size, size=4086)
            seqs.append(P.assemble_input(q, d, cfg.max_positions))
        return P.PackedBatch.from_sequences(seqs)


    cfg = dict(bench.ELECTRA, max_positions=4099)
    batch = bench.make_batch(P, cfg, 4086, 4, 0)
    want = doc_batch(4, P.EncoderConfig(**cases.ELECTRA_DOC, precision="bf16"))
    assert np.array_equal(batch.ids, want.ids)


def test_bench_reference_arm_line_matches_gpu_arm_config():
    """`bench.py --impl reference` (the CPU arm the driver times beside ours) prints one contract line
    with the same metric and the same ``config`` dict the GPU arm prints for the same flags."""
    import json
    import subprocess
    import sys
    import types

    import bench

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3",
                          "--ref-budget", "1", "--doc-len", "164"], cwd=root, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["unit"] == "pairs/s"
    assert d["higher_is_better"] is True and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    args = types.SimpleNamespace(prune_last_layer=False, varlen=False)
    s = bench.QUERY_LEN + 164 + 3
    assert d["config"] == bench.bench_config(args, 1, 64, s, 164, True, 64 * s)


def test_bench_reference_arm_under_torchrun_world2():
    """The driver launches the reference arm like ours (torchrun, N ranks): rank 0 alone times and
    prints one line with n_gpus N; the other ranks exit 0 without work."""
    import json
    import socket
    import subprocess
    import sys

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl",
                          "reference", "--gpus", "2", "--steps", "1", "--warmup", "3", "--ref-budget", "1",
                          "--doc-len", "164"], cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["config"]["parallelism"] == "dp2"
