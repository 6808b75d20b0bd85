"""Host-side trainer logic vs the reference (no GPU): losses, AdamW, synthetic task.

Fixtures: tests/golden/training.npz, made by the unmodified reference
(tests/golden/make_golden.py gen_training); hand values from
T/test_training.py:45-139.
"""

import math
import os

import numpy as np
import pytest
import torch

import cases
from paper_2312_17649_b200 import training as TR

GOLD = os.path.join(os.path.dirname(__file__), "golden", "training.npz")


@pytest.fixture(scope="module")
def G():
    return np.load(GOLD)


class TestLosses:
    def test_margin_mse_values(self):
        assert TR.margin_mse_loss(3.0, 1.0, 5.0, 3.0) == 0.0
        assert TR.margin_mse_loss(2.0, 1.0, 3.0, 1.0) == pytest.approx(1.0)

    def test_ranknet_values(self):
        assert TR.ranknet_loss(1.5, 1.5) == pytest.approx(math.log(2.0))
        assert TR.ranknet_loss(2.0, 1.0) == pytest.approx(0.31326168751822286, abs=1e-12)
        assert TR.ranknet_loss(1e3, 0.0) == pytest.approx(0.0, abs=1e-12)
        assert TR.ranknet_loss(0.0, 50.0) == pytest.approx(50.0, rel=1e-9)
        assert math.isfinite(TR.ranknet_loss(-1e5, 1e5))

    @pytest.mark.parametrize("which", ["margin_mse", "ranknet"])
    def test_grads_match_finite_differences(self, which):
        rng = np.random.default_rng(0)
        sp, sn, tp, tn = (rng.normal(size=4) for _ in range(4))
        if which == "margin_mse":
            f = lambda a, b: TR.margin_mse_loss(a, b, tp, tn)  # noqa: E731
            gp, gn = TR.margin_mse_grad(sp, sn, tp, tn)
        else:
            f = TR.ranknet_loss
            gp, gn = TR.ranknet_grad(sp, sn)
        eps = 1e-6
        for i in range(4):
            e = eps * np.eye(4)[i]
            assert gp[i] == pytest.approx((f(sp + e, sn) - f(sp - e, sn)) / (2 * eps), rel=1e-5, abs=1e-9)
            assert gn[i] == pytest.approx((f(sp, sn + e) - f(sp, sn - e)) / (2 * eps), rel=1e-5, abs=1e-9)

    def test_tensor_inputs(self):
        sp = torch.tensor([1.0, 2.0])
        sn = torch.tensor([0.5, 3.0])
        gp, gn = TR.ranknet_grad(sp, sn)
        assert torch.is_tensor(gp) and gp.dtype == torch.float64
        assert TR.ranknet_loss(sp, sn) == pytest.approx(TR.ranknet_loss(sp.numpy(), sn.numpy()))


class TestAdamW:
    def test_matches_reference_updates(self, G):
        ws, gs = cases.adamw_inputs()
        tw = {n: torch.tensor(a) for n, a in ws.items()}
        opt = TR.AdamW(lr=0.05, weight_decay=0.1, warmup_steps=2, total_steps=6, moment_dtype=torch.float64)
        for step in range(5):
            opt.step(tw, {n: torch.tensor(g) for n, g in gs[step].items()})
        for n in ws:
            np.testing.assert_allclose(tw[n].numpy(), G[f"adamw|{n}"], rtol=0, atol=1e-15)

    def test_zero_grad_zero_decay_is_exact_noop(self):
        w = {"w": torch.tensor([1.0, -2.0, 3.0])}
        before = w["w"].clone()
        opt = TR.AdamW(lr=0.1, weight_decay=0.0)
        for _ in range(3):
            opt.step(w, {"w": torch.zeros(3)})
        assert torch.equal(w["w"], before)

    def test_schedule(self):
        opt = TR.AdamW(lr=1.0, warmup_steps=10, total_steps=110)
        for t, want in ((5, 0.5), (10, 1.0), (60, 0.5), (110, 0.0), (200, 0.0)):
            opt.step_count = t
            assert opt.current_lr() == pytest.approx(want)
        opt = TR.AdamW(lr=0.3)
        opt.step_count = 1000
        assert opt.current_lr() == 0.3


class TestSyntheticTask:
    def test_triples_follow_reference_draws(self, G):
        task = TR.SyntheticTask(**cases.TASK)
        rng = np.random.default_rng(3)
        got = [task.sample_triple(rng) for _ in range(5)]
        arr = np.array([list(t.query) + list(t.positive) + list(t.negative) for t in got])
        np.testing.assert_array_equal(arr, G["task_triples"])
        for t in got:
            assert task.overlap(t.query, t.positive) == task.query_terms
            assert task.overlap(t.query, t.negative) == 0
            assert (t.teacher_pos, t.teacher_neg) == (float(task.query_terms), 0.0)

    def test_validation_pools_follow_reference_draws(self, G):
        task = TR.SyntheticTask(**cases.TASK)
        val = task.sample_validation(np.random.default_rng(4), 2, per_level=2)
        np.testing.assert_array_equal([[int(d[1:]) for d, _ in vq.candidates] for vq in val], G["task_val"])
        np.testing.assert_array_equal([[list(doc) for _, doc in vq.candidates] for vq in val], G["task_val_docs"])
        for vq in val:
            for did, doc in vq.candidates:
                assert vq.relevance[did] == task.overlap(vq.query, doc)

    def test_rejects_bad_settings(self):
        with pytest.raises(TR.TrainingError):
            TR.SyntheticTask(vocab_words=3, query_terms=2, doc_len=6)
        with pytest.raises(TR.TrainingError):
            TR.SyntheticTask(query_terms=5, doc_len=4)

    def test_triple_validation(self):
        with pytest.raises(TR.TrainingError):
            TR.Triple((3,), (4, 5), (4, 5))
        with pytest.raises(TR.TrainingError):
            TR.Triple((3,), (4, 5), (5, 4), teacher_pos=1.0)


def test_unknown_loss_rejected_before_device_work():
    cfg = TR.EncoderConfig(**cases.task_config_kw("full", 4), precision="f32")
    with pytest.raises(TR.TrainingError):
        TR.train_toy(cfg, TR.SyntheticTask(**cases.TASK), steps=1, lr=1e-3, loss="hinge")
    with pytest.raises(TR.TrainingError):
        TR.train_toy(cfg, [], steps=1, lr=1e-3)


def test_trace_csv(tmp_path):
    rows = [TR.TraceRow(1, 0.5), TR.TraceRow(2, 0.25, 0.75)]
    p = tmp_path / "t.csv"
    TR.write_trace_csv(rows, p)
    assert p.read_text().splitlines() == ["step,loss,ndcg10", "1,0.50000000,", "2,0.25000000,0.750000"]
