"""GPU parity of the backward path and the trainer.

Pins: band / attention / encoder gradients against the reference's own
adjoints (tests/golden/training.npz from R/band.py:239-274,
R/attention.py:476-507, R/encoder.py:511-533), a 3-step train_toy run
against the reference trainer, and the reference's trainer properties
(T/test_training.py:170-240).  Tolerances: fp32 device arithmetic vs the
reference's f64 -- gradients within 1e-4 of their tensor's max magnitude
(1e-3 on the 2-layer encoder chains); bf16 within 3e-2.
"""

import math
import os

import numpy as np
import pytest
import torch

import cases

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "training.npz")


@pytest.fixture(scope="module")
def P():
    import paper_2312_17649_b200 as pkg

    return pkg


@pytest.fixture(scope="module")
def G():
    return np.load(GOLD)


def close(got, want, tol):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    scale = max(1.0, float(np.abs(want).max(initial=0.0)))
    err = float(np.abs(got - want).max(initial=0.0))
    assert err <= tol * scale, f"max err {err:.3e} > {tol:.1e} x {scale:.3e}"


# ---------------------------------------------------------------------------
# band adjoints
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("idx", range(len(cases.BAND_CASES)))
def test_band_backward_vs_reference(P, G, idx):
    case = cases.BAND_CASES[idx]
    s, t, w, d = case
    q, k, p, v = (torch.tensor(a, dtype=torch.float32, device="cuda") for a in cases.band_inputs(idx, case))
    gb, go = (torch.tensor(a, dtype=torch.float32, device="cuda") for a in cases.band_grad_inputs(idx, case))
    gq, gk = P.band_scores_backward(gb, q, k, w)
    gp, gv = P.band_apply_backward(go, p, v, w)
    for got, key in ((gq, "gq"), (gk, "gk"), (gp, "gp"), (gv, "gv")):
        close(got.cpu().numpy(), G[f"band_{key}_{idx}"], 1e-5)


def test_band_backward_2d_wrappers_and_errors(P):
    q = torch.randn(6, 3, device="cuda")
    k = torch.randn(6, 3, device="cuda")
    g = torch.randn(6, 3, device="cuda")
    gq, gk = P.band_qk_backward(g, q, k, 1)
    assert gq.shape == (6, 3) and gk.shape == (6, 3)
    with pytest.raises(P.BandShapeError):
        P.band_scores_backward(torch.randn(6, 5, device="cuda"), q, k, 1)
    with pytest.raises(P.BandShapeError):
        P.band_apply_backward(torch.randn(5, 3, device="cuda"), g, k, 1)


# ---------------------------------------------------------------------------
# fused attention adjoint
# ---------------------------------------------------------------------------

def attention_grads(P, x, go, m, n, pattern, padding, dtype=torch.float32):
    """x (3, H, s, d), go (H, s, d) -> (dq, dk, dv) each (H, s, d) float64 through sc_attn_bwd."""
    from paper_2312_17649_b200.training import PatternAttention

    _, H, s, d = x.shape
    lay = P.PackedLayout.from_lengths([s], [m + 1], device="cuda",
                                      qds_positions=[pattern.global_positions] if pattern.global_positions else None)
    qkv = torch.from_numpy(np.ascontiguousarray(x.transpose(2, 0, 1, 3).reshape(s, 3 * H * d))).cuda().to(dtype)
    qkv.requires_grad_(True)
    out = PatternAttention.apply(qkv, lay, pattern, H, math.sqrt(d), padding, True)
    g = torch.from_numpy(np.ascontiguousarray(go.transpose(1, 0, 2).reshape(s, H * d))).cuda().to(dtype)
    out.backward(g)
    gr = qkv.grad.double().cpu().numpy().reshape(s, 3, H, d).transpose(1, 2, 0, 3)
    return gr[0], gr[1], gr[2]


@pytest.mark.parametrize("idx", range(len(cases.ATTN_CASES)))
def test_attention_backward_vs_reference(P, G, idx):
    case = cases.ATTN_CASES[idx]
    name, w, pad, m, n, heads, d, dt = case
    x = cases.attn_inputs(idx, case)
    go = cases.attn_grad_out(idx, case)
    pat = P.make_pattern(name, w, cases.attn_globals(name, m, n))
    got = attention_grads(P, x, go, m, n, pat, pad)
    for tag, g in zip(("dq", "dk", "dv"), got):
        want = G[f"attn_{tag}_{idx}"]
        if want.shape != g.shape:  # large cases are stored as 4 projections per row
            g = g @ cases.grad_projection(idx, d)
        close(g, want, 1e-4)


@pytest.mark.parametrize("idx", [0, 13, 24, 29, 36])
def test_attention_backward_bf16(P, G, idx):
    case = cases.ATTN_CASES[idx]
    name, w, pad, m, n, heads, d, dt = case
    x = cases.attn_inputs(idx, case)
    go = cases.attn_grad_out(idx, case)
    pat = P.make_pattern(name, w, cases.attn_globals(name, m, n))
    got = attention_grads(P, x, go, m, n, pat, pad, torch.bfloat16)
    for tag, g in zip(("dq", "dk", "dv"), got):
        want = G[f"attn_{tag}_{idx}"]
        if want.shape != g.shape:
            g = g @ cases.grad_projection(idx, d)
        close(g, want, 3e-2)


@pytest.mark.parametrize("pattern,window,padding", [
    ("sparse", 4, "exclude"), ("sparse", 16, "zero-logit"), ("longformer", 8, "exclude"),
    ("full", math.inf, "exclude"), ("qds", 4, "exclude"), ("qds", 2, "zero-logit"),
])
def test_attention_backward_packed_varlen_vs_dense_autograd(P, pattern, window, padding):
    """Many ragged sequences in one launch vs a dense masked fp64 torch autograd reference."""
    from paper_2312_17649_b200.training import PatternAttention

    rng = np.random.default_rng(21)
    m = rng.integers(1, 12, size=6)
    n = rng.integers(1, 150, size=6)
    seq = m + n + 3
    H, d = 2, 32
    lay = P.PackedLayout.from_lengths(seq, m + 1, device="cuda", qds_every=7 if pattern == "qds" else 0)
    pat = P.make_pattern(pattern, window)
    T = int(seq.sum())
    qkv = (torch.randn(T, 3 * H * d, device="cuda", generator=torch.Generator("cuda").manual_seed(3)))
    qkv.requires_grad_(True)
    out = PatternAttention.apply(qkv, lay, pat, H, math.sqrt(d), padding, True)
    go = torch.randn_like(out)
    out.backward(go)
    # dense reference per sequence
    ref = torch.zeros(T, 3 * H * d, dtype=torch.float64, device="cuda")
    cu = np.concatenate([[0], np.cumsum(seq)])
    for j in range(len(seq)):
        a, b = int(cu[j]), int(cu[j + 1])
        s = b - a
        mask = torch.from_numpy(lay.mask(j, pat)).cuda()
        x = qkv.detach()[a:b].double().reshape(s, 3, H, d).requires_grad_(True)
        q, k, v = x[:, 0].transpose(0, 1), x[:, 1].transpose(0, 1), x[:, 2].transpose(0, 1)
        logits = q @ k.transpose(-1, -2) / math.sqrt(d)
        logits = logits.masked_fill(~mask, -math.inf)
        if padding == "zero-logit":
            # out-of-range band slots join the softmax with logit 0 and no value
            nz = torch.from_numpy(zero_logit_slots(lay, j, pat)).cuda().double()
            mx = torch.maximum(logits.amax(-1), torch.where(nz > 0, 0.0, -math.inf))
            e = torch.exp(logits - mx[..., None])
            den = e.sum(-1) + nz * torch.exp(-mx)
            o = (e / den[..., None]) @ v
        else:
            o = torch.softmax(logits, -1) @ v
        o.transpose(0, 1).reshape(s, H * d).backward(go[a:b].double())
        ref[a:b] = x.grad.reshape(s, 3 * H * d)
    close(qkv.grad.double().cpu().numpy(), ref.cpu().numpy(), 1e-4)


def zero_logit_slots(lay, j, pat):
    """Per source row of sequence j: number of out-of-range windowed slots (R/attention.py:244-247)."""
    L = pat.links().reshape(3, 3)
    ql = int(lay.qlen_host[j])
    s = int(lay.cu_host[j + 1] - lay.cu_host[j])
    lens = (1, ql, s - 1 - ql)
    offs = (0, 1, 1 + ql)
    cnt = np.zeros(s)
    flags = None if lay.tok_flags is None else lay.tok_flags.cpu().numpy()
    for i in range(s):
        gs = 0 if i == 0 else (1 if i < 1 + ql else 2)
        r = i - offs[gs]
        if gs == 2 and flags is not None and flags[int(lay.cu_host[j]) + i]:
            continue  # QDS global rows attend densely
        for t in range(3):
            w = int(L[gs, t])
            if w < 0:
                continue
            lo, hi = max(0, r - w), min(lens[t], r + w + 1)
            cnt[i] += (2 * w + 1) - max(0, hi - lo)
    return cnt


# ---------------------------------------------------------------------------
# encoder gradients and the trainer
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["full", "longformer", "qds", "sparse"])
@pytest.mark.parametrize("pad", ["exclude", "zero-logit"])
def test_encoder_gradients_vs_reference(P, G, name, pad):
    cfg = P.EncoderConfig(**cases.TINY, pattern=name, padding=pad, precision="f64")
    model = P.TrainableCrossEncoder(cfg, seed=15)
    seqs = [P.assemble_input(*cases.tiny_sequence(16 + j, 4, 13, cfg.vocab_size), cfg.max_positions)
            for j in range(2)]
    ids = np.stack([s.ids for s in seqs])
    scores, cache = model.score(ids, seqs[0].partition, want_cache=True)
    key = f"grad_{name}_{pad}"
    close(scores, G[key + "_scores"], 1e-5)
    grads = model.backward(cache, cases.TRAIN_GRAD_SCORES)
    names = {k.split("|", 1)[1] for k in G.files if k.startswith(key + "|")}
    assert names == set(grads)
    for wn in names:
        close(grads[wn].cpu().numpy(), G[f"{key}|{wn}"], 1e-4)


@pytest.mark.parametrize("pattern,window", [("full", 4), ("sparse", 1), ("qds", 4)])
def test_train_toy_matches_reference_trainer(P, G, pattern, window):
    cfg = P.EncoderConfig(**cases.task_config_kw(pattern, window), precision="f32")
    res = P.train_toy(cfg, P.SyntheticTask(**cases.TASK), steps=3, lr=1e-3, seed=0, batch_pairs=4)
    key = f"toy_{pattern}_{window}"
    np.testing.assert_allclose([r.loss for r in res.trace], G[key + "_loss"], rtol=1e-4)
    last_ln2_b = f"L{cfg.layers - 1}.ln2_b"
    for wn, t in res.model.weights.items():
        if wn.endswith(".bk") or wn == last_ln2_b:
            # exact gradient 0: the key bias shifts every logit of a row equally; the last
            # LayerNorm bias reaches the loss only through sum(dL/ds) = 0 of a pairwise loss.
            # Both trainers feed Adam pure rounding noise, which it normalises to +-lr.
            assert float(t.detach().abs().max()) <= 2e-3
            continue
        # Adam's first steps move every weight by ~lr * sign(g): compare at a fraction of lr
        close(t.detach().cpu().numpy(), G[f"{key}|{wn}"], 2e-4)


TASK_KW = cases.TASK


def task_cfg(P, pattern="full", window=4, **kw):
    d = cases.task_config_kw(pattern, window)
    d.update(kw)
    d.setdefault("precision", "f32")
    return P.EncoderConfig(**d)


def test_zero_learning_rate_changes_nothing(P):
    task = P.SyntheticTask(**TASK_KW)
    rng = np.random.default_rng(9)
    fixed = [task.sample_triple(rng) for _ in range(16)]
    cfg = task_cfg(P)
    res = P.train_toy(cfg, fixed, steps=5, lr=0.0, seed=3)
    fresh = P.init_weights(cfg, 3)
    for n, a in fresh.items():
        np.testing.assert_array_equal(res.model.weights[n].detach().cpu().numpy(), a.astype(np.float32))
    losses = [r.loss for r in res.trace]
    assert losses == [losses[0]] * len(losses)


@pytest.mark.parametrize("pattern", ["full", "longformer", "qds", "sparse"])
@pytest.mark.parametrize("window", [math.inf, 4])
def test_loss_decreases_over_first_100_steps(P, pattern, window):
    res = P.train_toy(task_cfg(P, pattern, window), P.SyntheticTask(**TASK_KW), steps=100, lr=3e-3, seed=0,
                      lr_decay=False)
    losses = [r.loss for r in res.trace]
    assert np.mean(losses[-10:]) < np.mean(losses[:10])


def test_bf16_training_decreases_loss(P):
    cfg = task_cfg(P, "sparse", 2, precision="bf16")
    res = P.train_toy(cfg, P.SyntheticTask(**TASK_KW), steps=100, lr=3e-3, seed=0, lr_decay=False)
    losses = [r.loss for r in res.trace]
    assert np.mean(losses[-10:]) < np.mean(losses[:10])


def test_determinism(P):
    cfg = task_cfg(P)
    r1 = P.train_toy(cfg, P.SyntheticTask(**TASK_KW), steps=8, lr=1e-3, seed=11)
    r2 = P.train_toy(cfg, P.SyntheticTask(**TASK_KW), steps=8, lr=1e-3, seed=11)
    for n in r1.model.weights:  # bit-exact: the attention adjoint has no atomics
        assert torch.equal(r1.model.weights[n], r2.model.weights[n]), n
    assert [r.loss for r in r1.trace] == [r.loss for r in r2.trace]


def test_divergence_aborts_with_step_index(P):
    task = P.SyntheticTask(**TASK_KW)
    base = task.sample_triple(np.random.default_rng(10))
    bad = P.Triple(base.query, base.positive, base.negative, 1e200, -1e200)
    with pytest.raises(P.TrainingDivergedError) as exc:
        P.train_toy(task_cfg(P), [bad] * 16, steps=5, lr=1e-3, seed=0)
    assert exc.value.step == 1


def test_validation_trace(P, tmp_path):
    task = P.SyntheticTask(**TASK_KW)
    val = task.sample_validation(np.random.default_rng(7), 4, per_level=2)
    res = P.train_toy(task_cfg(P), task, steps=6, lr=1e-3, seed=0, eval_every=3, val_set=val)
    assert [r.step for r in res.trace if r.ndcg10 is not None] == [3, 6]
    assert 0.0 <= res.final_ndcg <= 1.0
    P.write_trace_csv(res.trace, tmp_path / "trace.csv")
    assert (tmp_path / "trace.csv").read_text().startswith("step,loss,ndcg10\n")


@pytest.mark.parametrize("pattern,window,layers,loss", [
    ("full", 4, 0, "margin_mse"), ("full", 4, 2, "margin_mse"), ("sparse", 1, 2, "margin_mse"),
    ("qds", 4, 1, "ranknet"),
])
def test_grad_check_directional(P, pattern, window, layers, loss):
    task = P.SyntheticTask(**TASK_KW)
    model = P.TrainableCrossEncoder(task_cfg(P, pattern, window, layers=layers), seed=1)
    triples = [task.sample_triple(np.random.default_rng(5)) for _ in range(2)]
    assert P.grad_check(model, triples, eps=1e-3, samples=6, loss=loss) < 2e-2


def test_trained_weights_serve_through_inference_engine(P):
    cfg = task_cfg(P, "sparse", 2)
    res = P.train_toy(cfg, P.SyntheticTask(**TASK_KW), steps=4, lr=1e-3, seed=0)
    eng = res.model.to_inference()
    task = P.SyntheticTask(**TASK_KW)
    t = task.sample_triple(np.random.default_rng(1))
    seq = P.assemble_input(t.query, t.positive, cfg.max_positions)
    a = res.model.score(seq.ids[None], seq.partition)
    b = eng.score(seq.ids[None], seq.partition)
    np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("pattern,window,padding", [
    ("sparse", 4, "exclude"), ("sparse", 8, "zero-logit"), ("longformer", 16, "exclude"),
    ("sparse", 24, "exclude"), ("longformer", 2, "zero-logit"), ("sparse", 0, "exclude"),
])
def test_attention_backward_bf16_tiled_path_vs_fp32(P, pattern, window, padding):
    """bf16 d=64 batches take the tiled tensor-core doc-band kernels; compare with the fp32
    generic adjoint on the same (bf16-rounded) inputs, ragged docs incl. 1-token and 64-multiples."""
    from paper_2312_17649_b200.training import attention_backward

    rng = np.random.default_rng(5)
    m = rng.integers(1, 30, size=9)
    n = np.concatenate([rng.integers(1, 300, size=6), [1, 63, 128]])
    seq = m + n + 3
    H, d = 3, 64
    lay = P.PackedLayout.from_lengths(seq, m + 1, device="cuda")
    pat = P.make_pattern(pattern, window)
    T = int(seq.sum())
    gen = torch.Generator("cuda").manual_seed(11)
    qkv = torch.randn(T, 3 * H * d, device="cuda", generator=gen).bfloat16()
    dout = torch.randn(T, H * d, device="cuda", generator=gen).bfloat16()
    out16 = P.attend_packed(qkv[:, :H * d], qkv[:, H * d:2 * H * d], qkv[:, 2 * H * d:], lay, pat, H,
                            padding=padding)
    g16 = torch.empty(T, 3 * H * d, device="cuda")
    attention_backward(qkv, out16, dout, g16, lay, pat, H, 8.0, padding)
    q32 = qkv.float()
    out32 = P.attend_packed(q32[:, :H * d], q32[:, H * d:2 * H * d], q32[:, 2 * H * d:], lay, pat, H,
                            padding=padding, algo="generic")
    g32 = torch.empty_like(g16)
    attention_backward(q32, out32, dout.float(), g32, lay, pat, H, 8.0, padding)
    assert torch.isfinite(g16).all()
    for c in range(3):
        a, b = g16[:, c * H * d:(c + 1) * H * d], g32[:, c * H * d:(c + 1) * H * d]
        err = float((a - b).abs().max())
        assert err <= 3e-2 * max(1.0, float(b.abs().max())), (c, err)


def test_fused_adamw_matches_float64_reference_path(P):
    """sc_adamw_step on a ParamDict == the per-tensor float64 path (the reference's update)."""
    from paper_2312_17649_b200.training import AdamW, ParamDict

    ws, gs = cases.adamw_inputs()
    order = sorted(ws)
    flat = torch.cat([torch.tensor(np.asarray(ws[n], np.float32)).reshape(-1) for n in order]).cuda()
    views, off = {}, 0
    for n in order:
        k = int(np.size(ws[n]))
        views[n] = flat[off:off + k].view(np.shape(ws[n]))
        off += k
    pd = ParamDict(views, flat, order)
    ref = {n: torch.tensor(np.asarray(ws[n], np.float32)).double() for n in order}
    o1 = AdamW(lr=0.05, weight_decay=0.1, warmup_steps=2, total_steps=6)
    o2 = AdamW(lr=0.05, weight_decay=0.1, warmup_steps=2, total_steps=6, moment_dtype=torch.float64)
    for step in range(5):
        o1.step(pd, {n: torch.tensor(np.asarray(gs[step][n], np.float32)).cuda() for n in order})
        o2.step(ref, {n: torch.tensor(np.asarray(gs[step][n], np.float32)).double() for n in order})
    for n in order:
        np.testing.assert_allclose(pd[n].cpu().numpy(), ref[n].numpy(), rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("cols", [16, 96, 768, 1000])
@pytest.mark.parametrize("adt,bdt", [(torch.float32, torch.bfloat16), (torch.float32, None),
                                     (torch.bfloat16, torch.float32), (torch.float32, torch.float32)])
def test_residual_layernorm_kernels_vs_torch(P, cols, adt, bdt):
    from paper_2312_17649_b200.training import ResidualLayerNorm

    gen = torch.Generator("cuda").manual_seed(cols)
    rows = 1531
    a = (torch.randn(rows, cols, device="cuda", generator=gen) * 3 + 1).to(adt).requires_grad_(True)
    b = None if bdt is None else torch.randn(rows, cols, device="cuda", generator=gen).to(bdt).requires_grad_(True)
    g = (torch.rand(cols, device="cuda", generator=gen) + 0.5).requires_grad_(True)
    be = torch.randn(cols, device="cuda", generator=gen).requires_grad_(True)
    y = ResidualLayerNorm.apply(a, b, g, be)
    dy = torch.randn(rows, cols, device="cuda", generator=gen)
    y.backward(dy)
    a64 = a.detach().double().requires_grad_(True)
    b64 = None if b is None else b.detach().double().requires_grad_(True)
    g64, be64 = g.detach().double().requires_grad_(True), be.detach().double().requires_grad_(True)
    x = a64 + (0 if b64 is None else b64)
    y64 = torch.nn.functional.layer_norm(x, (cols,), g64, be64, 1e-12)
    y64.backward(dy.double())
    close(y.detach().cpu().numpy(), y64.detach().cpu().numpy(), 2e-5)
    tol_x = 2e-5 if adt == torch.float32 else 2e-2
    close(a.grad.float().cpu().numpy(), a64.grad.cpu().numpy(), tol_x)
    if b is not None:
        close(b.grad.float().cpu().numpy(), b64.grad.cpu().numpy(), 2e-2 if bdt == torch.bfloat16 else 2e-5)
    close(g.grad.cpu().numpy(), g64.grad.cpu().numpy(), 1e-4)
    close(be.grad.cpu().numpy(), be64.grad.cpu().numpy(), 1e-4)


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("rows,cols", [(1, 8), (777, 3072), (5000, 768), (33, 13)])
def test_colsum_vs_torch(P, dt, rows, cols):
    from paper_2312_17649_b200.training import column_sum

    x = torch.randn(rows, cols + 5, device="cuda").to(dt)[:, :cols]  # strided rows
    got = column_sum(x)
    want = x.double().sum(0)
    close(got.cpu().numpy(), want.cpu().numpy(), 1e-5)
    assert torch.equal(column_sum(x), got)  # deterministic


@pytest.mark.parametrize("dt,tol", [(torch.float32, 1e-5), (torch.bfloat16, 2e-2)])
def test_linear_gelu_vs_torch(P, dt, tol):
    from paper_2312_17649_b200.training import LinearGelu

    gen = torch.Generator("cuda").manual_seed(2)
    x = torch.randn(1000, 96, device="cuda", generator=gen).requires_grad_(True)
    w = (torch.randn(96, 256, device="cuda", generator=gen) * 0.2).requires_grad_(True)
    b = torch.randn(256, device="cuda", generator=gen).requires_grad_(True)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        y = LinearGelu.apply(x, w, None, b, None, dt)
        gy = torch.randn(y.shape, device="cuda", generator=gen)
        y.backward(gy.to(y.dtype))
        x64, w64, b64 = (t.detach().double().requires_grad_(True) for t in (x, w, b))
        if dt == torch.bfloat16:  # the reference sees the same bf16-rounded GEMM inputs
            x64 = x.detach().bfloat16().double().requires_grad_(True)
            w64 = w.detach().bfloat16().double().requires_grad_(True)
        y64 = torch.nn.functional.gelu(x64 @ w64 + b64)
        y64.backward(gy.to(y.dtype).double())
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    close(y.float().detach().cpu().numpy(), y64.detach().cpu().numpy(), tol)
    close(x.grad.cpu().numpy(), x64.grad.cpu().numpy(), tol)
    close(w.grad.cpu().numpy(), w64.grad.cpu().numpy(), tol)
    close(b.grad.cpu().numpy(), b64.grad.cpu().numpy(), tol)


@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_graphed_train_step_matches_eager(P, precision):
    """GraphedTrainStep (CUDA-graph forward+backward, fused AdamW) == eager train_step."""
    from paper_2312_17649_b200.training import GraphedTrainStep, _batch_arrays, train_step

    task = P.SyntheticTask(**TASK_KW)
    cfg = task_cfg(P, "sparse", 2, precision=precision)
    rng = np.random.default_rng(0)
    batches = [[task.sample_triple(rng) for _ in range(4)] for _ in range(3)]
    m1 = P.TrainableCrossEncoder(cfg, seed=0)
    o1 = P.AdamW(1e-3)
    eager = [train_step(m1, o1, b) for b in batches]
    m2 = P.TrainableCrossEncoder(cfg, seed=0)
    o2 = P.AdamW(1e-3)
    ids, part = _batch_arrays(batches[0], cfg.max_positions)
    g = GraphedTrainStep(m2, o2, P.PackedBatch.from_ids(ids, part), warmup=0)
    graphed = []
    for b in batches:
        ids, part = _batch_arrays(b, cfg.max_positions)
        gap = np.array([t.teacher_pos - t.teacher_neg for t in b])
        graphed.append(float(g(ids.reshape(-1), gap)))
    np.testing.assert_allclose(graphed, eager, rtol=1e-6)
    for n in m1.weights:
        torch.testing.assert_close(m2.weights[n], m1.weights[n], rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("pattern,window,padding", [("sparse", 4, "exclude"), ("longformer", 8, "zero-logit")])
def test_attention_backward_long_sequences_split_head_pass(P, pattern, window, padding):
    """Few long sequences: the head-row pass splits each (sequence, head)'s keys over CTAs
    (ordered partial reductions); bf16 tiled path vs the fp32 generic adjoint."""
    from paper_2312_17649_b200.training import attention_backward

    m = np.array([10, 25])
    n = np.array([2600, 3333])
    seq = m + n + 3
    H, d = 2, 64
    lay = P.PackedLayout.from_lengths(seq, m + 1, device="cuda")
    pat = P.make_pattern(pattern, window)
    T = int(seq.sum())
    gen = torch.Generator("cuda").manual_seed(17)
    qkv = torch.randn(T, 3 * H * d, device="cuda", generator=gen).bfloat16()
    dout = torch.randn(T, H * d, device="cuda", generator=gen).bfloat16()
    out16 = P.attend_packed(qkv[:, :H * d], qkv[:, H * d:2 * H * d], qkv[:, 2 * H * d:], lay, pat, H,
                            padding=padding)
    g16 = torch.empty(T, 3 * H * d, device="cuda")
    attention_backward(qkv, out16, dout, g16, lay, pat, H, 8.0, padding)
    q32 = qkv.float()
    out32 = P.attend_packed(q32[:, :H * d], q32[:, H * d:2 * H * d], q32[:, 2 * H * d:], lay, pat, H,
                            padding=padding, algo="generic")
    g32 = torch.empty_like(g16)
    attention_backward(q32, out32, dout.float(), g32, lay, pat, H, 8.0, padding)
    for c in range(3):
        a, b = g16[:, c * H * d:(c + 1) * H * d], g32[:, c * H * d:(c + 1) * H * d]
        err = float((a - b).abs().max())
        assert err <= 3e-2 * max(1.0, float(b.abs().max())), (c, err)
    # the head rows (cls + query group) specifically
    for j in range(2):
        r0 = int(lay.cu_host[j])
        a, b = g16[r0:r0 + m[j] + 2, :H * d], g32[r0:r0 + m[j] + 2, :H * d]
        assert float((a - b).abs().max()) <= 3e-2 * max(1.0, float(b.abs().max()))
    # deterministic
    g16b = torch.empty_like(g16)
    attention_backward(qkv, out16, dout, g16b, lay, pat, H, 8.0, padding)
    assert torch.equal(g16, g16b)


def test_attention_backward_minimal_workspace_fallback(P):
    """sc_attn_bwd with only the T*H*8-byte statistics workspace: no head-key partials, no split
    head pass -> the generic head-key pass; same gradients as with the full workspace."""
    from paper_2312_17649_b200 import _lib

    rng = np.random.default_rng(9)
    m = rng.integers(1, 12, size=5)
    n = rng.integers(50, 400, size=5)
    seq = m + n + 3
    H, d = 2, 64
    lay = P.PackedLayout.from_lengths(seq, m + 1, device="cuda")
    pat = P.make_pattern("sparse", 4)
    T = int(seq.sum())
    qkv = torch.randn(T, 3 * H * d, device="cuda").bfloat16()
    dout = torch.randn(T, H * d, device="cuda").bfloat16()
    out = P.attend_packed(qkv[:, :H * d], qkv[:, H * d:2 * H * d], qkv[:, 2 * H * d:], lay, pat, H)

    def run(ws_bytes):
        g = torch.empty(T, 3 * H * d, device="cuda")
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
        base, gb = qkv.data_ptr(), g.data_ptr()
        _lib.call("sc_attn_bwd", base, base + H * d * 2, base + 2 * H * d * 2, qkv.stride(0), out.data_ptr(),
                  out.stride(0), dout.data_ptr(), dout.stride(0), gb, gb + H * d * 4, gb + 2 * H * d * 4,
                  g.stride(0), _lib.DTYPE_F32, lay.cu_seqlens.data_ptr(), lay.qgroup_len.data_ptr(), lay.nseq, T,
                  H, d, pat.links().ctypes.data, _lib.PAD_EXCLUDE, 8.0, _lib.DTYPE_BF16, None, None, None,
                  lay.seq_tile_base.data_ptr(), lay.tile_rows, lay.max_qgroup_len, lay.n_tiles, ws.data_ptr(),
                  ws_bytes, _lib.stream_handle())
        return g

    full = run(_lib.load().sc_attn_bwd_workspace_bytes(T, H, lay.nseq, lay.max_qgroup_len))
    small = run(T * H * 8)
    close(small.cpu().numpy(), full.cpu().numpy(), 2e-2)  # bf16 P / dS in the mma paths


# ---------------------------------------------------------------------------
# reference-shaped primitives (R/encoder.py:250-443, R/attention.py:260-269, :348-378, :476-507)
# ---------------------------------------------------------------------------

def test_gelu_layer_norm_primitives_vs_formulas(P):
    from scipy.special import erf

    from paper_2312_17649_b200 import encoder as E

    rng = np.random.default_rng(3)
    x = rng.standard_normal((3, 7, 96)) * 3
    want = 0.5 * x * (1 + erf(x / np.sqrt(2)))
    close(E.gelu(x), want, 1e-5)
    dwant = 0.5 * (1 + erf(x / np.sqrt(2))) + x * np.exp(-0.5 * x * x) / np.sqrt(2 * np.pi)
    close(E.gelu_grad(x), dwant, 1e-5)
    g, b = rng.random(96) + 0.5, rng.standard_normal(96)
    y, (xhat, inv) = E.layer_norm(x, g, b)
    mu = x.mean(-1, keepdims=True)
    iv = 1 / np.sqrt(((x - mu) ** 2).mean(-1, keepdims=True) + 1e-12)
    close(y, g * (x - mu) * iv + b, 1e-5)
    close(inv, iv, 1e-5)
    gy = rng.standard_normal(x.shape)
    dx, dg, db = E.layer_norm_backward(gy, (xhat, inv), g)
    xh = (x - mu) * iv
    dxh = gy * g
    dx_want = iv * (dxh - dxh.mean(-1, keepdims=True) - xh * (dxh * xh).mean(-1, keepdims=True))
    close(dx, dx_want, 1e-4)
    close(dg, (gy * xh).sum((0, 1)), 1e-4)
    close(db, gy.sum((0, 1)), 1e-4)


@pytest.mark.parametrize("idx", [0, 7, 13, 19, 25, 31, 34, 35])
def test_group_attention_backward_api_vs_reference(P, G, idx):
    """group_attention(want_cache=True) + group_attention_backward per group, summed like layer_backward."""
    case = cases.ATTN_CASES[idx]
    name, w, pad, m, n, heads, d, dt = case
    x = cases.attn_inputs(idx, case)
    go = cases.attn_grad_out(idx, case)
    spans = cases.attn_spans(m, n)
    qkv = {g: tuple(a[:, lo:hi, :] for a in x) for g, (lo, hi) in zip(P.GROUPS, spans)}
    pat = P.make_pattern(name, w, cases.attn_globals(name, m, n))
    s = m + n + 3
    dq, dk, dv = (np.zeros((heads, s, d)) for _ in range(3))
    span = dict(zip(P.GROUPS, spans))
    for g in P.GROUPS:
        lo, hi = span[g]
        _, cache = P.group_attention(qkv, g, pat, math.sqrt(d), pad, want_cache=True)
        gq, contrib = P.group_attention_backward(cache, go[..., lo:hi, :], g, pat)
        dq[..., lo:hi, :] += gq
        for target, idxs, gk, gv in contrib:
            t0, t1 = span[target]
            dk[..., t0:t1, :] += gk
            dv[..., t0:t1, :] += gv
    for tag, got in (("dq", dq), ("dk", dk), ("dv", dv)):
        want = G[f"attn_{tag}_{idx}"]
        if want.shape != got.shape:
            got = got @ cases.grad_projection(idx, d)
        close(got, want, 1e-4)


@pytest.mark.parametrize("pad", ["exclude", "zero-logit"])
def test_attend_segments_backward_api_vs_oracle(P, pad):
    from oracle import sparsecross_oracle as O

    rng = np.random.default_rng(8)
    s, d = 19, 16
    q = rng.standard_normal((2, s, d))
    k1, v1 = rng.standard_normal((2, s, d)), rng.standard_normal((2, s, d))
    k2, v2 = rng.standard_normal((2, 5, d)), rng.standard_normal((2, 5, d))
    extra = np.zeros((s, 7), bool)
    extra[3, 2] = extra[10, 5] = True
    segs = [(k2, v2, math.inf, None), (k1, v1, 3, extra)]
    out, cache = P.attend_segments(q, segs, 4.0, pad, want_cache=True)
    close(out, O.attend_segments(q, segs, 4.0, pad), 1e-5)
    go = rng.standard_normal(out.shape)
    gq, kv = P.attend_segments_backward(cache, go)
    oq, okv = O.attend_segments_backward(q, segs, 4.0, go, pad)
    close(gq, oq, 1e-4)
    for (a, b), (c, e) in zip(kv, okv):
        close(a, c, 1e-4)
        close(b, e, 1e-4)
    probs = [rng.random((4, 6)), rng.random((4, 3))]
    gps = [rng.standard_normal((4, 6)), rng.standard_normal((4, 3))]
    dot = sum((p * g).sum(-1, keepdims=True) for p, g in zip(probs, gps))
    for got, p, g in zip(P.masked_segment_softmax_backward(probs, gps), probs, gps):
        close(got, p * (g - dot), 1e-6)


@pytest.mark.parametrize("name", ["full", "sparse", "qds"])
def test_layer_forward_backward_compose_reference_backward(P, G, name):
    """CrossEncoder.backward (R/encoder.py:511-533) restated with layer_forward / layer_backward:
    the weight gradients equal the reference's."""
    from paper_2312_17649_b200 import encoder as E

    pad = "exclude"
    cfg = P.EncoderConfig(**cases.TINY, pattern=name, padding=pad, precision="f64")
    wt = P.init_weights(cfg, 15)
    seqs = [P.assemble_input(*cases.tiny_sequence(16 + j, 4, 13, cfg.vocab_size), cfg.max_positions) for j in range(2)]
    ids = np.stack([sq.ids for sq in seqs])
    part = seqs[0].partition
    pat = P.resolve_pattern(cfg, part)
    x = wt["tok_emb"][ids] + wt["pos_emb"][:ids.shape[1]]
    caches = []
    for i in range(cfg.layers):
        x, c = E.layer_forward(x, part, pat, wt, i, cfg, want_cache=True)
        caches.append(c)
    gs = cases.TRAIN_GRAD_SCORES
    grads = {"head_w": gs @ x[:, 0, :], "head_b": gs.sum()}
    dx = np.zeros_like(x)
    dx[:, 0, :] = gs[:, None] * wt["head_w"]
    for i in reversed(range(cfg.layers)):
        dx = E.layer_backward(dx, caches[i], part, pat, wt, i, cfg, grads)
    d_tok = np.zeros_like(wt["tok_emb"])
    np.add.at(d_tok, ids.reshape(-1), dx.reshape(-1, dx.shape[-1]))
    grads["tok_emb"] = d_tok
    d_pos = np.zeros_like(wt["pos_emb"])
    d_pos[:ids.shape[1]] = dx.sum(0)
    grads["pos_emb"] = d_pos
    key = f"grad_{name}_{pad}"
    for wn in grads:
        close(grads[wn], G[f"{key}|{wn}"], 1e-4)


def test_band_matrix_api(P):
    """BandMatrix / band_qk / band_pv / their adjoints / band_to_dense (R/band.py:55-366)."""
    rng = np.random.default_rng(12)
    s, t, h, w = 7, 9, 4, 2
    q = torch.tensor(rng.standard_normal((s, h)), dtype=torch.float32, device="cuda")
    k = torch.tensor(rng.standard_normal((t, h)), dtype=torch.float32, device="cuda")
    v = torch.tensor(rng.standard_normal((t, h)), dtype=torch.float32, device="cuda")
    band = P.band_qk(q, k, w)
    assert isinstance(band, P.BandMatrix) and band.target_len == t and band.seq_len == s
    dense = P.band_to_dense(band)
    off = np.arange(t)[None, :] - np.arange(s)[:, None]
    want = np.where(np.abs(off) <= w, (q @ k.T).cpu().numpy(), 0.0)
    close(dense.cpu().numpy(), want, 1e-5)
    back = P.BandMatrix.from_dense(dense, w)
    assert torch.equal(back.data, band.data)
    out = P.band_pv(band, v)
    close(out.cpu().numpy(), (dense @ v).cpu().numpy(), 1e-5)
    gp, gv = P.band_pv_backward(out, band, v)
    assert isinstance(gp, P.BandMatrix)
    gq, gk = P.band_qk_backward(band, q, k, w)
    close(gq.cpu().numpy(), (dense @ k).cpu().numpy(), 1e-5)
    close(gk.cpu().numpy(), (dense.T @ q).cpu().numpy(), 1e-5)
    with pytest.raises(P.BandShapeError):
        P.BandMatrix(torch.ones(s, 2 * w + 1, device="cuda"), w, t)  # nonzero invalid slots
    with pytest.raises(P.BandShapeError):
        P.band_pv(band, torch.zeros(t + 1, h, device="cuda"))


def _concat_softmax(blocks, valids, scale):
    """numpy joint softmax over concatenated segments (the reference tests' concatenation oracle)."""
    ys = [np.where(ok, b / scale, -np.inf) if ok is not None else b / scale for b, ok in zip(blocks, valids)]
    cat = np.concatenate(ys, axis=1)
    e = np.exp(cat - cat.max(axis=1, keepdims=True))
    e /= e.sum(axis=1, keepdims=True)
    return np.split(e, np.cumsum([y.shape[1] for y in ys])[:-1], axis=1)


def _random_band(P, rng, s, w, t):
    ok = P.band_validity(s, w, t).cpu().numpy()
    data = np.where(ok, rng.standard_normal((s, 2 * w + 1)), 0.0)
    return P.BandMatrix(torch.tensor(data, device="cuda"), w, t), data, ok


class TestSegmentSoftmax:
    """segment_softmax / SegmentScores (R/attention.py:164-225), float64 on the device."""

    def test_uniform(self, P):
        probs = P.segment_softmax([np.zeros((4, 2)), np.zeros((4, 3))], scale=2.0)
        for seg in probs.segments:
            np.testing.assert_allclose(seg, np.full(seg.shape, 0.2))

    def test_matches_concatenation(self, P):
        rng = np.random.default_rng(0)
        band, data, ok = _random_band(P, rng, 6, 1, 6)
        dense = rng.standard_normal((6, 4))
        res = P.segment_softmax([dense, band], 2.0)
        want_d, want_b = _concat_softmax([dense, data], [None, ok], 2.0)
        np.testing.assert_allclose(res.segments[0], want_d, atol=1e-14)
        got = res.segments[1]
        assert isinstance(got, P.BandMatrix)
        gd = got.data.cpu().numpy()
        np.testing.assert_allclose(gd[ok], want_b[ok], atol=1e-14)
        assert not gd[~ok].any()

    def test_rows_sum_to_one_and_zero_logit(self, P):
        rng = np.random.default_rng(1)
        band, data, ok = _random_band(P, rng, 8, 2, 8)
        dense = rng.standard_normal((8, 3))
        res = P.segment_softmax([band, dense], scale=1.7)
        total = res.segments[0].data.cpu().numpy().sum(axis=1) + res.segments[1].sum(axis=1)
        np.testing.assert_allclose(total, 1.0, atol=1e-12)
        zl = P.segment_softmax([band, dense], scale=1.7, padding="zero-logit")
        ys = [np.where(ok, data / 1.7, 0.0), dense / 1.7]
        want = _concat_softmax(ys, [None, None], 1.0)
        np.testing.assert_allclose(zl.segments[0].data.cpu().numpy(), np.where(ok, want[0], 0.0), atol=1e-14)
        np.testing.assert_allclose(zl.segments[1], want[1], atol=1e-14)

    def test_rejects_zero_valid_row(self, P):
        band = P.BandMatrix(torch.zeros(6, 1, dtype=torch.float64, device="cuda"), 0, 3)
        with pytest.raises(P.AttentionError):
            P.segment_softmax([band], scale=1.0)


class TestBenchHarnessGpu:
    """benchmark.measure / run_bench on the device (R/bench.py:234-310)."""

    @staticmethod
    def spec(P, **kw):
        d = dict(pattern="sparse", window=4, query_len=10, doc_lens=(16,), batch_size=2, repetitions=3,
                 warmup=1, precision="f32", seed=0)
        d.update(kw)
        return P.BenchSpec(**d)

    def test_record_fields_and_determinism(self, P):
        s = self.spec(P)
        cfg = P.default_model_config(s)
        model = P.CrossEncoder(cfg, seed=0)
        batch = P.gen_random_batch(s, 16, cfg)
        r1, r2 = P.measure(model, batch, s), P.measure(model, batch, s)
        assert r1.flops == r2.flops and r1.peak_bytes == r2.peak_bytes
        assert r1.time_per_doc > 0 and r1.peak_bytes >= model.weight_nbytes and not r1.oom
        assert r1.attn_score_bytes == 0

    def test_oom_recorded_not_raised(self, P):
        s = self.spec(P)
        cfg = P.default_model_config(s)
        model = P.CrossEncoder(cfg, seed=0)
        r = P.measure(model, P.gen_random_batch(s, 16, cfg), s, mem_limit_bytes=model.weight_nbytes + 1)
        assert r.oom and r.time_per_doc is None and r.peak_bytes is None and r.flops > 0

    def test_run_bench_and_report(self, P):
        recs = P.run_bench(self.spec(P, doc_lens=(16, 164), precision="bf16"))
        assert [r.doc_len for r in recs] == [16, 164]
        assert len(P.emit_report(recs, "csv").strip().split("\n")) == 3


def test_dense_band_oracle_and_masked(P):
    """dense_band_oracle (cuBLAS) vs band_to_dense(band_qk, MASKED) (R/band.py:344-386)."""
    rng = np.random.default_rng(3)
    q, k = rng.standard_normal((11, 5)), rng.standard_normal((9, 5))
    want = P.dense_band_oracle(q, k, 3)
    got = P.band_to_dense(P.band_qk(q, k, 3), fill=P.MASKED)
    assert isinstance(got, np.ma.MaskedArray)
    np.testing.assert_array_equal(got.mask, want.mask)
    np.testing.assert_allclose(got.compressed(), want.compressed(), atol=1e-5)  # f64 in -> fp32 band kernel
    with pytest.raises(P.BandShapeError):
        P.dense_band_oracle(q, rng.standard_normal((9, 4)), 3)
