"""GPU fine-tuning of the sparse cross-encoder (R/training.py, R/encoder.py:374-533).

SURVEY §8(f)-4: the reference's backward path -- band adjoints
(R/band.py:239-274), the segment/group attention adjoints (R/attention.py:
260-269, :348-378, :476-507), ``layer_backward`` / ``CrossEncoder.backward``
(R/encoder.py:374-443, :511-533) -- and its toy trainer (AdamW, margin-MSE /
RankNet, the synthetic term-overlap task, ``train_toy``, ``grad_check``),
rebuilt on the device:

* attention forward = ``sc_attn_fwd`` (the inference kernels), attention
  backward = ``sc_attn_bwd`` (query-major dQ + key-major dK/dV kernels over
  the transposed pattern: every pattern, window, padding mode and the QDS
  globals, deterministic) behind a ``torch.autograd.Function``;
* the dense layers: GEMMs on cuBLAS (``Linear``: bf16 or fp32 with TF32 off,
  weight gradients accumulated in fp32, bias gradients by ``sc_colsum``),
  residual add + post-LN LayerNorm (eps 1e-12) by ``sc_layernorm_fwd`` /
  ``sc_layernorm_bwd``, exact-erf GELU by ``sc_gelu_fwd`` / ``sc_gelu_bwd``
  (the latter also reducing the W1 bias gradient), embeddings and the [CLS]
  head by torch ops and autograd;
* AdamW keeps the reference's update exactly (decoupled decay on every
  tensor, bias correction, linear warmup then linear decay).

Gradients come back keyed like the reference's ``grads`` dict
(``L{i}.wq`` ... ``head_b``, ``tok_emb``, ``pos_emb``) with the reference's
shapes ((in, out) weight matrices).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.nn.functional as F

from . import _lib
from .attention import AttentionError, attend_packed, make_pattern
from .encoder import (
    LAYER_NORM_EPS,
    CrossEncoder,
    EncoderConfig,
    EncoderError,
    NonFiniteActivationError,
    PackedBatch,
    _fp32_gemms,
    assemble_input,
    init_weights,
)
from .layout import PackedLayout, to_device
from .tokenizer import NUM_SPECIAL_TOKENS


class TrainingError(ValueError):
    """Bad trainer arguments (R/training.py:22-23)."""


class TrainingDivergedError(RuntimeError):
    """A non-finite loss; ``step`` is the 1-based step index (R/training.py:26-29)."""

    def __init__(self, step: int):
        super().__init__(f"loss became non-finite at step {step}")
        self.step = step


# ---------------------------------------------------------------------------
# Attention with a device adjoint.
# ---------------------------------------------------------------------------

class PatternAttention(torch.autograd.Function):
    """out = attention(qkv) under a pattern; backward through ``sc_attn_bwd``.

    qkv: contiguous [T, 3*H*d] (the fused projection), fp32 or bf16.
    Returns out [T, H*d] of the same dtype.  The adjoint writes dq, dk and dv
    in fp32 into one [T, 3*H*d] buffer (deterministic, no atomics).
    """

    @staticmethod
    def forward(ctx, qkv, layout: PackedLayout, pattern, heads: int, scale: float, padding: str,
                check: bool = True):
        hd = qkv.shape[1] // 3
        out = attend_packed(qkv[:, :hd], qkv[:, hd:2 * hd], qkv[:, 2 * hd:], layout, pattern, heads, scale,
                            padding, check=check)
        ctx.save_for_backward(qkv, out)
        ctx.meta = (layout, pattern, heads, scale, padding)
        return out

    @staticmethod
    def backward(ctx, dout):
        qkv, out = ctx.saved_tensors
        layout, pattern, heads, scale, padding = ctx.meta
        dout = dout.to(qkv.dtype).contiguous()
        T, hd3 = qkv.shape
        g = torch.empty((T, hd3), dtype=qkv.dtype, device=qkv.device)  # written in the input dtype
        attention_backward(qkv, out, dout, g, layout, pattern, heads, scale, padding)
        return g, None, None, None, None, None, None


def attention_backward(qkv: torch.Tensor, out: torch.Tensor, dout: torch.Tensor, grad: torch.Tensor,
                       layout: PackedLayout, pattern, heads: int, scale: float, padding: str) -> None:
    """Writes grad[:, :hd] = dQ, grad[:, hd:2hd] = dK, grad[:, 2hd:] = dV ([T, 3*H*d], fp32 or bf16)."""
    T, hd3 = qkv.shape
    hd = hd3 // 3
    d = hd // heads
    es = qkv.element_size()
    qds = pattern.name == "qds" and layout.tok_flags is not None
    base, gbase = qkv.data_ptr(), grad.data_ptr()
    ges = grad.element_size()
    ws_bytes = _lib.load().sc_attn_bwd_workspace_bytes(T, heads, layout.nseq, layout.max_qgroup_len)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=qkv.device)
    _lib.call(
        "sc_attn_bwd",
        base, base + hd * es, base + 2 * hd * es, qkv.stride(0), out.data_ptr(), out.stride(0),
        dout.data_ptr(), dout.stride(0), gbase, gbase + hd * ges, gbase + 2 * hd * ges, grad.stride(0),
        _dcode(grad),
        layout.cu_seqlens.data_ptr(), layout.qgroup_len.data_ptr(), layout.nseq, T, heads, d,
        pattern.links().ctypes.data, _lib.PAD_EXCLUDE if padding == "exclude" else _lib.PAD_ZERO_LOGIT,
        float(scale), _lib.DTYPE_BF16 if qkv.dtype == torch.bfloat16 else _lib.DTYPE_F32,
        _lib.ptr(layout.tok_flags) if qds else None, _lib.ptr(layout.glob_cu) if qds else None,
        _lib.ptr(layout.glob_pos) if qds else None, layout.seq_tile_base.data_ptr(), layout.tile_rows,
        layout.max_qgroup_len, layout.n_tiles, ws.data_ptr(), ws_bytes, _lib.stream_handle(),
        exc=AttentionError,
    )


# ---------------------------------------------------------------------------
# Dense-layer blocks with device adjoints.
# ---------------------------------------------------------------------------

def _dcode(t: torch.Tensor) -> int:
    return _lib.DTYPE_BF16 if t.dtype == torch.bfloat16 else _lib.DTYPE_F32


class ResidualLayerNorm(torch.autograd.Function):
    """y = LN(a + b) (fp32 out) with sc_layernorm_fwd / sc_layernorm_bwd (R/encoder.py:267-285).

    a, b: [rows, cols] contiguous fp32 or bf16 (b may be None).  With ``want16`` it also returns
    a bf16 copy of y for the next GEMM; the backward sums the gradients of both outputs inside
    the kernel and recomputes xhat from a + b and the saved per-row mean / rstd.
    """

    @staticmethod
    def forward(ctx, a, b, gamma, beta, want16=False):
        rows, cols = a.shape
        y = torch.empty(rows, cols, dtype=torch.float32, device=a.device)
        y16 = torch.empty(rows, cols, dtype=torch.bfloat16, device=a.device) if want16 else None
        mean = torch.empty(rows, dtype=torch.float32, device=a.device)
        rstd = torch.empty_like(mean)
        _lib.call("sc_layernorm_fwd", a.data_ptr(), _dcode(a), _lib.ptr(b), 0 if b is None else _dcode(b),
                  gamma.data_ptr(), beta.data_ptr(), y.data_ptr(), _lib.ptr(y16), mean.data_ptr(), rstd.data_ptr(),
                  rows, cols, float(LAYER_NORM_EPS), _lib.stream_handle(), exc=EncoderError)
        ctx.save_for_backward(a, b, gamma, mean, rstd)
        ctx.set_materialize_grads(False)
        if want16:
            return y, y16
        return y

    @staticmethod
    def backward(ctx, dy, dy16=None):
        a, b, gamma, mean, rstd = ctx.saved_tensors
        rows, cols = a.shape
        dy = torch.zeros(rows, cols, dtype=torch.float32, device=a.device) if dy is None else dy.float().contiguous()
        dy16 = None if dy16 is None else dy16.to(torch.bfloat16).contiguous()
        # the kernel writes the input gradient in fp32 and/or bf16, as the inputs' dtypes need
        dtypes = {a.dtype} | ({b.dtype} if b is not None else set())
        dx = torch.empty(rows, cols, dtype=torch.float32, device=a.device) if torch.float32 in dtypes else None
        dx16 = torch.empty(rows, cols, dtype=torch.bfloat16, device=a.device) if torch.bfloat16 in dtypes else None
        dg = torch.empty(cols, dtype=torch.float32, device=a.device)
        db = torch.empty_like(dg)
        parts = torch.empty(2 * _lib.load().sc_ln_partials(rows) * cols, dtype=torch.float32, device=a.device)
        _lib.call("sc_layernorm_bwd", dy.data_ptr(), _lib.ptr(dy16), a.data_ptr(), _dcode(a), _lib.ptr(b),
                  0 if b is None else _dcode(b), gamma.data_ptr(), mean.data_ptr(), rstd.data_ptr(), _lib.ptr(dx),
                  _lib.ptr(dx16), dg.data_ptr(), db.data_ptr(), parts.data_ptr(), rows, cols, _lib.stream_handle(),
                  exc=EncoderError)
        pick = lambda t: dx if t.dtype == torch.float32 else dx16  # noqa: E731
        return pick(a), (None if b is None else pick(b)), dg, db, None


def residual_layer_norm(a, b, gamma, beta, want16=False):
    """LN(a + b) -> y, or (y, bf16 copy of y) with want16."""
    if a.shape[1] > 1024 or a.shape[1] % 4:  # outside the kernel's envelope: torch's LayerNorm on the device
        y = F.layer_norm(a.float() + (0 if b is None else b.float()), (a.shape[1],), gamma, beta, LAYER_NORM_EPS)
        return (y, y.to(torch.bfloat16)) if want16 else y
    return ResidualLayerNorm.apply(a.contiguous(), None if b is None else b.contiguous(), gamma, beta, want16)


def column_sum(x: torch.Tensor) -> torch.Tensor:
    """fp32 column sums of a [rows, cols] matrix (sc_colsum, deterministic)."""
    rows, cols = x.shape
    out = torch.empty(cols, dtype=torch.float32, device=x.device)
    parts = torch.empty(_lib.load().sc_ln_partials(rows) * cols, dtype=torch.float32, device=x.device)
    _lib.call("sc_colsum", x.data_ptr(), _dcode(x), x.stride(0), rows, cols, out.data_ptr(), parts.data_ptr(),
              _lib.stream_handle(), exc=EncoderError)
    return out


class Linear(torch.autograd.Function):
    """out = x @ w + bias in compute dtype `cdt` (w in the reference's (in, out) layout, fp32 master).

    ``w16`` / ``b16``: optional compute-dtype copies of w / bias (the optimizer's bf16 shadow), so
    the forward does not cast the weights.  Backward: dX = dY w^T and dW = x^T dY on cuBLAS (dW
    accumulated and returned in fp32), the bias gradient by sc_colsum.
    """

    @staticmethod
    def forward(ctx, x, w, w16, bias, b16, cdt):
        xc = x.to(cdt).contiguous()
        wc = w16 if w16 is not None else w.to(cdt)
        out = torch.addmm(b16 if b16 is not None else bias.to(cdt), xc, wc)
        ctx.save_for_backward(xc, wc)
        ctx.meta = (cdt, x.dtype)
        return out

    @staticmethod
    def backward(ctx, go):
        xc, wc = ctx.saved_tensors
        cdt, xdt = ctx.meta
        go = go.to(cdt).contiguous()
        if cdt == torch.float32:
            dx, dw = torch.mm(go, wc.t()), torch.mm(xc.t(), go)
        else:  # fp32 outputs straight from the bf16 GEMMs (no cast passes)
            dx = torch.mm(go, wc.t(), out_dtype=torch.float32) if xdt == torch.float32 else torch.mm(go, wc.t())
            dw = torch.mm(xc.t(), go, out_dtype=torch.float32)
        return dx.to(xdt), dw, None, column_sum(go), None, None


class LinearQKV(torch.autograd.Function):
    """Linear over the column-concatenated [wq | wk | wv] (R/encoder.py:325-327) from the compute-dtype
    concatenation ``w16`` / ``b16`` only: the fp32 masters are never concatenated (a strided copy per
    layer per step); their gradients come back as column views of one dW GEMM."""

    @staticmethod
    def forward(ctx, x, wq, wk, wv, bq, bk, bv, w16, b16, cdt):
        xc = x.to(cdt).contiguous()
        out = torch.addmm(b16, xc, w16)
        ctx.save_for_backward(xc, w16)
        ctx.meta = (cdt, x.dtype, wq.shape[1], wk.shape[1])
        return out

    @staticmethod
    def backward(ctx, go):
        xc, wc = ctx.saved_tensors
        cdt, xdt, nq, nk = ctx.meta
        go = go.to(cdt).contiguous()
        dx = torch.mm(go, wc.t(), out_dtype=torch.float32) if xdt == torch.float32 else torch.mm(go, wc.t())
        dw = torch.mm(xc.t(), go, out_dtype=torch.float32)
        db = column_sum(go)
        a, b = nq, nq + nk
        return (dx.to(xdt), dw[:, :a], dw[:, a:b], dw[:, b:], db[:a], db[a:b], db[b:], None, None, None)


class LinearGelu(torch.autograd.Function):
    """gelu(x @ w + bias) (R/encoder.py:350-351) with sc_gelu_fwd / sc_gelu_bwd; the backward's
    GELU kernel also reduces the bias gradient (no second pass over dF)."""

    @staticmethod
    def forward(ctx, x, w, w16, bias, b16, cdt):
        xc = x.to(cdt).contiguous()
        wc = w16 if w16 is not None else w.to(cdt)
        rows, k = xc.shape
        n = wc.shape[1]
        if cdt == torch.bfloat16 and n % 256 == 0 and k % 64 == 0:
            # one tcgen05 GEMM writing gelu(x W + b) and the pre-activation (sc_gemm_bias_gelu_pre)
            f = torch.empty(rows, n, dtype=cdt, device=xc.device)
            g = torch.empty_like(f)
            wt = wc.t().contiguous()  # [N, K] (nn.Linear layout)
            _lib.call("sc_gemm_bias_gelu_pre", xc.data_ptr(), k, wt.data_ptr(), k, bias.float().contiguous().data_ptr(),
                      g.data_ptr(), n, f.data_ptr(), n, rows, n, k, _lib.stream_handle(), exc=EncoderError)
        else:
            f = torch.addmm(b16 if b16 is not None else bias.to(cdt), xc, wc)
            g = torch.empty_like(f)
            _lib.call("sc_gelu_fwd", f.data_ptr(), g.data_ptr(), _dcode(f), f.numel(), _lib.stream_handle(),
                      exc=EncoderError)
        ctx.save_for_backward(xc, wc, f)
        ctx.meta = (cdt, x.dtype)
        return g

    @staticmethod
    def backward(ctx, dg):
        xc, wc, f = ctx.saved_tensors
        cdt, xdt = ctx.meta
        rows, cols = f.shape
        dg = dg.to(cdt).contiguous()
        df = torch.empty_like(f)
        db = torch.empty(cols, dtype=torch.float32, device=f.device)
        parts = torch.empty(_lib.load().sc_ln_partials(rows) * cols, dtype=torch.float32, device=f.device)
        _lib.call("sc_gelu_bwd", f.data_ptr(), dg.data_ptr(), df.data_ptr(), _dcode(f), rows, cols, db.data_ptr(),
                  parts.data_ptr(), _lib.stream_handle(), exc=EncoderError)
        if cdt == torch.float32:
            dx, dw = torch.mm(df, wc.t()), torch.mm(xc.t(), df)
        else:
            dx = torch.mm(df, wc.t(), out_dtype=torch.float32) if xdt == torch.float32 else torch.mm(df, wc.t())
            dw = torch.mm(xc.t(), df, out_dtype=torch.float32)
        return dx.to(xdt), dw, None, db, None, None


def _gelu_ok(cols: int) -> bool:
    return cols % 8 == 0


# ---------------------------------------------------------------------------
# Trainable encoder.
# ---------------------------------------------------------------------------

class ParamDict(dict):
    """Reference-named parameters that are views of one flat fp32 device buffer (``flat``),
    so the optimizer updates every tensor with one fused kernel (sc_adamw_step)."""

    def __init__(self, items, flat: torch.Tensor, order, shadow: torch.Tensor | None = None):
        super().__init__(items)
        self.flat = flat
        self.order = list(order)
        self.shadow = shadow          # optional bf16 copy of `flat`, kept current by the fused AdamW
        self.shadow_version = -1      # flat._version the shadow was last synced at
        self.shadow_views = {}
        if shadow is not None:
            off = 0
            for n in self.order:
                k = items[n].numel()
                self.shadow_views[n] = shadow[off:off + k].view(items[n].shape)
                off += k

    def bf16_views(self) -> dict:
        """bf16 views of the weights, re-synced if the fp32 weights were modified in place."""
        if self.shadow is None:
            return None
        if self.shadow_version != self.flat._version:
            with torch.no_grad():
                self.shadow.copy_(self.flat)
            self.shadow_version = self.flat._version
        return self.shadow_views


def _layer_block(x, xh, W, S, p, layout, pattern, H, scale, cfg, check_keys):
    """One post-LN layer (R/encoder.py:306-371) on the device, differentiable: returns (x, the GEMM
    input copy of x).  W: fp32 parameters by reference name; S: their bf16 shadows or None."""
    bf16 = cfg.precision == "bf16"
    cd = torch.bfloat16 if bf16 else torch.float32

    def lin(xin, wname, bname):
        return Linear.apply(xin, W[wname], None if S is None else S[wname], W[bname],
                            None if S is None else S[bname], cd)

    if S is not None and cd == torch.bfloat16:
        w16 = torch.cat([S[p + "wq"], S[p + "wk"], S[p + "wv"]], dim=1)
        b16 = torch.cat([S[p + "bq"], S[p + "bk"], S[p + "bv"]])
        qkv = LinearQKV.apply(xh, W[p + "wq"], W[p + "wk"], W[p + "wv"], W[p + "bq"], W[p + "bk"], W[p + "bv"],
                              w16, b16, cd)
    else:
        wqkv = torch.cat([W[p + "wq"], W[p + "wk"], W[p + "wv"]], dim=1)
        bqkv = torch.cat([W[p + "bq"], W[p + "bk"], W[p + "bv"]])
        w16 = None if S is None else torch.cat([S[p + "wq"], S[p + "wk"], S[p + "wv"]], dim=1)
        b16 = None if S is None else torch.cat([S[p + "bq"], S[p + "bk"], S[p + "bv"]])
        qkv = Linear.apply(xh, wqkv, w16, bqkv, b16, cd)
    o = PatternAttention.apply(qkv, layout, pattern, H, scale, cfg.padding, check_keys)
    if bf16:
        ln1, ln1h = residual_layer_norm(x, lin(o, p + "wo", p + "bo"), W[p + "ln1_g"], W[p + "ln1_b"], want16=True)
    else:
        ln1 = ln1h = residual_layer_norm(x, lin(o, p + "wo", p + "bo"), W[p + "ln1_g"], W[p + "ln1_b"])
    if _gelu_ok(cfg.ff_dim):
        g1 = LinearGelu.apply(ln1h, W[p + "w1"], None if S is None else S[p + "w1"], W[p + "b1"],
                              None if S is None else S[p + "b1"], cd)
    else:
        g1 = F.gelu(lin(ln1h, p + "w1", p + "b1"))
    if bf16:
        return residual_layer_norm(ln1, lin(g1, p + "w2", p + "b2"), W[p + "ln2_g"], W[p + "ln2_b"], want16=True)
    x = residual_layer_norm(ln1, lin(g1, p + "w2", p + "b2"), W[p + "ln2_g"], W[p + "ln2_b"])
    return x, x


class GradDict(dict):
    """Gradients that are views of one flat fp32 buffer in ParamDict order (``flat``)."""

    def __init__(self, flat: torch.Tensor):
        super().__init__()
        self.flat = flat


class TrainableCrossEncoder:
    """Reference-named fp32 device parameters with a differentiable packed forward.

    Mirrors ``CrossEncoder`` of R/encoder.py:450-538 for training:
    ``score(ids, partition, want_cache=True)`` -> (scores, cache) and
    ``backward(cache, grad_scores)`` -> grads dict.  ``weights`` holds
    leaf tensors with ``requires_grad``; AdamW updates them in place.
    """

    def __init__(self, config: EncoderConfig, weights: dict | None = None, seed: int = 0, device="cuda"):
        self.config = config
        self.device = torch.device(device)
        host = init_weights(config, seed) if weights is None else weights
        order = sorted(host)
        arrs = [np.asarray(host[n], dtype=np.float32) for n in order]
        flat = torch.empty(sum(a.size for a in arrs), dtype=torch.float32, device=self.device)
        views, off = {}, 0
        for n, a in zip(order, arrs):
            v = flat[off:off + a.size].view(a.shape)
            v.copy_(torch.from_numpy(a.copy()))
            views[n] = v.requires_grad_(True)
            off += a.size
        shadow = torch.empty(flat.numel(), dtype=torch.bfloat16, device=self.device) \
            if config.precision == "bf16" else None
        self.weights = ParamDict(views, flat, order, shadow)
        self.pattern = make_pattern(config.pattern, config.window)

    @property
    def host_weights(self) -> dict:
        """numpy copies in the config's storage dtype (save_model / the inference CrossEncoder)."""
        dt = np.float64 if self.config.precision == "f64" else np.float32
        return {n: t.detach().cpu().numpy().astype(dt) for n, t in self.weights.items()}

    @property
    def weight_nbytes(self) -> int:
        return sum(int(t.numel() * t.element_size()) for t in self.weights.values())

    def to_inference(self, **kw) -> CrossEncoder:
        """The inference engine (fused kernels, graphs) over the current weights."""
        return CrossEncoder(self.config, self.host_weights, device=self.device, **kw)

    def gemm_mode(self):
        """fp32 configs: full-precision cuBLAS (TF32 off) for the forward and the adjoint GEMMs."""
        return _fp32_gemms(self.config.precision != "bf16")

    def make_layout(self, batch: PackedBatch) -> PackedLayout:
        qds = self.config.qds_global_every if self.config.pattern == "qds" else 0
        return PackedLayout.from_lengths(batch.seq_lens, batch.qgroup_lens, device=self.device, qds_every=qds)

    # -- differentiable packed forward -------------------------------------

    def hidden_packed(self, ids_dev: torch.Tensor, layout: PackedLayout, check_finite: bool = True) -> torch.Tensor:
        """Final-layer activations [T, h] with the autograd graph (R/encoder.py:475-500)."""
        cfg, W = self.config, self.weights
        H = cfg.heads
        bf16 = cfg.precision == "bf16"
        scale = math.sqrt(cfg.head_dim)
        x = W["tok_emb"][ids_dev.long()] + W["pos_emb"][layout.tok_pos.long()]
        S = W.bf16_views() if (bf16 and isinstance(W, ParamDict)) else None

        flags = []
        xh = x  # GEMM input of the layer (bf16 copy of the previous LayerNorm in the bf16 path)
        with self.gemm_mode():
            for i in range(cfg.layers):
                x, xh = _layer_block(x, xh, W, S, f"L{i}.", layout, self.pattern, H, scale, cfg, i == 0)
                if check_finite:
                    flags.append(torch.isfinite(x.detach()).all())
        if flags:
            ok = torch.stack(flags).cpu()
            if not bool(ok.all()):
                raise NonFiniteActivationError(int((~ok).nonzero()[0, 0]))
        return x.float()

    def score_packed(self, ids_dev: torch.Tensor, layout: PackedLayout, check_finite: bool = True) -> torch.Tensor:
        """Scores [nseq] = x[cls] . head_w + head_b, differentiable (R/encoder.py:502-509)."""
        x = self.hidden_packed(ids_dev, layout, check_finite)
        return x[layout.cls_rows] @ self.weights["head_w"] + self.weights["head_b"]

    # -- reference-shaped entry points ---------------------------------------

    def _check_ids(self, ids, partition) -> np.ndarray:
        ids = np.asarray(ids, dtype=np.int64)
        if ids.ndim == 1:
            ids = ids[None, :]
        if ids.ndim != 2 or ids.shape[1] != partition.seq_len:
            raise EncoderError(f"ids shape {ids.shape} inconsistent with partition length {partition.seq_len}")
        if ids.shape[1] > self.config.max_positions:
            raise EncoderError("sequence longer than max_positions")
        if ids.min() < 0 or ids.max() >= self.config.vocab_size:
            raise EncoderError("token id outside vocabulary")
        return ids

    def score(self, ids, partition, want_cache: bool = False):
        """Scores (batch,) as numpy; with ``want_cache`` also the cache ``backward`` consumes."""
        ids = self._check_ids(ids, partition)
        batch = PackedBatch.from_ids(ids, partition)
        layout = self.make_layout(batch)
        ids_dev = to_device(batch.ids, self.device)
        if not want_cache:
            with torch.no_grad():
                return self.score_packed(ids_dev, layout).double().cpu().numpy()
        s = self.score_packed(ids_dev, layout)
        return s.detach().double().cpu().numpy(), {"scores": s, "layout": layout}

    def forward(self, ids, partition) -> np.ndarray:
        """Final-layer embeddings (batch, seq, embed) (R/encoder.py:475-500)."""
        ids = self._check_ids(ids, partition)
        batch = PackedBatch.from_ids(ids, partition)
        layout = self.make_layout(batch)
        with torch.no_grad():
            x = self.hidden_packed(to_device(batch.ids, self.device), layout)
        return x.double().cpu().numpy().reshape(ids.shape[0], ids.shape[1], -1)

    def backward(self, cache: dict, grad_scores) -> dict:
        """Weight gradients of sum(grad_scores * scores) (R/encoder.py:511-533), as device fp32 tensors."""
        s = cache["scores"]
        g = torch.as_tensor(np.asarray(grad_scores, dtype=np.float32) if not torch.is_tensor(grad_scores)
                            else grad_scores, device=s.device, dtype=s.dtype).reshape(s.shape)
        names = sorted(self.weights)
        with self.gemm_mode():
            grads = torch.autograd.grad(s, [self.weights[n] for n in names], grad_outputs=g, allow_unused=True)
        return {n: (torch.zeros_like(self.weights[n]) if gr is None else gr) for n, gr in zip(names, grads)}


# ---------------------------------------------------------------------------
# Losses (R/training.py:36-75).  Inputs: floats, numpy arrays or tensors.
# ---------------------------------------------------------------------------

def _f64(x):
    if torch.is_tensor(x):
        return x.detach().double()
    return torch.as_tensor(np.asarray(x, dtype=np.float64))


def margin_mse_loss(s_pos, s_neg, t_pos, t_neg) -> float:
    """mean(((s+ - s-) - (t+ - t-))^2) in float64 (R/training.py:36-41)."""
    sp, sn, tp, tn = (_f64(a) for a in (s_pos, s_neg, t_pos, t_neg))
    dev = sp.device
    gap = (sp - sn) - (tp.to(dev) - tn.to(dev))
    return float(torch.mean(gap * gap))


def margin_mse_grad(s_pos, s_neg, t_pos, t_neg):
    """(dL/ds+, dL/ds-) = (2 gap / n, -2 gap / n) (R/training.py:44-47)."""
    sp, sn, tp, tn = (_f64(a) for a in (s_pos, s_neg, t_pos, t_neg))
    dev = sp.device
    gap = (sp - sn) - (tp.to(dev) - tn.to(dev))
    scale = 2.0 / max(gap.numel(), 1)
    return _like(scale * gap, s_pos), _like(-scale * gap, s_pos)


def ranknet_loss(s_pos, s_neg) -> float:
    """mean(log(1 + exp(-(s+ - s-)))), overflow-safe (R/training.py:50-53)."""
    delta = _f64(s_pos) - _f64(s_neg).to(_f64(s_pos).device)
    return float(torch.mean(torch.logaddexp(torch.zeros_like(delta), -delta)))


def ranknet_grad(s_pos, s_neg):
    """d/ds+ = -sigmoid(-(s+ - s-)) / n (R/training.py:56-60)."""
    delta = _f64(s_pos) - _f64(s_neg).to(_f64(s_pos).device)
    g = -torch.sigmoid(-delta) / max(delta.numel(), 1)
    return _like(g, s_pos), _like(-g, s_pos)


def _like(t: torch.Tensor, ref):
    if torch.is_tensor(ref):
        return t
    out = t.cpu().numpy()
    return out if out.ndim else float(out)


LOSSES = ("margin_mse", "ranknet")


# ---------------------------------------------------------------------------
# Optimizer (R/training.py:79-137) on device tensors.
# ---------------------------------------------------------------------------

class AdamW:
    """Adam moments, bias correction, decoupled decay, linear warmup / decay.

    ``step(weights, grads)`` applies, for every name in sorted order,
    ``w -= lr_t * ((m/bc1) / (sqrt(v/bc2) + eps) + weight_decay * w)``.
    Device parameters from ``TrainableCrossEncoder`` (a ``ParamDict`` over one
    flat buffer) take one fused kernel per step (``sc_adamw_step``: fp64
    arithmetic, fp32 moments).  ``moment_dtype=torch.float64`` keeps the
    reference's float64 moments exactly (per-tensor torch ops).
    """

    def __init__(self, lr: float, betas=(0.9, 0.999), eps: float = 1e-8, weight_decay: float = 0.01,
                 warmup_steps: int = 0, total_steps: int | None = None, moment_dtype=torch.float32):
        self.lr = lr
        self.beta1, self.beta2 = betas
        self.eps = eps
        self.weight_decay = weight_decay
        self.warmup_steps = warmup_steps
        self.total_steps = total_steps
        self.step_count = 0
        self.moment_dtype = moment_dtype
        self._m: dict = {}
        self._v: dict = {}

    def current_lr(self) -> float:
        t = self.step_count
        if self.warmup_steps > 0 and t <= self.warmup_steps:
            return self.lr * t / self.warmup_steps
        if self.total_steps is not None and self.total_steps > self.warmup_steps:
            frac = (t - self.warmup_steps) / (self.total_steps - self.warmup_steps)
            return self.lr * max(0.0, 1.0 - min(1.0, frac))
        return self.lr

    @torch.no_grad()
    def step(self, weights: dict, grads: dict) -> None:
        self.step_count += 1
        t = self.step_count
        lr_t = self.current_lr()
        if isinstance(weights, ParamDict) and weights.flat.is_cuda and self.moment_dtype == torch.float32:
            self._fused_step(weights, grads, lr_t, t)
            return
        bc1 = 1.0 - self.beta1 ** t
        bc2 = 1.0 - self.beta2 ** t
        for name in sorted(weights):
            w = weights[name]
            g = grads[name]
            g = (g if torch.is_tensor(g) else torch.as_tensor(np.asarray(g))).to(w.device, self.moment_dtype)
            m = self._m.get(name)
            if m is None:
                m = self._m[name] = torch.zeros_like(g)
                self._v[name] = torch.zeros_like(g)
            v = self._v[name]
            m.mul_(self.beta1).add_(g, alpha=1.0 - self.beta1)
            v.mul_(self.beta2).addcmul_(g, g, value=1.0 - self.beta2)
            update = (m / bc1) / ((v / bc2).sqrt() + self.eps)
            w.sub_((lr_t * (update + self.weight_decay * w.to(self.moment_dtype))).to(w.dtype))


    def _fused_step(self, weights: ParamDict, grads: dict, lr_t: float, t: int) -> None:
        flat = weights.flat
        gf = getattr(grads, "flat", None)
        if gf is not None and gf.numel() == flat.numel() and gf.dtype == torch.float32:
            g = gf
        else:
            g = torch.cat([torch.as_tensor(grads[n], device=flat.device).reshape(-1).float() for n in weights.order])
        if self._m.get("__flat__") is None:
            self._m["__flat__"] = torch.zeros_like(flat)
            self._v["__flat__"] = torch.zeros_like(flat)
        shadow = weights.shadow if weights.shadow_version == flat._version else None
        _lib.call("sc_adamw_step", flat.data_ptr(), g.data_ptr(), self._m["__flat__"].data_ptr(),
                  self._v["__flat__"].data_ptr(), _lib.ptr(shadow), flat.numel(), float(lr_t), float(self.beta1), float(self.beta2),
                  float(self.eps), float(self.weight_decay), int(t), _lib.stream_handle(), exc=TrainingError)


# ---------------------------------------------------------------------------
# Synthetic term-overlap task (R/training.py:140-227): host-side sampling with
# the reference's random draws, so a seed yields the reference's triples.
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Triple:
    query: tuple
    positive: tuple
    negative: tuple
    teacher_pos: float | None = None
    teacher_neg: float | None = None

    def __post_init__(self):
        if tuple(self.positive) == tuple(self.negative):
            raise TrainingError("positive and negative documents must differ")
        if (self.teacher_pos is None) != (self.teacher_neg is None):
            raise TrainingError("teacher scores must be present for both documents or neither")


@dataclass(frozen=True)
class ValidationQuery:
    query_id: str
    query: tuple
    candidates: list
    relevance: dict


@dataclass(frozen=True)
class SyntheticTask:
    """Queries of distinct vocabulary terms; positives hold all of them, negatives none."""

    vocab_words: int = 64
    query_terms: int = 4
    doc_len: int = 16

    def __post_init__(self):
        if self.query_terms < 1 or self.doc_len < self.query_terms:
            raise TrainingError("doc_len must be >= query_terms >= 1")
        if self.vocab_words < 2 * self.query_terms:
            raise TrainingError("vocabulary too small for disjoint distractors")

    @property
    def vocab_size(self) -> int:
        return NUM_SPECIAL_TOKENS + self.vocab_words

    def overlap(self, query, doc) -> int:
        return len(set(query) & set(doc))

    def _draw_query(self, rng) -> tuple:
        words = np.arange(NUM_SPECIAL_TOKENS, self.vocab_size)
        return tuple(int(t) for t in rng.choice(words, size=self.query_terms, replace=False))

    def _draw_doc(self, rng, query, count: int) -> tuple:
        # draw order: the `count` query terms, the filler, then one shuffle
        q = np.asarray(query)
        picked = rng.choice(q, size=count, replace=False) if count else np.empty(0, int)
        pool = np.setdiff1d(np.arange(NUM_SPECIAL_TOKENS, self.vocab_size), q)
        filler = rng.choice(pool, size=self.doc_len - count, replace=True)
        doc = np.concatenate([picked, filler])
        rng.shuffle(doc)
        return tuple(int(t) for t in doc)

    def sample_triple(self, rng) -> Triple:
        query = self._draw_query(rng)
        pos = self._draw_doc(rng, query, self.query_terms)
        neg = self._draw_doc(rng, query, 0)
        return Triple(query, pos, neg, teacher_pos=float(self.query_terms), teacher_neg=0.0)

    def sample_validation(self, rng, n_queries: int, per_level: int = 4) -> list:
        pools = []
        for qi in range(n_queries):
            query = self._draw_query(rng)
            cands, rel = [], {}
            for level in range(self.query_terms + 1):
                for _ in range(per_level):
                    did = f"d{len(cands)}"
                    cands.append((did, self._draw_doc(rng, query, level)))
                    rel[did] = level
            perm = rng.permutation(len(cands))
            pools.append(ValidationQuery(f"q{qi}", query, [cands[j] for j in perm], rel))
        return pools


def validation_ndcg(model, val_set, k: int = 10):
    """(per-query nDCG@k, mean); pools ranked by (-score, position) (R/training.py:230-255)."""
    from .rerank import RunEntry, ndcg_at_k

    run, qrels = [], {}
    for vq in val_set:
        seqs = [assemble_input(vq.query, doc, model.config.max_positions) for _, doc in vq.candidates]
        scores = model.score(np.stack([s.ids for s in seqs]), seqs[0].partition)
        order = sorted(range(len(seqs)), key=lambda j: (-float(scores[j]), j))
        for rank, j in enumerate(order, 1):
            run.append(RunEntry(vq.query_id, vq.candidates[j][0], rank, float(scores[j])))
        qrels[vq.query_id] = dict(vq.relevance)
    return ndcg_at_k(run, qrels, k)


# ---------------------------------------------------------------------------
# Training loop (R/training.py:258-357).
# ---------------------------------------------------------------------------

@dataclass
class TraceRow:
    step: int
    loss: float
    ndcg10: float | None = None


@dataclass
class TrainResult:
    model: TrainableCrossEncoder
    trace: list = field(default_factory=list)

    @property
    def final_ndcg(self):
        for row in reversed(self.trace):
            if row.ndcg10 is not None:
                return row.ndcg10
        return None


def _batch_arrays(triples, max_positions):
    """[positives; negatives] ids (2B, s) and their shared partition (R/training.py:277-284)."""
    seqs = [assemble_input(t.query, t.positive, max_positions) for t in triples]
    seqs += [assemble_input(t.query, t.negative, max_positions) for t in triples]
    if len({s.ids.shape[0] for s in seqs}) != 1:
        raise TrainingError("triples in one batch must share sequence length")
    return np.stack([s.ids for s in seqs]), seqs[0].partition


def _loss_tensor(name, scores, triples):
    b = len(triples)
    sp, sn = scores[:b].double(), scores[b:].double()
    if name == "margin_mse":
        if any(t.teacher_pos is None for t in triples):
            raise TrainingError("margin_mse requires teacher scores on every triple")
        tgap = torch.tensor([t.teacher_pos - t.teacher_neg for t in triples], dtype=torch.float64,
                            device=scores.device)
        gap = (sp - sn) - tgap
        return torch.mean(gap * gap)
    delta = sp - sn
    return torch.mean(torch.logaddexp(torch.zeros_like(delta), -delta))


def train_step(model: TrainableCrossEncoder, opt: AdamW, triples, loss: str = "margin_mse",
               step: int | None = None, process_group=None) -> float:
    """One optimisation step on a batch of triples; returns the loss value.  Under
    torch.distributed with ``process_group`` (or the default group) set up, each rank passes its
    own triples and the gradients are averaged before the update (data parallel)."""
    ids, partition = _batch_arrays(triples, model.config.max_positions)
    ids = model._check_ids(ids, partition)
    batch = PackedBatch.from_ids(ids, partition)
    layout = model.make_layout(batch)
    scores = model.score_packed(to_device(batch.ids, model.device), layout)
    lt = _loss_tensor(loss, scores, triples)
    value = float(lt.detach())
    if not math.isfinite(value):
        raise TrainingDivergedError(opt.step_count + 1 if step is None else step)
    names = sorted(model.weights)
    with model.gemm_mode():
        gr = torch.autograd.grad(lt, [model.weights[n] for n in names], allow_unused=True)
    grads = {n: (torch.zeros_like(model.weights[n]) if g is None else g) for n, g in zip(names, gr)}
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(process_group) > 1:
        grads = flat_gradients(model, grads)
        allreduce_gradients(grads, process_group)
    opt.step(model.weights, grads)
    return value


def allreduce_gradients(grads, group=None) -> None:
    """Data-parallel fine-tuning: average the gradients over the ranks of `group`, in place.

    One collective on the flat fp32 buffer when the gradients are a ``GradDict`` (NCCL over
    NVLink on the GPU; any torch.distributed backend works), else one per tensor.  Every rank
    then applies the same AdamW update to identical weights.
    """
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return
    world = dist.get_world_size(group)
    if world == 1:
        return
    flat = getattr(grads, "flat", None)
    tensors = [flat] if flat is not None else [g for g in grads.values() if torch.is_tensor(g)]
    for t in tensors:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        t.div_(world)


def flat_gradients(model: "TrainableCrossEncoder", grads_by_name: dict) -> "GradDict":
    """Copy per-tensor gradients into one flat fp32 buffer in ParamDict order."""
    names = sorted(model.weights)
    flat = torch.cat([grads_by_name[n].reshape(-1).float() for n in names])
    out, off = GradDict(flat), 0
    for n in names:
        k = model.weights[n].numel()
        out[n] = flat[off:off + k].view(model.weights[n].shape)
        off += k
    return out


class GraphedTrainStep:
    """One fine-tuning step (forward, loss, backward) captured as a CUDA graph for a fixed batch
    shape, plus the fused AdamW update outside the graph (its step-dependent scalars change).

    The packed layout, the static id / teacher buffers and every intermediate live in the
    graph's memory pool; each call copies new ids (and teacher margins) in, replays, and
    applies AdamW.  Margin-MSE or RankNet loss, as in ``train_step``.  The replayed forward
    reads the bf16 shadow weights the fused AdamW keeps current: change the weights only
    through this object's optimizer (or call ``model.weights.bf16_views()`` after an in-place
    edit, before the next call).
    """

    def __init__(self, model: TrainableCrossEncoder, opt: AdamW, batch: PackedBatch, loss: str = "margin_mse",
                 warmup: int = 2, process_group=None):
        if loss not in LOSSES:
            raise TrainingError(f"unknown loss {loss!r}; expected one of {LOSSES}")
        if batch.nseq % 2:
            raise TrainingError("a training batch holds positives then negatives (even nseq)")
        self.model, self.opt, self.loss = model, opt, loss
        self.process_group = process_group  # data parallel: gradients averaged over its ranks
        self.layout = model.make_layout(batch)
        self.ids = to_device(batch.ids, model.device)
        self.teacher_gap = torch.zeros(batch.nseq // 2, dtype=torch.float64, device=model.device)
        self.names = sorted(model.weights)
        W = model.weights
        if isinstance(W, ParamDict):
            W.bf16_views()  # sync the shadow before capture
        side = torch.cuda.Stream(device=model.device)
        side.wait_stream(torch.cuda.current_stream(model.device))
        with torch.cuda.stream(side):
            for _ in range(warmup):
                self._fwd_bwd()
        torch.cuda.current_stream(model.device).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.loss_value, self.grad_flat = self._fwd_bwd()

    def _fwd_bwd(self):
        m = self.model
        s = m.score_packed(self.ids, self.layout, check_finite=False)
        b = s.shape[0] // 2
        delta = s[:b].double() - s[b:].double()
        if self.loss == "margin_mse":
            gap = delta - self.teacher_gap
            lt = torch.mean(gap * gap)
        else:
            lt = torch.mean(torch.logaddexp(torch.zeros_like(delta), -delta))
        with m.gemm_mode():
            gr = torch.autograd.grad(lt, [m.weights[n] for n in self.names], allow_unused=True)
        flat = torch.cat([(torch.zeros_like(m.weights[n]) if g is None else g).reshape(-1).float()
                          for n, g in zip(self.names, gr)])
        return lt.detach(), flat

    def __call__(self, ids, teacher_gap=None) -> torch.Tensor:
        """One step on new ids of the captured shape; returns the loss (device scalar, float64)."""
        src = torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int32)) if isinstance(ids, np.ndarray) else ids
        if tuple(src.shape) != tuple(self.ids.shape):
            raise EncoderError(f"ids shape {tuple(src.shape)} does not match the captured layout "
                               f"{tuple(self.ids.shape)}")
        if src.numel():  # sc_embed reads tok_emb[id] unchecked: the reference's _check_ids range rule
            lo, hi = int(src.min()), int(src.max())
            if lo < 0 or hi >= self.model.config.vocab_size:
                raise EncoderError("token id outside vocabulary")
        self.ids.copy_(src, non_blocking=True)
        if teacher_gap is not None:
            self.teacher_gap.copy_(torch.as_tensor(teacher_gap, dtype=torch.float64), non_blocking=True)
        self.graph.replay()
        if not math.isfinite(float(self.loss_value)):  # as train_step: never feed NaN gradients to AdamW
            raise TrainingDivergedError(self.opt.step_count + 1)
        W = self.model.weights
        grads, off = GradDict(self.grad_flat), 0
        for n in self.names:  # == ParamDict.order (sorted names)
            k = W[n].numel()
            grads[n] = self.grad_flat[off:off + k].view(W[n].shape)
            off += k
        allreduce_gradients(grads, self.process_group)
        self.opt.step(W, grads)
        return self.loss_value


def train_toy(config: EncoderConfig, dataset, steps: int, lr: float, seed: int = 0, batch_pairs: int = 16,
              loss: str = "margin_mse", weight_decay: float = 0.01, warmup_fraction: float = 0.01,
              lr_decay: bool = True, eval_every: int = 0, val_set=None, val_k: int = 10,
              device="cuda") -> TrainResult:
    """Train a fresh model on triples (R/training.py:287-357), on the GPU.

    ``dataset``: a SyntheticTask (sampled afresh each step with the
    reference's RNG stream) or a fixed sequence of triples cycled in order.
    """
    if loss not in LOSSES:
        raise TrainingError(f"unknown loss {loss!r}; expected one of {LOSSES}")
    synthetic = isinstance(dataset, SyntheticTask)
    if synthetic and config.vocab_size < dataset.vocab_size:
        raise TrainingError("encoder vocabulary smaller than task vocabulary")
    if not synthetic and not dataset:
        raise TrainingError("fixed dataset must be nonempty")
    model = TrainableCrossEncoder(config, seed=seed, device=device)
    opt = AdamW(lr, weight_decay=weight_decay, warmup_steps=max(1, round(warmup_fraction * steps)),
                total_steps=steps if lr_decay else None)
    rng = np.random.default_rng(seed + 0x5EED)
    result = TrainResult(model)
    cursor = 0
    for step in range(1, steps + 1):
        if synthetic:
            triples = [dataset.sample_triple(rng) for _ in range(batch_pairs)]
        else:
            triples = [dataset[(cursor + i) % len(dataset)] for i in range(batch_pairs)]
            cursor += batch_pairs
        value = train_step(model, opt, triples, loss, step)
        row = TraceRow(step, value)
        if val_set is not None and (step == steps or (eval_every > 0 and step % eval_every == 0)):
            row.ndcg10 = validation_ndcg(model, val_set, val_k)[1]
        result.trace.append(row)
    return result


def write_trace_csv(trace, path) -> None:
    """step,loss,ndcg10 (R/training.py:360-365)."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("step,loss,ndcg10\n")
        for row in trace:
            nd = "" if row.ndcg10 is None else f"{row.ndcg10:.6f}"
            fh.write(f"{row.step},{row.loss:.8f},{nd}\n")


def grad_check(model: TrainableCrossEncoder, triples, eps: float = 1e-3, samples: int = 8,
               loss: str = "margin_mse", seed: int = 0) -> float:
    """Max relative error of directional derivatives: analytic <grad, u> vs central differences.

    The reference (R/training.py:372-433) perturbs single float64
    coordinates; the device path computes in fp32, where a single-coordinate
    difference drowns in rounding, so this checks ``samples`` random
    Rademacher directions spanning every weight tensor instead.
    """
    triples = list(triples)
    ids, partition = _batch_arrays(triples, model.config.max_positions)
    batch = PackedBatch.from_ids(model._check_ids(ids, partition), partition)
    layout = model.make_layout(batch)
    ids_dev = to_device(batch.ids, model.device)
    names = sorted(model.weights)

    def loss_value():
        with torch.no_grad():
            return float(_loss_tensor(loss, model.score_packed(ids_dev, layout), triples))

    lt = _loss_tensor(loss, model.score_packed(ids_dev, layout), triples)
    with model.gemm_mode():
        grads = torch.autograd.grad(lt, [model.weights[n] for n in names], allow_unused=True)
    gen = torch.Generator(device=model.device).manual_seed(seed)
    worst = 0.0
    for _ in range(samples):
        dirs = [torch.randint(0, 2, model.weights[n].shape, generator=gen, device=model.device).float() * 2 - 1
                for n in names]
        analytic = sum(float((g * u).sum()) for g, u in zip(grads, dirs) if g is not None)
        orig = [model.weights[n].detach().clone() for n in names]
        with torch.no_grad():
            for n, w0, u in zip(names, orig, dirs):
                model.weights[n].copy_(w0 + eps * u)
        up = loss_value()
        with torch.no_grad():
            for n, w0, u in zip(names, orig, dirs):
                model.weights[n].copy_(w0 - eps * u)
        down = loss_value()
        with torch.no_grad():
            for n, w0 in zip(names, orig):
                model.weights[n].copy_(w0)
        fd = (up - down) / (2 * eps)
        denom = max(abs(analytic), abs(fd))
        err = abs(analytic - fd) if denom < 1e-6 else abs(analytic - fd) / denom
        worst = max(worst, err)
    return worst


# ---------------------------------------------------------------------------
# Reference-shaped layer primitives (R/encoder.py:250-443) on the device; numpy in -> numpy out.
# ---------------------------------------------------------------------------

def _dev(a):
    if torch.is_tensor(a):
        return a, False, None
    arr = np.asarray(a)
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).cuda(), True, arr.dtype


def _back(t, was_np, dt):
    return t.detach().cpu().numpy().astype(dt, copy=False) if was_np else t


def _padded_flat(t, mult):
    n = t.numel()
    buf = torch.zeros(((n + mult - 1) // mult) * mult, dtype=torch.float32, device=t.device)
    buf[:n] = t.reshape(-1).float()
    return buf, n


def gelu(x):
    """Exact-erf GELU (R/encoder.py:258-259) by sc_gelu_fwd."""
    t, was_np, dt = _dev(x)
    buf, n = _padded_flat(t, 1024)
    out = torch.empty_like(buf)
    _lib.call("sc_gelu_fwd", buf.data_ptr(), out.data_ptr(), _lib.DTYPE_F32, buf.numel(), _lib.stream_handle(),
              exc=EncoderError)
    return _back(out[:n].reshape(t.shape), was_np, dt)


def gelu_grad(x):
    """d gelu / dx = Phi(x) + x phi(x) (R/encoder.py:262-264) by sc_gelu_bwd with a unit upstream."""
    t, was_np, dt = _dev(x)
    buf, n = _padded_flat(t, 1024)
    ones = torch.ones_like(buf)
    out = torch.empty_like(buf)
    _lib.call("sc_gelu_bwd", buf.data_ptr(), ones.data_ptr(), out.data_ptr(), _lib.DTYPE_F32, buf.numel() // 1024,
              1024, None, None, _lib.stream_handle(), exc=EncoderError)
    return _back(out[:n].reshape(t.shape), was_np, dt)


def layer_norm(x, gain, bias):
    """(gain * xhat + bias, (xhat, inv)) with eps 1e-12 (R/encoder.py:267-273), by sc_layernorm_fwd."""
    t, was_np, dt = _dev(x)
    g, b = _dev(gain)[0].float().contiguous(), _dev(bias)[0].float().contiguous()
    h = t.shape[-1]
    x2 = t.reshape(-1, h).float().contiguous()
    rows = x2.shape[0]
    y = torch.empty_like(x2)
    mean = torch.empty(rows, dtype=torch.float32, device=x2.device)
    rstd = torch.empty_like(mean)
    if h % 4 == 0 and h <= 1024:
        _lib.call("sc_layernorm_fwd", x2.data_ptr(), _lib.DTYPE_F32, None, 0, g.data_ptr(), b.data_ptr(), y.data_ptr(),
                  None, mean.data_ptr(), rstd.data_ptr(), rows, h, float(LAYER_NORM_EPS), _lib.stream_handle(),
                  exc=EncoderError)
    else:
        mean = x2.mean(dim=-1)
        rstd = torch.rsqrt(((x2 - mean[:, None]) ** 2).mean(dim=-1) + LAYER_NORM_EPS)
        y = (x2 - mean[:, None]) * rstd[:, None] * g + b
    xhat = ((x2 - mean[:, None]) * rstd[:, None]).reshape(t.shape)
    inv = rstd.reshape(*t.shape[:-1], 1)
    return _back(y.reshape(t.shape), was_np, dt), (_back(xhat, was_np, dt), _back(inv, was_np, dt))


def layer_norm_backward(grad_y, cache, gain):
    """(dx, dgain, dbias) of layer_norm (R/encoder.py:276-285), by sc_layernorm_bwd on xhat."""
    gy, was_np, dt = _dev(grad_y)
    xhat, inv = (_dev(c)[0].float() for c in cache)
    g = _dev(gain)[0].float().contiguous()
    h = gy.shape[-1]
    dy = gy.reshape(-1, h).float().contiguous()
    xh = xhat.reshape(-1, h).contiguous()
    rows = dy.shape[0]
    if h % 4 == 0 and h <= 1024:
        zeros = torch.zeros(rows, dtype=torch.float32, device=dy.device)
        ones = torch.ones_like(zeros)
        dxh = torch.empty_like(dy)
        dg = torch.empty(h, dtype=torch.float32, device=dy.device)
        db = torch.empty_like(dg)
        parts = torch.empty(2 * _lib.load().sc_ln_partials(rows) * h, dtype=torch.float32, device=dy.device)
        # with mean 0 and rstd 1 the kernel's xhat is xhat itself; dx = inv * (g dy - m1 - xhat m2)
        _lib.call("sc_layernorm_bwd", dy.data_ptr(), None, xh.data_ptr(), _lib.DTYPE_F32, None, 0, g.data_ptr(),
                  zeros.data_ptr(), ones.data_ptr(), dxh.data_ptr(), None, dg.data_ptr(), db.data_ptr(),
                  parts.data_ptr(), rows, h, _lib.stream_handle(), exc=EncoderError)
        dx = dxh.reshape(gy.shape) * inv
    else:
        gd = dy * g
        m1 = gd.mean(dim=-1, keepdim=True)
        m2 = (gd * xh).mean(dim=-1, keepdim=True)
        dx = ((gd - m1 - xh * m2)).reshape(gy.shape) * inv
        dg, db = (dy * xh).sum(0), dy.sum(0)
    return _back(dx, was_np, dt), _back(dg, was_np, dt), _back(db, was_np, dt)


def weight_nbytes(weights: dict) -> int:
    return sum(int(np.asarray(w).nbytes) if not torch.is_tensor(w) else w.numel() * w.element_size()
               for w in weights.values())


_LAYER_KEYS = ("wq", "bq", "wk", "bk", "wv", "bv", "wo", "bo", "ln1_g", "ln1_b", "w1", "b1", "w2", "b2",
               "ln2_g", "ln2_b")


def layer_forward(x, partition, pattern, weights, layer_index, config, want_cache=False):
    """One post-LN layer over a (batch, seq, embed) activation (R/encoder.py:306-371) on the device:
    fused attention kernels, cuBLAS GEMMs, LayerNorm / GELU kernels.  With ``want_cache`` it also
    returns the cache ``layer_backward`` consumes (the device autograd graph)."""
    xt, was_np, dt = _dev(x)
    b, s, h = xt.shape
    p = f"L{layer_index}."
    W = {p + k: _dev(weights[p + k])[0].float().contiguous().detach().requires_grad_(want_cache) for k in _LAYER_KEYS}
    globals_ = getattr(pattern, "global_positions", ())
    layout = PackedLayout.from_lengths([s] * b, [partition.group_len("query")] * b, device="cuda",
                                       qds_positions=[globals_] * b if globals_ else None)
    x2 = xt.reshape(b * s, h).float().contiguous().detach().requires_grad_(want_cache)
    with torch.set_grad_enabled(want_cache), _fp32_gemms(config.precision != "bf16"):
        out, _ = _layer_block(x2, x2, W, None, p, layout, pattern, config.heads, math.sqrt(config.head_dim), config,
                              True)
    if not bool(torch.isfinite(out.detach()).all()):
        raise NonFiniteActivationError(layer_index)
    res = _back(out.float().reshape(b, s, h), was_np, dt)
    if not want_cache:
        return res
    return res, {"x": x2, "out": out, "W": W, "shape": (b, s, h), "was_np": was_np, "dtype": dt}


def layer_backward(grad_out, cache, partition, pattern, weights, layer_index, config, grads):
    """Adjoint of layer_forward (R/encoder.py:374-443): returns d_x and accumulates the layer's weight
    gradients into ``grads`` by reference name (through the device adjoints of the layer blocks)."""
    g = _dev(grad_out)[0].float().reshape(cache["out"].shape)
    names = list(cache["W"])
    with _fp32_gemms(config.precision != "bf16"):
        res = torch.autograd.grad(cache["out"], [cache["x"]] + [cache["W"][n] for n in names], grad_outputs=g,
                                  allow_unused=True)
    for n, gr in zip(names, res[1:]):
        val = torch.zeros_like(cache["W"][n]) if gr is None else gr
        val = _back(val, cache["was_np"], cache["dtype"]) if cache["was_np"] else val
        grads[n] = grads.get(n, 0) + val
    dx = res[0].reshape(cache["shape"])
    return _back(dx, cache["was_np"], cache["dtype"])
