"""Band-matrix kernels ⊡_w / ⊙_w on device (R/band.py).

Band storage is (rows, 2w+1): slot j of row i addresses target row i+j-w and
is valid iff 0 <= i+j-w < target_len (R/band.py:48-52).  These wrap the
standalone ``sc_band_scores`` / ``sc_band_apply`` kernels; the encoder never
materialises bands (the fused attention kernels fold them into the softmax).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


class BandShapeError(ValueError):
    """Band/dense operands have inconsistent shapes (R/band.py:31-32)."""


def _check_window(window) -> int:
    if not isinstance(window, (int, np.integer)) or window < 0:
        raise BandShapeError(f"window must be a non-negative integer, got {window!r}")
    return int(window)


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return _lib.DTYPE_F32
    if t.dtype == torch.bfloat16:
        return _lib.DTYPE_BF16
    raise BandShapeError(f"unsupported dtype {t.dtype}")


def band_validity(seq_len: int, window: int, target_len: int, device="cuda") -> torch.Tensor:
    """Bool (seq_len, 2w+1) validity mask computed on device (R/band.py:48-52)."""
    w = _check_window(window)
    out = torch.empty((seq_len, 2 * w + 1), dtype=torch.uint8, device=device)
    _lib.call("sc_band_validity", seq_len, w, target_len, out.data_ptr(), _lib.stream_handle(),
              exc=BandShapeError)
    return out.bool()


def _flatten(a: torch.Tensor, b: torch.Tensor):
    lead = torch.broadcast_shapes(a.shape[:-2], b.shape[:-2])
    a = a.expand(*lead, *a.shape[-2:]).reshape(-1, *a.shape[-2:]).contiguous()
    b = b.expand(*lead, *b.shape[-2:]).reshape(-1, *b.shape[-2:]).contiguous()
    return lead, a, b


def band_scores(q: torch.Tensor, k: torch.Tensor, window: int) -> torch.Tensor:
    """out[..., i, j] = q[..., i, :] . k[..., i+j-w, :]; 0 out of range (R/band.py:154-177)."""
    w = _check_window(window)
    if q.shape[-1] != k.shape[-1]:
        raise BandShapeError(f"feature dims differ: q has {q.shape[-1]}, k has {k.shape[-1]}")
    if q.dtype != k.dtype:
        raise BandShapeError("q and k dtypes differ")
    lead, qf, kf = _flatten(q, k)
    B, s, d = qf.shape
    t = kf.shape[1]
    out = torch.empty((B, s, 2 * w + 1), dtype=q.dtype, device=q.device)
    _lib.call("sc_band_scores", qf.data_ptr(), kf.data_ptr(), out.data_ptr(), B, s, t, d, w, _dt(qf),
              _lib.stream_handle(), exc=BandShapeError)
    return out.reshape(*lead, s, 2 * w + 1)


def band_apply(p: torch.Tensor, v: torch.Tensor, window: int) -> torch.Tensor:
    """out[..., i, :] = sum_j p[..., i, j] v[..., i+j-w, :]; invalid slots ignored (R/band.py:197-218)."""
    w = _check_window(window)
    if p.shape[-1] != 2 * w + 1:
        raise BandShapeError(f"band width {p.shape[-1]} inconsistent with window {w}")
    if p.dtype != v.dtype:
        raise BandShapeError("p and v dtypes differ")
    lead, pf, vf = _flatten(p, v)
    B, s, _ = pf.shape
    t, d = vf.shape[1], vf.shape[2]
    out = torch.empty((B, s, d), dtype=v.dtype, device=v.device)
    _lib.call("sc_band_apply", pf.data_ptr(), vf.data_ptr(), out.data_ptr(), B, s, t, d, w, _dt(pf),
              _lib.stream_handle(), exc=BandShapeError)
    return out.reshape(*lead, s, d)


def band_qk(q: torch.Tensor, k: torch.Tensor, window: int) -> torch.Tensor:
    """2-D windowed query-key product (R/band.py:290-303); returns the (s, 2w+1) band data."""
    if q.dim() != 2 or k.dim() != 2:
        raise BandShapeError("Q and K must be 2-D")
    return band_scores(q, k, window)


def band_pv(p: torch.Tensor, v: torch.Tensor, window: int) -> torch.Tensor:
    """2-D band-probability-value product (R/band.py:306-313)."""
    if p.dim() != 2 or v.dim() != 2:
        raise BandShapeError("P and V must be 2-D")
    return band_apply(p, v, window)


def band_scores_backward(grad_band: torch.Tensor, q: torch.Tensor, k: torch.Tensor, window: int):
    """Adjoint of band_scores (R/band.py:239-253): (grad_q, grad_k); invalid slots never read."""
    w = _check_window(window)
    if grad_band.shape[-1] != 2 * w + 1 or grad_band.shape[-2] != q.shape[-2]:
        raise BandShapeError("gradient band inconsistent with forward shapes")
    if not (grad_band.dtype == q.dtype == k.dtype):
        raise BandShapeError("gradient, q and k dtypes differ")
    lead = torch.broadcast_shapes(grad_band.shape[:-2], q.shape[:-2], k.shape[:-2])
    g = grad_band.expand(*lead, *grad_band.shape[-2:]).reshape(-1, *grad_band.shape[-2:]).contiguous()
    qf = q.expand(*lead, *q.shape[-2:]).reshape(-1, *q.shape[-2:]).contiguous()
    kf = k.expand(*lead, *k.shape[-2:]).reshape(-1, *k.shape[-2:]).contiguous()
    B, s, d = qf.shape
    t = kf.shape[1]
    gq, gk = torch.empty_like(qf), torch.empty_like(kf)
    _lib.call("sc_band_scores_backward", g.data_ptr(), qf.data_ptr(), kf.data_ptr(), gq.data_ptr(), gk.data_ptr(),
              B, s, t, d, w, _dt(qf), _lib.stream_handle(), exc=BandShapeError)
    return gq.reshape(*lead, s, d), gk.reshape(*lead, t, d)


def band_apply_backward(grad_out: torch.Tensor, p: torch.Tensor, v: torch.Tensor, window: int):
    """Adjoint of band_apply (R/band.py:256-274): (grad_p, grad_v); grad_p is 0 at invalid slots."""
    w = _check_window(window)
    if p.shape[-1] != 2 * w + 1:
        raise BandShapeError(f"band width {p.shape[-1]} inconsistent with window {w}")
    if grad_out.shape[-2] != p.shape[-2] or grad_out.shape[-1] != v.shape[-1]:
        raise BandShapeError("grad_out shape inconsistent with forward output")
    if not (grad_out.dtype == p.dtype == v.dtype):
        raise BandShapeError("gradient, p and v dtypes differ")
    lead = torch.broadcast_shapes(grad_out.shape[:-2], p.shape[:-2], v.shape[:-2])
    go = grad_out.expand(*lead, *grad_out.shape[-2:]).reshape(-1, *grad_out.shape[-2:]).contiguous()
    pf = p.expand(*lead, *p.shape[-2:]).reshape(-1, *p.shape[-2:]).contiguous()
    vf = v.expand(*lead, *v.shape[-2:]).reshape(-1, *v.shape[-2:]).contiguous()
    B, s, _ = pf.shape
    t, d = vf.shape[1], vf.shape[2]
    gp, gv = torch.empty_like(pf), torch.empty_like(vf)
    _lib.call("sc_band_apply_backward", go.data_ptr(), pf.data_ptr(), vf.data_ptr(), gp.data_ptr(), gv.data_ptr(),
              B, s, t, d, w, _dt(pf), _lib.stream_handle(), exc=BandShapeError)
    return gp.reshape(*lead, s, 2 * w + 1), gv.reshape(*lead, t, d)


def band_qk_backward(grad_band: torch.Tensor, q: torch.Tensor, k: torch.Tensor, window: int):
    """2-D adjoint of band_qk (R/band.py:316-328)."""
    if q.dim() != 2 or k.dim() != 2 or grad_band.dim() != 2:
        raise BandShapeError("gradient band, Q and K must be 2-D")
    return band_scores_backward(grad_band, q, k, window)


def band_pv_backward(grad_out: torch.Tensor, p: torch.Tensor, v: torch.Tensor, window: int):
    """2-D adjoint of band_pv (R/band.py:331-341)."""
    if grad_out.dim() != 2 or p.dim() != 2 or v.dim() != 2:
        raise BandShapeError("grad_out, P and V must be 2-D")
    return band_apply_backward(grad_out, p, v, window)


class _BandScoresFn(torch.autograd.Function):
    """band_scores with its adjoint on the device (sc_band_scores_backward)."""

    @staticmethod
    def forward(ctx, q, k, window):
        ctx.save_for_backward(q, k)
        ctx.window = window
        return band_scores(q, k, window)

    @staticmethod
    def backward(ctx, g):
        q, k = ctx.saved_tensors
        gq, gk = band_scores_backward(g.contiguous().to(q.dtype), q, k, ctx.window)
        return gq, gk, None


class _BandApplyFn(torch.autograd.Function):
    """band_apply with its adjoint on the device (sc_band_apply_backward)."""

    @staticmethod
    def forward(ctx, p, v, window):
        ctx.save_for_backward(p, v)
        ctx.window = window
        return band_apply(p, v, window)

    @staticmethod
    def backward(ctx, g):
        p, v = ctx.saved_tensors
        gp, gv = band_apply_backward(g.contiguous().to(p.dtype), p, v, ctx.window)
        return gp, gv, None


def band_scores_ad(q: torch.Tensor, k: torch.Tensor, window: int) -> torch.Tensor:
    """Differentiable band_scores (autograd through the device adjoint kernels)."""
    return _BandScoresFn.apply(q, k, window)


def band_apply_ad(p: torch.Tensor, v: torch.Tensor, window: int) -> torch.Tensor:
    """Differentiable band_apply (autograd through the device adjoint kernels)."""
    return _BandApplyFn.apply(p, v, window)
