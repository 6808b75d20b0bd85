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


def _as_tensor(x) -> torch.Tensor:
    return x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _kernel_operand(x) -> torch.Tensor:
    """Device operand for the band kernels: float64 (the reference's numpy default) computes in fp32."""
    t = _as_tensor(x)
    return t.float() if t.dtype == torch.float64 else t


class BandMatrix:
    """Band storage on the device (R/band.py:55-114): ``data`` (seq_len, 2w+1), invalid slots exactly 0,
    ``target_len`` = rows of the attended-to matrix."""

    def __init__(self, data, window: int, target_len: int):
        self.window = _check_window(window)
        self.data = _as_tensor(data)
        if self.data.dim() != 2 or self.data.shape[1] != 2 * self.window + 1:
            raise BandShapeError(f"band data must be (s, {2 * self.window + 1}), got {tuple(self.data.shape)}")
        self.target_len = int(target_len)
        if self.target_len < 1:
            raise BandShapeError("target_len must be >= 1")
        if not bool(torch.isfinite(self.data).all()):
            raise BandShapeError("band data contains non-finite entries")
        if bool((self.data[~self.valid] != 0).any()):
            raise BandShapeError("entries at invalid band positions must be exactly 0")

    @property
    def seq_len(self) -> int:
        return self.data.shape[0]

    @property
    def width(self) -> int:
        return self.data.shape[1]

    @property
    def valid(self) -> torch.Tensor:
        return band_validity(self.seq_len, self.window, self.target_len, device=self.data.device)

    def to_dense(self, fill=0.0) -> torch.Tensor:
        return band_to_dense(self, fill=fill)

    @classmethod
    def from_dense(cls, dense, window: int) -> "BandMatrix":
        """The in-band entries of a dense (s, s') matrix (R/band.py:100-114)."""
        d = _as_tensor(dense)
        if d.dim() != 2:
            raise BandShapeError("dense input must be 2-D")
        w = _check_window(window)
        s, t = d.shape
        cols = torch.arange(s, device=d.device)[:, None] + torch.arange(2 * w + 1, device=d.device)[None, :] - w
        ok = (cols >= 0) & (cols < t)
        data = torch.where(ok, d.gather(1, cols.clamp(0, t - 1)), torch.zeros((), dtype=d.dtype, device=d.device))
        return cls(data, w, t)


MASKED = np.ma.masked   # band_to_dense fill marker (R/band.py:36)


def band_to_dense(band: BandMatrix, target_cols: int | None = None, fill=0.0):
    """Re-expand a band to a dense (s, target_cols) device matrix, other entries ``fill``
    (R/band.py:344-366); ``fill=MASKED`` returns a host numpy masked array instead."""
    t = band.target_len if target_cols is None else int(target_cols)
    if t < 1:
        raise BandShapeError("target_cols must be >= 1")
    s, w = band.seq_len, band.window
    dev = band.data.device
    cols = torch.arange(s, device=dev)[:, None] + torch.arange(2 * w + 1, device=dev)[None, :] - w
    ok = (cols >= 0) & (cols < t)
    masked = fill is MASKED
    dense = torch.full((s, t + 1), 0.0 if masked else float(fill), dtype=band.data.dtype, device=dev)
    dense.scatter_(1, torch.where(ok, cols, torch.full_like(cols, t)), band.data)  # invalid slots -> spare column
    if not masked:
        return dense[:, :t]
    off = torch.arange(t, device=dev)[None, :] - torch.arange(s, device=dev)[:, None]
    return np.ma.MaskedArray(dense[:, :t].cpu().numpy(), mask=(off.abs() > w).cpu().numpy())


def dense_band_oracle(q, k, window: int) -> np.ma.MaskedArray:
    """Full Q K^T (cuBLAS) with out-of-band entries masked (R/band.py:369-386): the
    independent dense check of band_qk, returned as a host masked array."""
    q, k = _as_tensor(q), _as_tensor(k)
    if q.dim() != 2 or k.dim() != 2:
        raise BandShapeError("Q and K must be 2-D")
    if q.shape[1] != k.shape[1]:
        raise BandShapeError(f"embedding dims differ: Q has {q.shape[1]}, K has {k.shape[1]}")
    w = _check_window(window)
    off = np.arange(k.shape[0])[None, :] - np.arange(q.shape[0])[:, None]
    return np.ma.MaskedArray((q @ k.T).cpu().numpy(), mask=np.abs(off) > w)


def band_qk(q, k, window: int) -> BandMatrix:
    """Windowed query-key product of (s, h) and (s', h) matrices as a BandMatrix (R/band.py:290-303)."""
    q, k = _kernel_operand(q), _kernel_operand(k)
    if q.dim() != 2 or k.dim() != 2:
        raise BandShapeError("Q and K must be 2-D")
    return BandMatrix(band_scores(q, k, window), window, k.shape[0])


def band_pv(p, v, window: int | None = None) -> torch.Tensor:
    """Band probabilities (BandMatrix, or raw band data with ``window``) times a dense (s', h) value
    matrix (R/band.py:306-313)."""
    v = _kernel_operand(v)
    if isinstance(p, BandMatrix):
        if v.dim() != 2 or v.shape[0] != p.target_len:
            raise BandShapeError(f"V has {v.shape[0]} rows but band was built against {p.target_len}")
        return band_apply(_kernel_operand(p.data), v, p.window)
    p = _kernel_operand(p)
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


def band_qk_backward(grad_band, q, k, window: int):
    """2-D adjoint of band_qk (R/band.py:316-328); grad_band a BandMatrix or raw band data."""
    q, k = _kernel_operand(q), _kernel_operand(k)
    if isinstance(grad_band, BandMatrix):
        if grad_band.window != _check_window(window) or grad_band.seq_len != q.shape[0]:
            raise BandShapeError("gradient band inconsistent with forward shapes")
        if grad_band.target_len != k.shape[0]:
            raise BandShapeError("gradient band target length inconsistent with K")
        grad_band = grad_band.data
    grad_band = _kernel_operand(grad_band)
    if q.dim() != 2 or k.dim() != 2 or grad_band.dim() != 2:
        raise BandShapeError("gradient band, Q and K must be 2-D")
    return band_scores_backward(grad_band, q, k, window)


def band_pv_backward(grad_out, p, v, window: int | None = None):
    """2-D adjoint of band_pv (R/band.py:331-341): (grad_p, grad_v); grad_p a BandMatrix when p is."""
    grad_out, v = _kernel_operand(grad_out), _kernel_operand(v)
    if isinstance(p, BandMatrix):
        if v.shape[0] != p.target_len:
            raise BandShapeError("V rows inconsistent with band target length")
        if grad_out.dim() != 2 or tuple(grad_out.shape) != (p.seq_len, v.shape[1]):
            raise BandShapeError("grad_out shape inconsistent with forward output")
        gp, gv = band_apply_backward(grad_out, _kernel_operand(p.data), v, p.window)
        return BandMatrix(gp, p.window, p.target_len), gv
    p = _kernel_operand(p)
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
