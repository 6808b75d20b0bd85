"""Attention patterns and the fused windowed cross-attention on B200.

Mirrors the reference module ``sparsecross.attention`` (R/attention.py):
the same pattern objects, names, error class and argument meaning, with the
computation done by the sm_100a kernels behind ``sc_attn_fwd``.

* ``AttentionPattern`` / ``make_pattern`` / ``*_pattern`` -- R/attention.py:55-157
* ``attend_packed``  -- NEW packed varlen entry point used by the encoder:
  all groups of all sequences of a packed batch in one kernel call.
* ``group_attention`` / ``apply_pattern`` / ``windowed_cross_attention`` /
  ``full_attention`` -- compatibility shims with the reference signatures
  (R/attention.py:276-287, :381-400, :416-473, :510-537); inputs may be torch
  CUDA tensors or numpy arrays (uploaded; returned as numpy).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .layout import PackedLayout

FULL = math.inf                                  # R/attention.py:40
GROUPS = ("cls", "query", "doc")                 # R/attention.py:42
PADDING_MODES = ("exclude", "zero-logit")        # R/attention.py:44


class AttentionError(ValueError):
    """Malformed segment tuples, rows without valid targets, or bad patterns (R/attention.py:47-48)."""


def is_full(window) -> bool:
    return window == FULL


@dataclass(frozen=True)
class AttentionPattern:
    """Per-group targets: source group -> ((target group, window), ...) (R/attention.py:55-89)."""

    name: str
    targets: dict
    global_positions: tuple = ()

    def __post_init__(self):
        for source, tlist in self.targets.items():
            if source not in GROUPS:
                raise AttentionError(f"unknown source group {source!r}")
            seen = [t for t, _ in tlist]
            if len(set(seen)) != len(seen):
                raise AttentionError(f"duplicate target group for source {source!r}")
            for target, window in tlist:
                if target not in GROUPS:
                    raise AttentionError(f"unknown target group {target!r}")
                if not is_full(window) and (int(window) != window or window < 0):
                    raise AttentionError(f"bad window {window!r} for {source}->{target}")
        if any(p < 0 for p in self.global_positions):
            raise AttentionError("global positions must be non-negative")
        if self.global_positions and self.name != "qds":
            raise AttentionError("global positions are only meaningful for the qds pattern")

    def targets_of(self, source: str):
        try:
            return self.targets[source]
        except KeyError:
            raise AttentionError(f"pattern {self.name!r} has no targets for group {source!r}")

    def links(self) -> np.ndarray:
        """int32[9] link table [src][tgt]: -2 none, -1 full, else the window (sc_attn_fwd ABI)."""
        out = np.full(9, _lib.LINK_NONE, dtype=np.int32)
        for si, src in enumerate(GROUPS):
            for tgt, w in self.targets.get(src, ()):
                out[si * 3 + GROUPS.index(tgt)] = _lib.LINK_FULL if is_full(w) else int(w)
        return out


_EVERY = (("cls", FULL), ("query", FULL), ("doc", FULL))


def full_pattern() -> AttentionPattern:
    return AttentionPattern("full", {g: _EVERY for g in GROUPS})


def longformer_pattern(window) -> AttentionPattern:
    return AttentionPattern("longformer", {"cls": _EVERY, "query": _EVERY,
                                           "doc": (("cls", FULL), ("query", FULL), ("doc", window))})


def qds_pattern(window, global_positions=()) -> AttentionPattern:
    return AttentionPattern("qds", {"cls": _EVERY, "query": _EVERY,
                                    "doc": (("cls", FULL), ("query", FULL), ("doc", window))},
                            global_positions=tuple(int(p) for p in global_positions))


def sparse_pattern(window) -> AttentionPattern:
    """Asymmetric pattern of Eqs. 1-3: query tokens attend only to query tokens."""
    return AttentionPattern("sparse", {"cls": _EVERY, "query": (("query", FULL),),
                                       "doc": (("cls", FULL), ("query", FULL), ("doc", window))})


PATTERN_FACTORIES = {
    "full": lambda window, globals_=(): full_pattern(),
    "longformer": lambda window, globals_=(): longformer_pattern(window),
    "qds": lambda window, globals_=(): qds_pattern(window, globals_),
    "sparse": lambda window, globals_=(): sparse_pattern(window),
}


def make_pattern(name: str, window, global_positions=()) -> AttentionPattern:
    try:
        factory = PATTERN_FACTORIES[name]
    except KeyError:
        raise AttentionError(f"unknown pattern {name!r}; expected one of {sorted(PATTERN_FACTORIES)}")
    return factory(window, global_positions)


# ---------------------------------------------------------------------------
# Host-side validation (no device sync): rows with zero valid keys raise like
# masked_segment_softmax does (R/attention.py:250-251).
# ---------------------------------------------------------------------------

def check_rows_have_keys(pattern: AttentionPattern, group_lens: np.ndarray, padding: str,
                         has_globals: bool = False) -> None:
    """group_lens: int array (nseq, 3).  Raises AttentionError if any row has no valid key."""
    for si, src in enumerate(GROUPS):
        tl = pattern.targets.get(src, ())
        if not tl:
            raise AttentionError(f"pattern {pattern.name!r} has no targets for group {src!r}")
        if any(is_full(w) for _, w in tl):
            continue
        if padding == "zero-logit" or (has_globals and src == "doc"):
            continue
        # Windowed only: row i has a key iff i < len_t + w for some target.
        reach = np.max(np.stack([group_lens[:, GROUPS.index(t)] + int(w) for t, w in tl]), axis=0)
        if np.any(group_lens[:, si] > reach):
            raise AttentionError("a row has zero valid entries across all segments")


# ---------------------------------------------------------------------------
# Packed varlen entry point.
# ---------------------------------------------------------------------------

def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return _lib.DTYPE_F32
    if t.dtype == torch.bfloat16:
        return _lib.DTYPE_BF16
    raise AttentionError(f"unsupported dtype {t.dtype}; expected float32 or bfloat16")


def attend_packed(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, layout: PackedLayout,
                  pattern: AttentionPattern, heads: int, scale: float | None = None,
                  padding: str = "exclude", out: torch.Tensor | None = None,
                  algo: str = "auto", check: bool = True, rows: str = "all") -> torch.Tensor:
    """Pattern attention over every row of a packed batch (all groups, all sequences).

    q/k/v: [T, >=heads*d] views sharing a row stride (e.g. the thirds of a
    packed QKV projection [T, 3*heads*d]).  Returns out [T, heads*d].
    rows="head" computes only the cls + query-group rows of every sequence
    (the other rows of ``out`` are left untouched).
    """
    if rows not in ("all", "head"):
        raise AttentionError(f"rows must be 'all' or 'head', got {rows!r}")
    if padding not in PADDING_MODES:
        raise AttentionError(f"unknown padding mode {padding!r}")
    T = layout.total_tokens
    if q.dim() != 2 or q.shape[0] != T:
        raise AttentionError(f"q must be [T={T}, heads*d], got {tuple(q.shape)}")
    hd = q.shape[1]
    if hd % heads:
        raise AttentionError("q width not divisible by heads")
    d = hd // heads
    if not (q.stride(1) == k.stride(1) == v.stride(1) == 1) or not (q.stride(0) == k.stride(0) == v.stride(0)):
        raise AttentionError("q/k/v must share a row stride with unit column stride")
    if scale is None:
        scale = math.sqrt(d)
    if scale <= 0:
        raise AttentionError(f"scale must be positive, got {scale}")
    qds = pattern.name == "qds" and layout.tok_flags is not None
    if pattern.global_positions and not qds:
        raise AttentionError("QDS globals need a layout built with qds globals")
    if check:
        check_rows_have_keys(pattern, layout.group_lens_host, padding, qds)
    dt = _dtype_code(q)
    if out is None:
        out = torch.empty((T, hd), dtype=q.dtype, device=q.device)
    algo_code = {"auto": _lib.ALGO_AUTO, "generic": _lib.ALGO_GENERIC, "band": _lib.ALGO_BAND_MMA,
                 "tc": _lib.ALGO_TC}[algo]
    if rows == "head":
        algo_code = _lib.ALGO_HEAD_ROWS
    links = pattern.links()
    ws = layout.attn_workspace(heads, d, links)
    _lib.call(
        "sc_attn_fwd",
        q.data_ptr(), k.data_ptr(), v.data_ptr(), q.stride(0), out.data_ptr(), out.stride(0),
        layout.cu_seqlens.data_ptr(), layout.qgroup_len.data_ptr(), layout.nseq, T, heads, d,
        links.ctypes.data, _lib.PAD_EXCLUDE if padding == "exclude" else _lib.PAD_ZERO_LOGIT,
        float(scale), dt, layout.tok_seq.data_ptr(), layout.seq_tile_base.data_ptr(),
        layout.seq_head_base.data_ptr(), layout.tile_rows, layout.max_qgroup_len,
        _lib.ptr(layout.tok_flags) if qds else None, _lib.ptr(layout.glob_cu) if qds else None,
        _lib.ptr(layout.glob_pos) if qds else None, algo_code,
        _lib.ptr(ws), 0 if ws is None else ws.numel(), None, _lib.stream_handle(),
        exc=AttentionError,
    )
    return out


# ---------------------------------------------------------------------------
# Reference-signature compatibility shims (one partition shared by all leading dims).
# ---------------------------------------------------------------------------

def _to_device(x):
    if isinstance(x, torch.Tensor):
        return x, False
    arr = np.asarray(x)
    return torch.from_numpy(np.ascontiguousarray(arr)).cuda(), True


def _compute_dtype(t: torch.Tensor):
    return t if t.dtype in (torch.float32, torch.bfloat16) else t.float()


def _run_groups(qkv: dict, pattern: AttentionPattern, scale: float, padding: str, store=None):
    """Pack the three groups of (Q, K, V) views, run the kernel, return per-group outputs."""
    for g in GROUPS:
        if g not in qkv:
            raise AttentionError(f"pattern references absent group {g!r}")
    mats, was_np, orig_dtype = [], False, None
    for g in GROUPS:
        trip = []
        for x in qkv[g]:
            t, from_np = _to_device(x)
            was_np |= from_np
            orig_dtype = orig_dtype or t.dtype
            trip.append(t)
        mats.append(trip)
    lead = mats[0][0].shape[:-2]
    d = mats[0][0].shape[-1]
    lens = [m[0].shape[-2] for m in mats]
    for g, m in zip(GROUPS, mats):
        for t in m:
            if t.shape[:-2] != lead or t.shape[-1] != d:
                raise AttentionError(f"incompatible shapes in group {g!r}")
        if m[1].shape[-2] != m[2].shape[-2] or m[0].shape[-2] != m[1].shape[-2]:
            raise AttentionError("key/value row counts differ")
    if lens[0] != 1:
        raise AttentionError("the cls group must have exactly one row")
    H = int(np.prod(lead)) if len(lead) else 1
    s = sum(lens)
    cat = []
    for which in range(3):
        x = torch.cat([_compute_dtype(m[which]) for m in mats], dim=-2)   # (*lead, s, d)
        x = x.reshape(H, s, d).permute(1, 0, 2).contiguous().reshape(s, H * d)
        cat.append(x)
    dtype = cat[0].dtype
    cat = [c.to(dtype) for c in cat]
    if pattern.global_positions and max(pattern.global_positions) >= lens[2]:  # R/attention.py:437-438
        raise AttentionError("global positions outside the document group")
    layout = PackedLayout.from_lengths([s], [lens[1]], device=cat[0].device,
                                       qds_positions=[pattern.global_positions] if pattern.global_positions else None)
    out = attend_packed(cat[0], cat[1], cat[2], layout, pattern, H, scale, padding)
    if store is not None:  # what group_attention_backward needs
        store.update(layout=layout, qkv=torch.cat(cat, dim=1).contiguous(), out=out, H=H, d=d, lens=lens, lead=lead,
                     was_np=was_np, np_dtype=np.dtype(str(orig_dtype).replace("torch.", "")) if was_np else None)
    out = out.reshape(s, H, d).permute(1, 0, 2).reshape(*lead, s, d) if len(lead) else out.reshape(s, d)
    outs, lo = [], 0
    for n in lens:
        o = out[..., lo:lo + n, :]
        if was_np:
            o = o.float().cpu().numpy().astype(np.dtype(str(orig_dtype).replace("torch.", "")), copy=False)
        outs.append(o)
        lo += n
    return outs


def group_attention(qkv: dict, source: str, pattern: AttentionPattern, scale: float,
                    padding: str = "exclude", want_cache: bool = False):
    """Output of one source group under a pattern (R/attention.py:416-473).  ``want_cache``
    also returns what ``group_attention_backward`` needs (the packed q/k/v and output)."""
    if source not in GROUPS:
        raise AttentionError(f"unknown source group {source!r}")
    pattern.targets_of(source)
    if not want_cache:
        return _run_groups(qkv, pattern, scale, padding)[GROUPS.index(source)]
    store = {}
    outs = _run_groups(qkv, pattern, scale, padding, store=store)
    store.update(pattern=pattern, scale=scale, padding=padding)
    return outs[GROUPS.index(source)], store


def group_attention_backward(cache, grad_out, source: str, pattern: AttentionPattern):
    """Adjoint of group_attention (R/attention.py:476-507) on the fused device kernel
    (sc_attn_bwd): (grad_q, [(target_group, None, grad_k, grad_v) for every group]).  The
    reference lists one entry per segment (plus the QDS globals by index); the per-target
    sums, which is what layer_backward accumulates, are identical."""
    from .training import attention_backward

    lay, qkv, out = cache["layout"], cache["qkv"], cache["out"]
    H, d, lens, lead = cache["H"], cache["d"], cache["lens"], cache["lead"]
    s = sum(lens)
    lo = sum(lens[:GROUPS.index(source)])
    go = _to_device(grad_out)[0].float().reshape(H, lens[GROUPS.index(source)], d)
    dout = torch.zeros(s, H, d, dtype=qkv.dtype, device=qkv.device)
    dout[lo:lo + go.shape[1]] = go.permute(1, 0, 2).to(qkv.dtype)
    g = torch.empty(s, 3 * H * d, dtype=torch.float32, device=qkv.device)
    attention_backward(qkv, out, dout.reshape(s, H * d), g, lay, cache["pattern"], H, cache["scale"],
                       cache["padding"])
    parts = g.reshape(s, 3, H, d).permute(1, 2, 0, 3)  # (3, H, s, d)

    def cut(t, a, n):
        t = t[:, a:a + n, :].reshape(*lead, n, d) if len(lead) else t[0, a:a + n, :]
        return t.cpu().numpy().astype(cache["np_dtype"], copy=False) if cache["was_np"] else t

    gq = cut(parts[0], lo, lens[GROUPS.index(source)])
    contrib, a = [], 0
    for gname, n in zip(GROUPS, lens):
        contrib.append((gname, None, cut(parts[1], a, n), cut(parts[2], a, n)))
        a += n
    return gq, contrib


def apply_pattern(partition, qkv: dict, pattern: AttentionPattern, scale: float | None = None,
                  padding: str = "exclude"):
    """(O_cls, O_query, O_doc) for all groups (R/attention.py:510-537)."""
    for g in GROUPS:
        if g not in qkv:
            raise AttentionError(f"missing Q/K/V for group {g!r}")
    if partition is not None:
        for g in GROUPS:
            if qkv[g][0].shape[-2] != partition.group_len(g):
                raise AttentionError(f"group {g!r} queries have {qkv[g][0].shape[-2]} rows, "
                                     f"partition says {partition.group_len(g)}")
    if scale is None:
        scale = math.sqrt(qkv["cls"][0].shape[-1])
    return tuple(_run_groups(qkv, pattern, scale, padding))


# ---------------------------------------------------------------------------
# Segment-level API (R/attention.py:228-400): arbitrary (K_i, V_i, w_i) tuples.
# Band segments run on the sc_band_scores / sc_band_apply kernels, dense ones on
# cuBLAS, the joint softmax in fp32 on the device.  Not the encoder hot path
# (that is attend_packed's fused kernels), but the same numerics.
# ---------------------------------------------------------------------------

class SegmentScores:
    """Ordered score blocks of one source group (R/attention.py:164-187): dense (rows, target_len)
    blocks (numpy or device tensors) for unwindowed targets, BandMatrix for windowed ones."""

    def __init__(self, segments):
        self.segments = list(segments)
        if not self.segments:
            raise AttentionError("segment tuple must be nonempty")
        rows = {self._rows(seg) for seg in self.segments}
        if len(rows) != 1:
            raise AttentionError(f"segments disagree on row count: {sorted(rows)}")

    @staticmethod
    def _rows(seg) -> int:
        from .band import BandMatrix
        return seg.seq_len if isinstance(seg, BandMatrix) else int(seg.shape[0])

    @property
    def rows(self) -> int:
        return self._rows(self.segments[0])


def segment_softmax(scores, scale: float, padding: str = "exclude") -> SegmentScores:
    """Joint softmax of a source group's score segments on the device (R/attention.py:190-225).

    Band segments stay BandMatrix (invalid slots exactly 0; in zero-logit mode the
    padded mass is computed but not stored); dense numpy blocks come back as numpy.
    float64 inputs are normalised in float64."""
    from .band import BandMatrix

    if scale <= 0:
        raise AttentionError(f"scale must be positive, got {scale}")
    if padding not in PADDING_MODES:
        raise AttentionError(f"unknown padding mode {padding!r}")
    if not isinstance(scores, SegmentScores):
        scores = SegmentScores(scores)
    values, valids, was_np = [], [], []
    for seg in scores.segments:
        if isinstance(seg, BandMatrix):
            values.append(seg.data)
            valids.append(seg.valid)
            was_np.append(False)
        else:
            t, np_in = _to_device(seg)
            values.append(t)
            valids.append(None)
            was_np.append(np_in)
    probs = masked_segment_softmax(values, valids, scale, padding)
    out = []
    for seg, p, ok, np_in in zip(scores.segments, probs, valids, was_np):
        if isinstance(seg, BandMatrix):
            p = torch.where(ok, p, torch.zeros((), dtype=p.dtype, device=p.device))
            out.append(BandMatrix(p.to(seg.data.dtype), seg.window, seg.target_len))
        elif np_in:
            out.append(p.cpu().numpy().astype(np.asarray(seg).dtype, copy=False))
        else:
            out.append(p.to(seg.dtype))
    return SegmentScores(out)


def masked_segment_softmax(values, valids, scale: float, padding: str = "exclude"):
    """Joint softmax over score blocks with optional validity masks (R/attention.py:228-257).

    values: tensors (..., rows, width_i); valids: matching bool masks or None.
    In zero-logit mode invalid slots take part with logit 0."""
    if padding not in PADDING_MODES:
        raise AttentionError(f"unknown padding mode {padding!r}")
    scaled = []
    for val, ok in zip(values, valids):
        y = (val if val.dtype == torch.float64 else val.float()) / scale
        if ok is not None:
            fill = 0.0 if padding == "zero-logit" else -math.inf
            y = torch.where(ok, y, torch.full_like(y, fill))
        scaled.append(y)
    row_max = torch.stack([y.amax(dim=-1) for y in scaled]).amax(dim=0)
    if bool(torch.isneginf(row_max).any()):
        raise AttentionError("a row has zero valid entries across all segments")
    exps = [torch.exp(y - row_max[..., None]) for y in scaled]
    denom = sum(e.sum(dim=-1, keepdim=True) for e in exps)
    return [e / denom for e in exps]


def masked_segment_softmax_backward(probs, grad_probs):
    """Adjoint of the joint softmax w.r.t. the scaled logits (R/attention.py:260-269):
    p * (g - sum over all segments of p * g); invalid slots (p = 0) get 0."""
    ts = [(_to_device(p)[0].float(), _to_device(g)[0].float()) for p, g in zip(probs, grad_probs)]
    dot = sum((p * g).sum(dim=-1, keepdim=True) for p, g in ts)
    out = [p * (g - dot) for p, g in ts]
    if probs and not isinstance(probs[0], torch.Tensor):
        return [o.cpu().numpy().astype(np.asarray(p).dtype, copy=False) for o, p in zip(out, probs)]
    return out


def attend_segments(q, segments, scale: float, padding: str = "exclude", want_cache: bool = False):
    """Windowed cross-attention core (R/attention.py:290-345).

    segments: nonempty list of (k, v, window, extra_invalid); extra_invalid is an
    optional bool (rows, 2w+1) mask of additionally excluded band slots (hard
    exclusions in both padding modes) and must be None for unwindowed segments.
    numpy in -> numpy out (float64 results are computed in fp32 on the device).
    ``want_cache`` also returns the cache ``attend_segments_backward`` consumes
    (the computation then carries autograd through the device band adjoints)."""
    from .band import band_apply, band_apply_ad, band_scores, band_scores_ad, band_validity

    if not segments:
        raise AttentionError("segment tuple must be nonempty")
    if want_cache:
        band_scores, band_apply = band_scores_ad, band_apply_ad  # noqa: F811
    qt, was_np = _to_device(q)
    qf = qt.float()
    if want_cache:
        qf = qf.detach().requires_grad_(True)
    s = qf.shape[-2]
    values, valids, metas, leaves = [], [], [], []
    for k, v, window, extra in segments:
        kt = _to_device(k)[0].float()
        vt = _to_device(v)[0].float()
        if want_cache:
            kt, vt = kt.detach().requires_grad_(True), vt.detach().requires_grad_(True)
            leaves.append((kt, vt))
        if qf.shape[-1] != kt.shape[-1]:
            raise AttentionError("query/key feature dims differ")
        if kt.shape[-2] != vt.shape[-2]:
            raise AttentionError("key/value row counts differ")
        if is_full(window):
            if extra is not None:
                raise AttentionError("extra_invalid only applies to windowed segments")
            sc = torch.matmul(qf, kt.transpose(-1, -2))
            ok = None
        else:
            w = int(window)
            sc = band_scores(qf, kt, w)
            ok = band_validity(s, w, kt.shape[-2], device=qf.device)
            if extra is not None:
                ex = _to_device(extra)[0].bool()
                if padding == "zero-logit":
                    sc = torch.where(ex, torch.full_like(sc, -math.inf), sc)
                else:
                    ok = ok & ~ex
        values.append(sc)
        valids.append(ok)
        metas.append((vt, window))
    with torch.set_grad_enabled(want_cache):
        probs = masked_segment_softmax(values, valids, scale, padding)
        out = None
        for p, (vt, window) in zip(probs, metas):
            part = torch.matmul(p, vt) if is_full(window) else band_apply(p.contiguous(), vt, int(window))
            out = part if out is None else out + part
    res = out.detach().cpu().numpy().astype(np.asarray(q).dtype, copy=False) if was_np else out.detach()
    if not want_cache:
        return res
    return res, {"q": qf, "leaves": leaves, "out": out, "was_np": was_np,
                 "dtype": np.asarray(q).dtype if was_np else None}


def attend_segments_backward(cache, grad_out):
    """Adjoint of attend_segments (R/attention.py:348-378): (grad_q, [(grad_k, grad_v), ...]) in
    segment order, through autograd over the device band adjoints and cuBLAS."""
    g = _to_device(grad_out)[0].float()
    inputs = [cache["q"]] + [t for kv in cache["leaves"] for t in kv]
    grads = torch.autograd.grad(cache["out"], inputs, grad_outputs=g, allow_unused=True)
    grads = [torch.zeros_like(t) if gr is None else gr for t, gr in zip(inputs, grads)]
    conv = (lambda t: t.cpu().numpy().astype(cache["dtype"], copy=False)) if cache["was_np"] else (lambda t: t)
    gq = conv(grads[0])
    kv = [(conv(grads[1 + 2 * i]), conv(grads[2 + 2 * i])) for i in range(len(cache["leaves"]))]
    return gq, kv


def qds_band_exclusions(doc_len: int, window: int, global_positions):
    """Band slots of the doc-doc segment that hit global tokens (R/attention.py:403-413)."""
    if not len(global_positions):
        return None
    w = int(window)
    targets = np.arange(doc_len)[:, None] + np.arange(2 * w + 1)[None, :] - w
    is_global = np.zeros(doc_len + 1, dtype=bool)
    is_global[list(global_positions)] = True
    valid = (targets >= 0) & (targets < doc_len)
    return is_global[np.clip(targets, 0, doc_len)] & valid


def windowed_cross_attention(q, kv, padding: str = "exclude"):
    """Attention of Q over (K_i, V_i, w_i) target segments, scale sqrt(d) (R/attention.py:381-400)."""
    kv = list(kv)
    if not kv:
        raise AttentionError("segment tuple must be nonempty")
    d = np.asarray(q).shape[-1] if not isinstance(q, torch.Tensor) else q.shape[-1]
    segs = []
    for k, v, window in kv:
        vd = v.shape[-1]
        if vd != d:
            raise AttentionError("value feature dim differs from query")
        segs.append((k, v, window, None))
    return attend_segments(q, segs, math.sqrt(d), padding)


def full_attention(q, k, v):
    """Scaled dot-product attention softmax(Q K^T / sqrt(d)) V (R/attention.py:276-287)."""
    qs, ks, vs = (x.shape for x in (q, k, v))
    if qs[-1] != ks[-1] or ks[-2] != vs[-2]:
        raise AttentionError(f"incompatible shapes: Q {tuple(qs)}, K {tuple(ks)}, V {tuple(vs)}")
    return attend_segments(q, [(k, v, FULL, None)], math.sqrt(qs[-1]))
