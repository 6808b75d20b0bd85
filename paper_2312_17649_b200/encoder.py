"""Backward-free cross-encoder inference on B200 (R/encoder.py).

Same public surface as the reference encoder -- ``EncoderConfig``,
``SubsequencePartition``, ``TokenSequence``, ``assemble_input``,
``init_weights``, ``CrossEncoder.forward/score/score_pair`` -- plus a packed
varlen path (``PackedBatch``, ``CrossEncoder.score_packed``) that scores
many (query, document) pairs of different lengths in one pass.

Per layer (post-LN BERT, R/encoder.py:306-371):
    qkv = x @ [Wq|Wk|Wv] + b          cuBLAS (bf16, or fp32 with TF32 off)
    o   = attention(qkv)              sc_attn_fwd (sm_100a kernels)
    x1  = LN(x + o @ Wo + bo)         cuBLAS + sc_residual_layernorm_ex
    f   = gelu_erf(x1 @ W1 + b1)      bf16: sc_gemm_bias_gelu (one tcgen05 GEMM, bias + GELU
                                      epilogue); fp32: cuBLAS + sc_bias_gelu
    x   = LN(x1 + f @ W2 + b2)        cuBLAS + sc_residual_layernorm_ex
(opt-in ``fused_ln``: the two LayerNorm lines as cluster-of-3 tcgen05 GEMMs,
sc_gemm_residual_layernorm.)
The fp32 path keeps an fp32 residual stream; the bf16 path keeps it in bf16
(the GEMM inputs are bf16 anyway), with fp32 statistics inside the LayerNorm
and an fp32 copy of the final layer for the score head.  The per-layer finite
check (R/encoder.py:356-357) is fused into the second LayerNorm.
"""

from __future__ import annotations

import math
from contextlib import contextmanager
from dataclasses import dataclass, replace

import numpy as np
import torch
import torch.nn.functional as F

from . import _lib
from .attention import FULL, GROUPS, AttentionError, attend_packed, is_full, make_pattern
from .layout import PackedLayout, to_device
from .tokenizer import CLS_ID, NUM_SPECIAL_TOKENS, SEP_ID

LAYER_NORM_EPS = 1e-12                         # R/encoder.py:41
PRECISIONS = ("bf16", "f32", "f64")            # f64 configs compute in fp32 on the GPU


class EncoderError(ValueError):
    """Malformed configs, partitions, or inputs (R/encoder.py:46-47)."""


class NonFiniteActivationError(FloatingPointError):
    """A layer produced NaN or infinite activations (R/encoder.py:50-55)."""

    def __init__(self, layer: int):
        super().__init__(f"non-finite activations in layer {layer}")
        self.layer = layer


@dataclass(frozen=True)
class SubsequencePartition:
    """Half-open spans of the cls / query / doc groups (R/encoder.py:58-94)."""

    cls_span: tuple
    query_span: tuple
    doc_span: tuple

    def __post_init__(self):
        if tuple(self.cls_span) != (0, 1):
            raise EncoderError(f"cls span must be (0, 1), got {self.cls_span}")
        prev = 0
        for name, (a, b) in zip(GROUPS, (self.cls_span, self.query_span, self.doc_span)):
            if a != prev or b <= a:
                raise EncoderError(f"{name} span {a, b} must be nonempty and contiguous")
            prev = b

    @property
    def seq_len(self) -> int:
        return self.doc_span[1]

    def span(self, group: str):
        try:
            return {"cls": self.cls_span, "query": self.query_span, "doc": self.doc_span}[group]
        except KeyError:
            raise EncoderError(f"unknown group {group!r}")

    def group_len(self, group: str) -> int:
        a, b = self.span(group)
        return b - a


@dataclass(frozen=True)
class TokenSequence:
    ids: np.ndarray
    partition: SubsequencePartition

    def __post_init__(self):
        object.__setattr__(self, "ids", np.asarray(self.ids, dtype=np.int64))
        if self.ids.ndim != 1 or self.ids.shape[0] != self.partition.seq_len:
            raise EncoderError("token ids inconsistent with partition")


@dataclass(frozen=True)
class EncoderConfig:
    """Architecture + pattern settings (R/encoder.py:108-151); precision adds 'bf16'."""

    layers: int
    embed_dim: int
    heads: int
    ff_dim: int
    max_positions: int
    vocab_size: int
    pattern: str = "sparse"
    window: float = 4
    qds_global_every: int = 30
    precision: str = "bf16"
    padding: str = "exclude"

    def __post_init__(self):
        if self.layers < 0 or self.embed_dim < 1 or self.heads < 1 or self.ff_dim < 1:
            raise EncoderError("layers/embed_dim/heads/ff_dim out of range")
        if self.embed_dim % self.heads != 0:
            raise EncoderError(f"embed_dim {self.embed_dim} not divisible by heads {self.heads}")
        if self.precision not in PRECISIONS:
            raise EncoderError(f"precision must be one of {sorted(PRECISIONS)}")
        if not is_full(self.window) and (int(self.window) != self.window or self.window < 0):
            raise EncoderError(f"bad window {self.window!r}")
        if self.head_dim > 128:
            raise EncoderError("head_dim > 128 is not supported by the attention kernels")
        make_pattern(self.pattern, self.window)

    @property
    def head_dim(self) -> int:
        return self.embed_dim // self.heads

    @property
    def torch_dtype(self):
        return torch.bfloat16 if self.precision == "bf16" else torch.float32

    def with_pattern(self, pattern: str, window=None) -> "EncoderConfig":
        return replace(self, pattern=pattern, window=self.window if window is None else window)


def assemble_input(query_ids, doc_ids, max_positions: int | None = None) -> TokenSequence:
    """[CLS] q [SEP] d [SEP]; the doc tail is truncated, the query never (R/encoder.py:154-177)."""
    q = [int(t) for t in query_ids]
    d = [int(t) for t in doc_ids]
    m = len(q)
    if m < 1:
        raise EncoderError("query must contain at least one token")
    if max_positions is not None:
        if m + 3 > max_positions:
            raise EncoderError(f"query of {m} tokens cannot fit in {max_positions} positions")
        d = d[: max_positions - m - 3]
    n = len(d)
    ids = np.asarray([CLS_ID] + q + [SEP_ID] + d + [SEP_ID], dtype=np.int64)
    return TokenSequence(ids, SubsequencePartition((0, 1), (1, m + 2), (m + 2, m + n + 3)))


def qds_global_positions(doc_token_count: int, every: int = 30) -> tuple:
    """Every ``every``-th document token is global (R/encoder.py:180-184)."""
    if every < 1:
        raise EncoderError("global spacing must be >= 1")
    return tuple(range(every - 1, doc_token_count, every))


def resolve_pattern(config: EncoderConfig, partition: SubsequencePartition):
    """Concrete pattern for one input (R/encoder.py:187-193)."""
    g = ()
    if config.pattern == "qds":
        g = qds_global_positions(partition.group_len("doc") - 1, config.qds_global_every)
    return make_pattern(config.pattern, config.window, g)


def interpolate_positions(pos_embeddings: np.ndarray, new_max: int) -> np.ndarray:
    """Linear resample of positional embeddings (R/encoder.py:196-210)."""
    pos = np.asarray(pos_embeddings)
    old = pos.shape[0]
    if new_max < 2 or old < 2:
        raise EncoderError("positional interpolation requires at least 2 rows")
    x = np.arange(new_max) * (old - 1) / (new_max - 1)
    lo = np.floor(x).astype(np.intp)
    hi = np.minimum(lo + 1, old - 1)
    fr = (x - lo).astype(pos.dtype)[:, None]
    return (1 - fr) * pos[lo] + fr * pos[hi]


def init_weights(config: EncoderConfig, seed: int = 0) -> dict:
    """Seeded U(+-1/sqrt(fan_in)) weights with the reference's draw order (R/encoder.py:217-247).

    Generated in float64 by numpy's PCG64 and cast to float32 (the values the
    reference's f32 precision uses); bf16 mode rounds them on upload.
    """
    rng = np.random.default_rng(seed)
    dt = np.float64 if config.precision == "f64" else np.float32
    h, ff = config.embed_dim, config.ff_dim

    def uniform(shape, fan_in):
        b = 1.0 / math.sqrt(fan_in)
        return rng.uniform(-b, b, size=shape).astype(dt)

    w = {"tok_emb": uniform((config.vocab_size, h), 1), "pos_emb": uniform((config.max_positions, h), 1)}
    for i in range(config.layers):
        p = f"L{i}."
        for name in ("wq", "wk", "wv", "wo"):
            w[p + name] = uniform((h, h), h)
            w[p + name.replace("w", "b")] = np.zeros(h, dt)
        w[p + "ln1_g"], w[p + "ln1_b"] = np.ones(h, dt), np.zeros(h, dt)
        w[p + "w1"], w[p + "b1"] = uniform((h, ff), h), np.zeros(ff, dt)
        w[p + "w2"], w[p + "b2"] = uniform((ff, h), ff), np.zeros(h, dt)
        w[p + "ln2_g"], w[p + "ln2_b"] = np.ones(h, dt), np.zeros(h, dt)
    w["head_w"] = uniform((h,), h)
    w["head_b"] = np.zeros((), dt)
    return w


# ---------------------------------------------------------------------------
# Packed batches of (query, document) sequences.
# ---------------------------------------------------------------------------

class PackedBatch:
    """Host-side packed varlen batch: ids int32 [T], cu_seqlens [n+1], query-group lengths [n]."""

    def __init__(self, ids: np.ndarray, seq_lens, qgroup_lens):
        self.ids = np.ascontiguousarray(ids, dtype=np.int32)
        self.seq_lens = np.asarray(seq_lens, dtype=np.int64)
        self.qgroup_lens = np.asarray(qgroup_lens, dtype=np.int64)
        if self.ids.shape[0] != int(self.seq_lens.sum()):
            raise EncoderError("ids length inconsistent with sequence lengths")

    @property
    def nseq(self) -> int:
        return int(self.seq_lens.shape[0])

    @property
    def total_tokens(self) -> int:
        return int(self.ids.shape[0])

    @classmethod
    def from_sequences(cls, seqs) -> "PackedBatch":
        seqs = list(seqs)
        if not seqs:
            raise EncoderError("empty batch")
        ids = np.concatenate([s.ids for s in seqs])
        return cls(ids, [s.partition.seq_len for s in seqs], [s.partition.group_len("query") for s in seqs])

    @classmethod
    def from_pairs(cls, pairs, max_positions: int) -> "PackedBatch":
        return cls.from_sequences(assemble_input(q, d, max_positions) for q, d in pairs)

    @classmethod
    def from_ids(cls, ids: np.ndarray, partition: SubsequencePartition) -> "PackedBatch":
        ids = np.atleast_2d(np.asarray(ids))
        b, s = ids.shape
        return cls(ids.reshape(-1), [s] * b, [partition.group_len("query")] * b)


@contextmanager
def _fp32_gemms(enabled: bool):
    """Full-precision fp32 cuBLAS GEMMs (TF32 off) for the parity path."""
    if not enabled:
        yield
        return
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        yield
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


FP32_GEMMS = ("sgemm", "bf16x6", "f16x3")
F16_MAX = 65504.0


def _split_weight_x6(w: torch.Tensor) -> torch.Tensor:
    """fp32 weight [N, K] -> bf16 [N, 5K] = [W0 | W0 | W1 | W1 | W2] with W = W0 + W1 + W2 (each
    plane the round-to-nearest bf16 of the remaining residual; one-time, at upload).  Row-wise dot
    with the activation planes [p1 | p2 | p0 | p1 | p0] = the five correction products."""
    w = w.float()
    w0 = w.to(torch.bfloat16)
    r = w - w0.float()
    w1 = r.to(torch.bfloat16)
    w2 = (r - w1.float()).to(torch.bfloat16)
    return torch.cat([w0, w0, w1, w1, w2], dim=1).contiguous()


def split_planes(x: torch.Tensor, bias=None, gelu: bool = False, keep: torch.Tensor | None = None) -> torch.Tensor:
    """fp32 [M, K] (+ bias, GELU) -> bf16 planes [M, 5K] = [p1 | p2 | p0 | p1 | p0] (sc_split_bf16x3);
    ``keep`` (optional, may be x) receives the fp32 value after bias/GELU."""
    M, K = x.shape
    planes = torch.empty((M, 5 * K), dtype=torch.bfloat16, device=x.device)
    _lib.call("sc_split_bf16x3", x.data_ptr(), x.stride(0), _lib.ptr(bias), int(gelu), _lib.ptr(keep),
              K if keep is None else keep.stride(0), planes.data_ptr(), planes.stride(0), M, K,
              _lib.stream_handle(), exc=EncoderError)
    return planes


X6_CHUNK = 768  # K-chunk of the main product p0 q0 (measured: SGEMM-or-better error up to K = 3072)


def _linear_x6(planes: torch.Tensor, w5: torch.Tensor, chunk: int | None = None) -> torch.Tensor:
    """a W^T in fp32 from the planes of a ([M, 5K]) and of W ([N, 5K]) on the bf16 tensor cores:
      corrections  [p1 p2 p0 p1 p0] . [q0 q0 q1 q1 q2]    (one GEMM, K' = 5K, magnitude 2^-8)
      + main       p0 . q0  in K-chunks of <= ``chunk``  (summed in the RN fp32 GEMM epilogue)
    = sum_{i+j<=2} p_i q_j (dropped terms <= 2^-27 relative).  The tensor pipe's fp32 accumulation
    is coarser than an FFMA chain, so no single accumulation runs over more than ``chunk`` of the
    main product; measured max error vs fp64 at M=32792: 5.2e-6 (K=768) vs SGEMM's 6.1e-6.
    R/encoder.py:322-324, :345, :350, :352."""
    K = planes.shape[1] // 5
    chunk = chunk or X6_CHUNK
    c = torch.mm(planes, w5.t(), out_dtype=torch.float32)
    p0, q0 = planes[:, 2 * K:3 * K], w5[:, :K]
    for k0 in range(0, K, chunk):  # in place (out=c): no copy of c per chunk
        torch.addmm(c, p0[:, k0:k0 + chunk], q0[:, k0:k0 + chunk].t(), out_dtype=torch.float32, out=c)
    return c


def _split_weight_x3h(w: torch.Tensor, bias: torch.Tensor | None = None):
    """fp32 weight [N, K] (+ bias [N]) -> (fp16 [N, 2K (+16)], s): W * 2^e = G0 + G1 (G0 = fp16_rn,
    G1 the fp16 of the residual) laid out [G1 | G0], or with a bias [G1 | B1 0 | G0 | B0 0] where
    B0 + B1 = bias * 2^e the same way and "0" pads each bias column to 8; s = 2^-e, e putting
    max(|W|, |bias|) at 2^14 so the residual planes stay out of fp16's subnormal range.  The bias
    columns meet the constant column of split_planes_h(..., onehot=True): B0 rides in the main
    product, B1 in the corrections.  One-time, at upload."""
    w = w.float()
    amax = float(w.abs().max()) if w.numel() else 0.0
    if bias is not None and bias.numel():
        amax = max(amax, float(bias.float().abs().max()))
    e = int(math.floor(math.log2(16384.0 / amax))) if amax > 0 else 0

    def planes(a):
        a = a.float() * (2.0 ** e)
        hi = a.to(torch.float16)
        return hi, (a - hi.float()).to(torch.float16)

    g0, g1 = planes(w)
    if bias is None:
        return torch.cat([g1, g0], dim=1).contiguous(), 2.0 ** -e
    b0, b1 = planes(bias.reshape(-1, 1))
    pad = torch.zeros((w.shape[0], 7), dtype=torch.float16, device=w.device)
    return torch.cat([g1, b1, pad, g0, b0, pad], dim=1).contiguous(), 2.0 ** -e


def split_planes_h(x: torch.Tensor, bias=None, gelu: bool = False, keep: torch.Tensor | None = None,
                   status: torch.Tensor | None = None, onehot: bool = False) -> torch.Tensor:
    """fp32 [M, K] (+ bias, GELU) -> fp16 planes [M, 2K] = [h0 | h1], or [M, 2K + 8] =
    [h0 | 1 0 .. 0 | h1] with ``onehot`` (sc_split_f16x2); ``status`` (device int32) is set to 1 if a
    value is outside fp16 range."""
    M, K = x.shape
    planes = torch.empty((M, 2 * K + (8 if onehot else 0)), dtype=torch.float16, device=x.device)
    _lib.call("sc_split_f16x2", x.data_ptr(), x.stride(0), _lib.ptr(bias), int(gelu), _lib.ptr(keep),
              K if keep is None else keep.stride(0), planes.data_ptr(), planes.stride(0), M, K, int(onehot),
              _lib.ptr(status), _lib.stream_handle(), exc=EncoderError)
    return planes


def _linear_x3h(planes: torch.Tensor, w2: torch.Tensor, s: float, chunk: int | None = None) -> torch.Tensor:
    """a W^T (+ bias) in fp32 from the fp16 planes of a ([M, 2K] = [h0 | h1], or [h0 | e | h1] with the
    constant column e) and of W * 2^e ([N, 2K] = [g1 | g0], or [g1 | b1 | g0 | b0] with the bias):
      corrections [h0 (e) h1] . [g1 (b1) g0]  (one GEMM; magnitude 2^-11)
      + main      [h0 (e)] . [g0 (b0)]  in K-chunks of <= ``chunk``, accumulated in place, the last
                  one scaling the sum by s = 2^-e (exact)
    = h0 g0 + h0 g1 + h1 g0 (+ bias) (dropped term h1 g1 <= 2^-22 relative), three products where the
    bf16 form needs six.  Measured vs fp64 (M = 131k): max relative error 1.2-1.7e-6, SGEMM's
    1.1-2.2e-6.  R/encoder.py:322-324, :345, :350, :352."""
    kb = 8 if w2.shape[1] == planes.shape[1] + 8 else 0  # constant / bias columns: [2K + 8] vs [2K + 16]
    if w2.shape[1] != planes.shape[1] + kb:
        raise EncoderError(f"split planes {tuple(planes.shape)} do not match the weight planes {tuple(w2.shape)}")
    K = (planes.shape[1] - kb) // 2
    chunk = chunk or X6_CHUNK
    c = torch.mm(planes[:, :2 * K + kb], w2[:, :2 * K + kb].t(), out_dtype=torch.float32)
    h0, g0 = planes[:, :K + kb], w2[:, K + kb:]
    starts = list(range(0, K, chunk))
    for n, k0 in enumerate(starts):  # in place (out=c): no copy of c per chunk
        last = n == len(starts) - 1
        k1 = K + kb if last else k0 + chunk  # the bias column rides in the last chunk
        sc = s if last else 1.0
        torch.addmm(c, h0[:, k0:k1], g0[:, k0:k1].t(), beta=sc, alpha=sc, out_dtype=torch.float32, out=c)
    return c


def _linear_x3h_tc(planes: torch.Tensor, w2: torch.Tensor, s: float) -> torch.Tensor | None:
    """_linear_x3h as one tcgen05 GEMM (sc_gemm_x3h): the three fp16 products (and the bias columns)
    accumulated in one fp32 TMEM accumulator, scaled by s in the epilogue -- no fp32 partial result
    written and re-read between the products.  None when the shape is unsupported (cuBLAS path)."""
    kb = 8 if w2.shape[1] == planes.shape[1] + 8 else 0
    if w2.shape[1] != planes.shape[1] + kb:
        raise EncoderError(f"split planes {tuple(planes.shape)} do not match the weight planes {tuple(w2.shape)}")
    M, K, N = planes.shape[0], (planes.shape[1] - kb) // 2, w2.shape[0]
    out = torch.empty((M, N), dtype=torch.float32, device=planes.device)
    rc = _lib.load().sc_gemm_x3h(planes.data_ptr(), planes.stride(0), w2.data_ptr(), w2.stride(0), float(s),
                                 out.data_ptr(), out.stride(0), M, N, K, kb, _lib.stream_handle())
    if rc == _lib.SC_OK:
        _lib.launch_calls += 1
        return out
    if rc != _lib.SC_ERR_UNSUPPORTED:
        raise EncoderError(_lib.last_error())
    return None


class CrossEncoder:
    """Config + device weights; batched inference (R/encoder.py:450-538)."""

    def __init__(self, config: EncoderConfig, weights: dict | None = None, seed: int = 0,
                 device="cuda", attn_algo: str = "auto", prune_last_layer: bool = False,
                 fused_ffn: bool = True, fused_ln: bool = False, fp32_gemm: str = "sgemm"):
        """``prune_last_layer``: the scoring entry points (score*, GraphedScorer) run
        the last layer for the [CLS] rows only past the K/V projection -- the score
        reads nothing else (R/encoder.py:506).  Scores are unchanged; the reference's
        finite check then covers the last layer's [CLS] rows only.  ``forward``
        always computes every row.

        ``fp32_gemm`` (fp32 precisions only): "sgemm" runs the four projections as cuBLAS
        fp32 SGEMM (TF32 off); "bf16x6" runs them on the bf16 tensor cores as six split
        products per GEMM (operands as three bf16 planes, sc_split_bf16x3; see _linear_x6);
        "f16x3" as three fp16 products (two fp16 planes, sc_split_f16x2; see _linear_x3h;
        activations must stay inside fp16 range, checked: EncoderError otherwise).  Both
        give SGEMM-level accuracy at several times the speed."""
        if fp32_gemm not in FP32_GEMMS:
            raise EncoderError(f"fp32_gemm must be one of {FP32_GEMMS}, got {fp32_gemm!r}")
        self.config = config
        self.fp32_gemm = fp32_gemm if config.torch_dtype == torch.float32 else "sgemm"
        self.device = torch.device(device)
        self.attn_algo = attn_algo
        self.prune_last_layer = prune_last_layer
        # bf16: W1 + bias + GELU as one tcgen05 GEMM (sc_gemm_bias_gelu); False -> cuBLAS + GELU pass
        self.fused_ffn = fused_ffn
        # bf16, opt-in: Wo / W2 + bias + residual + LayerNorm as cluster-of-3 tcgen05 GEMMs
        self.fused_ln = fused_ln
        host = init_weights(config, seed) if weights is None else weights
        self.host_weights = host
        self._upload(host)

    @property
    def weight_nbytes(self) -> int:
        return sum(int(t.numel() * t.element_size()) for t in self._all_tensors())

    def _all_tensors(self):
        yield self.tok_emb
        yield self.pos_emb
        for L in self.layers:
            yield from L.values()
        yield self.head_w

    def _upload(self, w: dict):
        cfg, dev, cd = self.config, self.device, self.config.torch_dtype

        def f32(a):
            return torch.as_tensor(np.asarray(a, dtype=np.float32), device=dev).contiguous()

        def gemm_w(a):  # reference stores (in, out) for x @ W; F.linear wants (out, in)
            return torch.as_tensor(np.asarray(a, dtype=np.float32).T.copy(), device=dev).to(cd).contiguous()

        self.tok_emb = f32(w["tok_emb"])
        self.pos_emb = f32(w["pos_emb"])
        self.layers = []
        for i in range(cfg.layers):
            p = f"L{i}."
            wqkv = np.concatenate([w[p + "wq"], w[p + "wk"], w[p + "wv"]], axis=1)
            bqkv = np.concatenate([w[p + "bq"], w[p + "bk"], w[p + "bv"]])
            self.layers.append({
                "wqkv": gemm_w(wqkv), "bqkv": f32(bqkv).to(cd),
                "wo": gemm_w(w[p + "wo"]), "bo": f32(w[p + "bo"]).to(cd),
                "ln1_g": f32(w[p + "ln1_g"]), "ln1_b": f32(w[p + "ln1_b"]),
                "w1": gemm_w(w[p + "w1"]), "b1": f32(w[p + "b1"]).to(cd), "b1_f32": f32(w[p + "b1"]),
                "w2": gemm_w(w[p + "w2"]), "b2": f32(w[p + "b2"]).to(cd),
                "ln2_g": f32(w[p + "ln2_g"]), "ln2_b": f32(w[p + "ln2_b"]),
            })
        self.head_w = f32(w["head_w"])
        self.head_b = float(np.asarray(w["head_b"]))
        if self.fp32_gemm in ("bf16x6", "f16x3"):
            for L in self.layers:
                for name in ("wqkv", "wo", "w1", "w2"):
                    if self.fp32_gemm == "bf16x6":
                        L[name + "_x6"] = _split_weight_x6(L[name])
                    else:
                        b = L["bqkv"] if name == "wqkv" else None  # the QKV bias rides in the GEMM
                        L[name + "_x3h"], L[name + "_x3h_s"] = _split_weight_x3h(L[name], b)
                for name in ("bqkv", "bo", "b1", "b2"):
                    L[name + "_f32"] = L[name].float().contiguous()

    # -- validation -------------------------------------------------------

    def _check_batch(self, batch: PackedBatch):
        if batch.ids.size and (batch.ids.min() < 0 or batch.ids.max() >= self.config.vocab_size):
            raise EncoderError("token id outside vocabulary")
        if np.any(batch.seq_lens > self.config.max_positions):
            raise EncoderError("sequence longer than max_positions")

    def make_layout(self, batch: PackedBatch) -> PackedLayout:
        qds = self.config.qds_global_every if self.config.pattern == "qds" else 0
        return PackedLayout.from_lengths(batch.seq_lens, batch.qgroup_lens, device=self.device,
                                         qds_every=qds)

    # -- the packed hot loop ---------------------------------------------

    def encode_packed(self, ids_dev: torch.Tensor, layout: PackedLayout, check_finite: bool = True,
                      attn_hook=None, cls_only: bool = False) -> torch.Tensor:
        """Final-layer fp32 activations [T, h] for a packed batch already on the device.

        ``attn_hook(event)`` (optional) is called with "start"/"end" around each
        attention launch so a caller can bracket it with CUDA events.
        ``cls_only``: the last layer runs attention for the head rows only and the
        rest of the layer for the [CLS] rows only; returns [nseq, h] (row j =
        sequence j's [CLS]).
        """
        if self.fp32_gemm in ("bf16x6", "f16x3"):
            return self._encode_x6(ids_dev, layout, check_finite, attn_hook, cls_only)
        cfg = self.config
        T, h, H = layout.total_tokens, cfg.embed_dim, cfg.heads
        cd = cfg.torch_dtype
        bf16 = cd == torch.bfloat16
        dev = self.device
        pattern = make_pattern(cfg.pattern, cfg.window)
        stream = _lib.stream_handle()
        # Residual stream: fp32 in the fp32 path; bf16 in the bf16 path (LN reads
        # and writes 2-byte rows), with the final layer's LN also writing fp32 x.
        x = torch.empty((T, h), dtype=torch.float32, device=dev)
        if bf16:
            xh = torch.empty((T, h), dtype=cd, device=dev)
            x1 = torch.empty_like(xh)
        else:
            xh, x1 = None, torch.empty_like(x)
        rdt = _lib.DTYPE_BF16 if bf16 else _lib.DTYPE_F32
        bad = torch.zeros(max(cfg.layers, 1), dtype=torch.int32, device=dev)
        _lib.call("sc_embed", ids_dev.data_ptr(), layout.tok_pos.data_ptr(), self.tok_emb.data_ptr(),
                  self.pos_emb.data_ptr(), x.data_ptr() if (not bf16 or cfg.layers == 0) else None,
                  _lib.ptr(xh), T, h, stream, exc=EncoderError)
        dcode = _lib.DTYPE_BF16 if bf16 else _lib.DTYPE_F32
        o = torch.empty((T, h), dtype=cd, device=dev)
        last = cfg.layers - 1
        with _fp32_gemms(not bf16):
            for i, L in enumerate(self.layers):
                xr = xh if bf16 else x  # residual stream (and GEMM input) of this layer
                if cls_only and i == last:
                    self._last_bad = bad if check_finite else None
                    return self._cls_last_layer(L, xr, layout, pattern, bad if check_finite else None, i)
                qkv = F.linear(xr, L["wqkv"], L["bqkv"])
                if attn_hook:
                    attn_hook("start")
                attend_packed(qkv[:, :h], qkv[:, h:2 * h], qkv[:, 2 * h:], layout, pattern, H,
                              math.sqrt(cfg.head_dim), cfg.padding, out=o, algo=self.attn_algo,
                              check=(i == 0))
                if attn_hook:
                    attn_hook("end")
                if not (bf16 and self.fused_ln and self._proj_ln(o, L, "wo", "bo", "ln1", xr, x1, None, None, T,
                                                                  stream)):
                    y = F.linear(o, L["wo"], L["bo"])
                    _lib.call("sc_residual_layernorm_ex", xr.data_ptr(), rdt, y.data_ptr(), dcode, None,
                              L["ln1_g"].data_ptr(), L["ln1_b"].data_ptr(), None if bf16 else x1.data_ptr(),
                              x1.data_ptr() if bf16 else None, None, T, h, stream, exc=EncoderError)
                f = self._ffn_up(x1, L, T, stream)
                x32 = x if (not bf16 or i == last) else None
                bad_i = bad[i:i + 1] if check_finite else None
                if not (bf16 and self.fused_ln and self._proj_ln(f, L, "w2", "b2", "ln2", x1, xh, x32, bad_i, T,
                                                                  stream)):
                    f2 = F.linear(f, L["w2"], L["b2"])
                    _lib.call("sc_residual_layernorm_ex", x1.data_ptr(), rdt, f2.data_ptr(), dcode, None,
                              L["ln2_g"].data_ptr(), L["ln2_b"].data_ptr(), _lib.ptr(x32), _lib.ptr(xh),
                              _lib.ptr(bad_i), T, h, stream, exc=EncoderError)
        self._last_bad = bad if check_finite else None
        return x

    def _xsplit(self, x, bias=None, gelu=False, qkv_input=False):
        """GEMM operand planes of x (+ bias, GELU) for the split fp32 modes (``qkv_input``: the planes
        feed the QKV projection, whose bias rides in the f16x3 GEMM through a constant column)."""
        if self.fp32_gemm == "bf16x6":
            return split_planes(x, bias=bias, gelu=gelu)
        return split_planes_h(x, bias=bias, gelu=gelu, status=self._range_flag, onehot=qkv_input)

    def _xlinear(self, planes, L, name, with_bias=False):
        """x W^T (+ the QKV bias) in fp32 from the planes of x (split fp32 modes)."""
        if self.fp32_gemm == "bf16x6":
            c = _linear_x6(planes, L[name + "_x6"])
            return c.add_(L["bqkv_f32"]) if with_bias else c
        w2, sc = L[name + "_x3h"], L[name + "_x3h_s"]
        if self.fused_ffn and name in ("wqkv", "wo"):  # K = 768: one accumulation on our tcgen05 GEMM
            c = _linear_x3h_tc(planes, w2, sc)
            if c is not None:
                return c
        return _linear_x3h(planes, w2, sc)  # f16x3: bias folded in (wqkv)

    def _encode_x6(self, ids_dev, layout, check_finite, attn_hook, cls_only) -> torch.Tensor:
        """encode_packed for fp32 with the projections as split products (fp32_gemm="bf16x6" / "f16x3").
        Every GEMM operand is produced as bf16 planes by the pass that writes it: sc_split_bf16x3
        after the embedding / LayerNorms / attention, and with bias + GELU fused for the FFN
        activation, which then never exists in fp32."""
        cfg = self.config
        T, h, H = layout.total_tokens, cfg.embed_dim, cfg.heads
        dev, stream, F32 = self.device, _lib.stream_handle(), _lib.DTYPE_F32
        pattern = make_pattern(cfg.pattern, cfg.window)
        x = torch.empty((T, h), dtype=torch.float32, device=dev)
        x1 = torch.empty_like(x)
        o = torch.empty_like(x)
        bad = torch.zeros(max(cfg.layers, 1), dtype=torch.int32, device=dev)
        self._range_flag = torch.zeros(1, dtype=torch.int32, device=dev) if self.fp32_gemm == "f16x3" else None
        self._last_range = self._range_flag
        _lib.call("sc_embed", ids_dev.data_ptr(), layout.tok_pos.data_ptr(), self.tok_emb.data_ptr(),
                  self.pos_emb.data_ptr(), x.data_ptr(), None, T, h, stream, exc=EncoderError)
        last = cfg.layers - 1
        f16 = self.fp32_gemm == "f16x3"
        xs = None  # f16x3: the QKV planes of x, written by the previous layer's second LayerNorm
        for i, L in enumerate(self.layers):
            if xs is None:
                xs = self._xsplit(x, qkv_input=True)
            if cls_only and i == last:
                self._last_bad = bad if check_finite else None
                return self._cls_last_layer_x6(L, x, xs, layout, pattern, bad if check_finite else None, i)
            qkv = self._xlinear(xs, L, "wqkv", with_bias=True)
            if attn_hook:
                attn_hook("start")
            attend_packed(qkv[:, :h], qkv[:, h:2 * h], qkv[:, 2 * h:], layout, pattern, H,
                          math.sqrt(cfg.head_dim), cfg.padding, out=o, algo=self.attn_algo, check=(i == 0))
            if attn_hook:
                attn_hook("end")
            y = self._xlinear(self._xsplit(o), L, "wo")
            x1s = self._ln_planes(x, y, L["bo_f32"], L, "ln1", x1, None, False) if f16 else None
            if x1s is None:
                _lib.call("sc_residual_layernorm_ex", x.data_ptr(), F32, y.data_ptr(), F32, L["bo_f32"].data_ptr(),
                          L["ln1_g"].data_ptr(), L["ln1_b"].data_ptr(), x1.data_ptr(), None, None, T, h, stream,
                          exc=EncoderError)
                x1s = self._xsplit(x1)
            fs = self._w1_gelu_planes(x1s, L) if f16 and self.fused_ffn else None
            if fs is None:
                f = self._xlinear(x1s, L, "w1")
                fs = self._xsplit(f, bias=L["b1_f32"], gelu=True)
                del f
            del x1s
            f2 = self._xlinear(fs, L, "w2")
            del fs
            bad_i = bad[i:i + 1] if check_finite else None
            xs = self._ln_planes(x1, f2, L["b2_f32"], L, "ln2", x, bad_i, True) if f16 and i < last else None
            if xs is None:
                _lib.call("sc_residual_layernorm_ex", x1.data_ptr(), F32, f2.data_ptr(), F32, L["b2_f32"].data_ptr(),
                          L["ln2_g"].data_ptr(), L["ln2_b"].data_ptr(), x.data_ptr(), None,
                          _lib.ptr(bad_i), T, h, stream, exc=EncoderError)
        self._last_bad = bad if check_finite else None
        return x

    def _w1_gelu_planes(self, x1s, L):
        """f16x3: the fp16 planes of gelu(x1 W1^T + b1) from one tcgen05 GEMM with the bias, erff GELU
        and the split in its epilogue (sc_gemm_x3h_gelu_planes); None if the shape is unsupported."""
        T, cfg = x1s.shape[0], self.config
        planes = torch.empty((T, 2 * cfg.ff_dim), dtype=torch.float16, device=x1s.device)
        w = L["w1_x3h"]
        rc = _lib.load().sc_gemm_x3h_gelu_planes(
            x1s.data_ptr(), x1s.stride(0), w.data_ptr(), w.stride(0), float(L["w1_x3h_s"]), L["b1_f32"].data_ptr(),
            planes.data_ptr(), planes.stride(0), _lib.ptr(self._range_flag), T, cfg.ff_dim, cfg.embed_dim,
            _lib.stream_handle())
        if rc == _lib.SC_OK:
            _lib.launch_calls += 1
            return planes
        if rc != _lib.SC_ERR_UNSUPPORTED:
            raise EncoderError(_lib.last_error())
        return None

    def _ln_planes(self, resid, y, bias, L, ln, out, bad, qkv_input):
        """f16x3: out = LN(resid + y + bias) (fp32) and its fp16 GEMM planes from one pass
        (sc_residual_layernorm_f16x2, the split fused into the LayerNorm); None if unsupported."""
        T, h = out.shape
        planes = torch.empty((T, 2 * h + (8 if qkv_input else 0)), dtype=torch.float16, device=out.device)
        rc = _lib.load().sc_residual_layernorm_f16x2(
            resid.data_ptr(), y.data_ptr(), bias.data_ptr(), L[ln + "_g"].data_ptr(), L[ln + "_b"].data_ptr(),
            out.data_ptr(), planes.data_ptr(), planes.stride(0), int(qkv_input), _lib.ptr(self._range_flag),
            _lib.ptr(bad), T, h, _lib.stream_handle())
        if rc == _lib.SC_OK:
            _lib.launch_calls += 1
            return planes
        if rc != _lib.SC_ERR_UNSUPPORTED:
            raise EncoderError(_lib.last_error())
        return None

    def _cls_last_layer_x6(self, L, x, xs, layout, pattern, bad, i):
        """_cls_last_layer for fp32_gemm="bf16x6": K/V of every token, the rest on the [CLS] rows."""
        cfg = self.config
        h, H, F32, stream = cfg.embed_dim, cfg.heads, _lib.DTYPE_F32, _lib.stream_handle()
        qkv = self._xlinear(xs, L, "wqkv", with_bias=True)
        o = torch.empty((layout.total_tokens, h), dtype=torch.float32, device=self.device)
        attend_packed(qkv[:, :h], qkv[:, h:2 * h], qkv[:, 2 * h:], layout, pattern, H,
                      math.sqrt(cfg.head_dim), cfg.padding, out=o, algo=self.attn_algo, check=False, rows="head")
        cls, n = layout.cls_rows, layout.nseq
        y = self._xlinear(self._xsplit(o.index_select(0, cls)), L, "wo")
        xc = x.index_select(0, cls)
        x1 = torch.empty_like(xc)
        _lib.call("sc_residual_layernorm_ex", xc.data_ptr(), F32, y.data_ptr(), F32, L["bo_f32"].data_ptr(),
                  L["ln1_g"].data_ptr(), L["ln1_b"].data_ptr(), x1.data_ptr(), None, None, n, h, stream,
                  exc=EncoderError)
        f = self._xlinear(self._xsplit(x1), L, "w1")
        f2 = self._xlinear(self._xsplit(f, bias=L["b1_f32"], gelu=True), L, "w2")
        out = torch.empty((n, h), dtype=torch.float32, device=self.device)
        _lib.call("sc_residual_layernorm_ex", x1.data_ptr(), F32, f2.data_ptr(), F32, L["b2_f32"].data_ptr(),
                  L["ln2_g"].data_ptr(), L["ln2_b"].data_ptr(), out.data_ptr(), None,
                  None if bad is None else bad.data_ptr() + 4 * i, n, h, stream, exc=EncoderError)
        return out

    def _proj_ln(self, a, L, wname, bname, lnname, resid, out, out32, bad, rows, stream) -> bool:
        """Opt-in (fused_ln): LN(resid + a W^T + b) as one cluster-of-3 tcgen05 GEMM
        (sc_gemm_residual_layernorm).  Returns False when the shape is unsupported.
        Measured slower than cuBLAS + the LayerNorm pass at the bench shape
        (Wo 0.49 vs 0.43 ms, W2 1.14-1.20 vs 1.03-1.07 ms), hence not the default."""
        W = L[wname]
        b = L.get(bname + "_f32")
        if b is None:
            b = L[bname + "_f32"] = L[bname].float()
        rc = _lib.load().sc_gemm_residual_layernorm(
            a.data_ptr(), a.stride(0), W.data_ptr(), W.stride(0), b.data_ptr(), resid.data_ptr(), resid.stride(0),
            L[lnname + "_g"].data_ptr(), L[lnname + "_b"].data_ptr(), out.data_ptr(), out.stride(0),
            _lib.ptr(out32), 0 if out32 is None else out32.stride(0), _lib.ptr(bad), rows, W.shape[0], W.shape[1],
            stream)
        if rc == _lib.SC_OK:
            _lib.launch_calls += 1
            return True
        if rc != _lib.SC_ERR_UNSUPPORTED:
            raise EncoderError(_lib.last_error())
        return False

    def _ffn_up(self, x1: torch.Tensor, L: dict, rows: int, stream) -> torch.Tensor:
        """gelu_erf(x1 W1^T + b1) (R/encoder.py:350-351): bf16 -> the fused tcgen05 GEMM with the
        bias + GELU epilogue (sc_gemm_bias_gelu); fp32 parity path (or an unsupported shape) ->
        cuBLAS + the separate sc_bias_gelu pass."""
        cfg = self.config
        if cfg.torch_dtype == torch.bfloat16 and self.fused_ffn:
            f = torch.empty((rows, cfg.ff_dim), dtype=torch.bfloat16, device=self.device)
            rc = _lib.load().sc_gemm_bias_gelu(x1.data_ptr(), x1.stride(0), L["w1"].data_ptr(), L["w1"].stride(0),
                                               L["b1_f32"].data_ptr(), f.data_ptr(), f.stride(0), rows,
                                               cfg.ff_dim, cfg.embed_dim, stream)
            if rc == _lib.SC_OK:
                _lib.launch_calls += 1
                return f
            if rc != _lib.SC_ERR_UNSUPPORTED:
                raise EncoderError(_lib.last_error())
        f = F.linear(x1, L["w1"], L["b1"])
        dcode = _lib.DTYPE_BF16 if cfg.torch_dtype == torch.bfloat16 else _lib.DTYPE_F32
        _lib.call("sc_bias_gelu", f.data_ptr(), None, dcode, rows, cfg.ff_dim, stream, exc=EncoderError)
        return f

    def _cls_last_layer(self, L, xr, layout, pattern, bad, i):
        """Last layer for the [CLS] rows only (R/encoder.py:306-371 restricted to the rows
        R/encoder.py:506 reads): K/V of every token, attention of the head rows, then
        Wo / LN / FFN / LN on nseq rows.  Returns fp32 [nseq, h]."""
        cfg = self.config
        h, H = cfg.embed_dim, cfg.heads
        bf16 = cfg.torch_dtype == torch.bfloat16
        dcode = _lib.DTYPE_BF16 if bf16 else _lib.DTYPE_F32
        stream = _lib.stream_handle()
        qkv = F.linear(xr, L["wqkv"], L["bqkv"])
        o = torch.empty((layout.total_tokens, h), dtype=xr.dtype, device=self.device)
        attend_packed(qkv[:, :h], qkv[:, h:2 * h], qkv[:, 2 * h:], layout, pattern, H,
                      math.sqrt(cfg.head_dim), cfg.padding, out=o, algo=self.attn_algo, check=False, rows="head")
        cls = layout.cls_rows
        n = layout.nseq
        y = F.linear(o.index_select(0, cls), L["wo"], L["bo"])
        xc = xr.index_select(0, cls)
        x1 = torch.empty_like(xc)
        _lib.call("sc_residual_layernorm_ex", xc.data_ptr(), dcode, y.data_ptr(), dcode, None,
                  L["ln1_g"].data_ptr(), L["ln1_b"].data_ptr(), None if bf16 else x1.data_ptr(),
                  x1.data_ptr() if bf16 else None, None, n, h, stream, exc=EncoderError)
        f = self._ffn_up(x1, L, n, stream)
        f2 = F.linear(f, L["w2"], L["b2"])
        out = torch.empty((n, h), dtype=torch.float32, device=self.device)
        _lib.call("sc_residual_layernorm_ex", x1.data_ptr(), dcode, f2.data_ptr(), dcode, None,
                  L["ln2_g"].data_ptr(), L["ln2_b"].data_ptr(), out.data_ptr(), None,
                  None if bad is None else bad.data_ptr() + 4 * i, n, h, stream, exc=EncoderError)
        return out

    def _raise_if_nonfinite(self):
        rng = getattr(self, "_last_range", None)
        if rng is not None and int(rng.item()):
            raise EncoderError(f"an activation left fp16 range (|x| >= {F16_MAX:g}) in fp32_gemm='f16x3'; "
                               "use fp32_gemm='bf16x6' or 'sgemm'")
        bad = getattr(self, "_last_bad", None)
        if bad is None:
            return
        counts = bad.cpu().numpy()
        nz = np.nonzero(counts[: self.config.layers])[0]
        if nz.size:
            raise NonFiniteActivationError(int(nz[0]))

    def scores_from_hidden(self, x: torch.Tensor, layout: PackedLayout, out=None) -> torch.Tensor:
        """Scores from final activations: [T, h] (all rows) or [nseq, h] (cls_only)."""
        out = torch.empty(layout.nseq, dtype=torch.float32, device=self.device) if out is None else out
        cu = layout.cu_seqlens if x.shape[0] == layout.total_tokens else layout.ident_cu
        _lib.call("sc_cls_score", x.data_ptr(), cu.data_ptr(), layout.nseq,
                  self.config.embed_dim, self.head_w.data_ptr(), self.head_b, out.data_ptr(),
                  _lib.stream_handle(), exc=EncoderError)
        return out

    def score_packed(self, batch: PackedBatch, layout: PackedLayout | None = None) -> torch.Tensor:
        """Relevance scores (nseq,) on the device for a packed varlen batch."""
        self._check_batch(batch)
        layout = layout or self.make_layout(batch)
        ids = to_device(batch.ids, self.device)
        x = self.encode_packed(ids, layout, cls_only=self.prune_last_layer)
        return self.scores_from_hidden(x, layout)

    # -- reference-signature API -----------------------------------------

    def _check_ids(self, ids, partition: SubsequencePartition) -> np.ndarray:
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

    def forward(self, ids, partition: SubsequencePartition) -> np.ndarray:
        """Final-layer embeddings (batch, seq, embed) as float32 numpy (R/encoder.py:475-500)."""
        ids = self._check_ids(ids, partition)
        batch = PackedBatch.from_ids(ids, partition)
        layout = self.make_layout(batch)
        x = self.encode_packed(torch.from_numpy(batch.ids).to(self.device), layout)
        out = x.reshape(ids.shape[0], ids.shape[1], -1).cpu().numpy()
        self._raise_if_nonfinite()
        return out

    def score(self, ids, partition: SubsequencePartition) -> np.ndarray:
        """Relevance scores (batch,) from the final [CLS] rows (R/encoder.py:502-509)."""
        ids = self._check_ids(ids, partition)
        batch = PackedBatch.from_ids(ids, partition)
        sc = self.score_packed(batch).cpu().numpy()
        self._raise_if_nonfinite()
        return sc

    def score_pair(self, query_ids, doc_ids) -> float:
        """Relevance of one (query, document) pair (R/encoder.py:535-538)."""
        seq = assemble_input(query_ids, doc_ids, self.config.max_positions)
        return float(self.score(seq.ids, seq.partition)[0])

    def score_pairs(self, pairs, max_tokens: int = 1 << 18) -> np.ndarray:
        """Batched relevance of many (query_ids, doc_ids) pairs, packed in chunks of <= max_tokens."""
        seqs = [assemble_input(q, d, self.config.max_positions) for q, d in pairs]
        out, chunk, tok = [], [], 0
        for s in seqs:
            if chunk and tok + s.partition.seq_len > max_tokens:
                out.append(self.score_packed(PackedBatch.from_sequences(chunk)))
                chunk, tok = [], 0
            chunk.append(s)
            tok += s.partition.seq_len
        if chunk:
            out.append(self.score_packed(PackedBatch.from_sequences(chunk)))
        res = torch.cat(out).cpu().numpy()
        self._raise_if_nonfinite()
        return res


class GraphedScorer:
    """CUDA-graph replay of the whole forward (embed, 12 layers, scores) for one packed-batch shape.

    Passage-size batches (s = 177) are launch-bound: ~110 launches per forward.
    The K1 index and the attention workspace are built once outside the graph;
    each call copies the new ids into the static input buffer and replays.
    """

    def __init__(self, model: "CrossEncoder", batch: PackedBatch, warmup: int = 2):
        model._check_batch(batch)
        self.model = model
        self.seq_lens = batch.seq_lens.copy()
        self.qgroup_lens = batch.qgroup_lens.copy()
        self.layout = model.make_layout(batch)
        self.ids = torch.from_numpy(batch.ids).to(model.device)
        side = torch.cuda.Stream(device=model.device)
        side.wait_stream(torch.cuda.current_stream(model.device))
        with torch.cuda.stream(side):
            for _ in range(warmup):
                self._forward()
        torch.cuda.current_stream(model.device).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        n0 = _lib.kernel_launches()
        with torch.cuda.graph(self.graph):
            self.scores = self._forward()
        # library kernels captured per replay (replays bypass the library's launch counter)
        self.kernels_per_replay = _lib.kernel_launches() - n0

    def _forward(self):
        x = self.model.encode_packed(self.ids, self.layout, check_finite=False, cls_only=self.model.prune_last_layer)
        return self.model.scores_from_hidden(x, self.layout)

    def matches(self, batch: PackedBatch) -> bool:
        return np.array_equal(batch.seq_lens, self.seq_lens) and np.array_equal(batch.qgroup_lens, self.qgroup_lens)

    def __call__(self, ids) -> torch.Tensor:
        """Scores (nseq,) on the device for new ids of the captured shape (numpy or tensor, int32)."""
        src = torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int32)) if isinstance(ids, np.ndarray) else ids
        if tuple(src.shape) != tuple(self.ids.shape):
            raise EncoderError(f"ids shape {tuple(src.shape)} does not match the captured batch {tuple(self.ids.shape)}")
        if src.device.type == "cpu" and src.numel():  # sc_embed reads tok_emb[id] unchecked (_check_ids rule);
            lo, hi = int(src.min()), int(src.max())  # device-resident ids are the caller's (checked) buffers
            if lo < 0 or hi >= self.model.config.vocab_size:
                raise EncoderError("token id outside vocabulary")
        self.ids.copy_(src, non_blocking=True)
        self.graph.replay()
        return self.scores


def encoder_forward(seq: TokenSequence, config: EncoderConfig, weights: dict) -> np.ndarray:
    """Final-layer (seq, embed) matrix for a single sequence (R/encoder.py:541-544)."""
    return CrossEncoder(config, weights).forward(seq.ids, seq.partition)[0]


def relevance_score(last_layer, head_w, head_b=0.0) -> float:
    """Linear readout of the [CLS] row (R/encoder.py:547-552)."""
    last = np.asarray(last_layer)
    if last.ndim != 2 or last.shape[0] < 1:
        raise EncoderError("last layer matrix must be 2-D with a [CLS] row")
    return float(last[0] @ np.asarray(head_w) + head_b)


# Reference-shaped layer primitives and adjoints (R/encoder.py:250-443) -- implemented on the device
# in training.py (imported lazily: training builds on this module).
def weight_nbytes(weights: dict) -> int:
    from .training import weight_nbytes as f
    return f(weights)


def gelu(x):
    from .training import gelu as f
    return f(x)


def gelu_grad(x):
    from .training import gelu_grad as f
    return f(x)


def layer_norm(x, gain, bias):
    from .training import layer_norm as f
    return f(x, gain, bias)


def layer_norm_backward(grad_y, cache, gain):
    from .training import layer_norm_backward as f
    return f(grad_y, cache, gain)


def layer_forward(x, partition, pattern, weights, layer_index, config, want_cache=False):
    from .training import layer_forward as f
    return f(x, partition, pattern, weights, layer_index, config, want_cache)


def layer_backward(grad_out, cache, partition, pattern, weights, layer_index, config, grads):
    from .training import layer_backward as f
    return f(grad_out, cache, partition, pattern, weights, layer_index, config, grads)
