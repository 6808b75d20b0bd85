"""ctypes binding of the in-tree C-ABI library ``_lib/libsparsecross_b200.so``.

The signatures mirror ``include/sparsecross_b200.h``.  There is no CPU
fallback: if the library is missing, every GPU entry point raises
``LibraryNotBuiltError`` (run ``python __graft_entry__.py build`` or
``make -C paper_2312_17649_b200/csrc``).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# SC_LIB_PATH: an alternative build of the same library (measurement A/B only)
LIB_PATH = os.environ.get("SC_LIB_PATH") or os.path.join(HERE, "_lib", "libsparsecross_b200.so")

SC_OK = 0
SC_ERR_INVALID = 1
SC_ERR_CUDA = 2
SC_ERR_UNSUPPORTED = 3
SC_ERR_NO_VALID_ROW = 4

LINK_NONE = -2
LINK_FULL = -1

DTYPE_F32 = 0
DTYPE_BF16 = 1

PAD_EXCLUDE = 0
PAD_ZERO_LOGIT = 1

ALGO_AUTO = 0
ALGO_GENERIC = 1
ALGO_BAND_MMA = 2
ALGO_TC = 3
ALGO_HEAD_ROWS = 4

_p = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_sz = C.c_size_t
_f32 = C.c_float

# name -> (restype, argtypes); the exact exported surface of sparsecross_b200.h.
SIGNATURES = {
    "sc_last_error": (C.c_char_p, []),
    "sc_version": (C.c_int, []),
    "sc_kernel_launches": (C.c_uint64, []),
    "sc_index_build": (C.c_int, [_p, _p, _i32, _i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "sc_mask_export": (C.c_int, [_p, _p, _i32, _i32, _i32, _p, _p, _p, _p]),
    "sc_band_validity": (C.c_int, [_i32, _i32, _i32, _p, _p]),
    "sc_band_scores": (C.c_int, [_p, _p, _p, _i64, _i32, _i32, _i32, _i32, _i32, _p]),
    "sc_band_apply": (C.c_int, [_p, _p, _p, _i64, _i32, _i32, _i32, _i32, _i32, _p]),
    "sc_attn_workspace_bytes": (_sz, [_i32, _i32, _i32, _i32, _i32, _i32, _p]),
    "sc_attn_workspace_bytes_qds": (_sz, [_i32, _i32, _i32, _i32, _i32, _i32, _p, _i32]),
    "sc_attn_fwd": (C.c_int, [_p, _p, _p, _i64, _p, _i64, _p, _p, _i32, _i32, _i32, _i32, _p, _i32,
                              _f32, _i32, _p, _p, _p, _i32, _i32, _p, _p, _p, _i32, _p, _sz, _p, _p]),
    "sc_band_scores_backward": (C.c_int, [_p, _p, _p, _p, _p, _i64, _i32, _i32, _i32, _i32, _i32, _p]),
    "sc_band_apply_backward": (C.c_int, [_p, _p, _p, _p, _p, _i64, _i32, _i32, _i32, _i32, _i32, _p]),
    "sc_attn_bwd_workspace_bytes": (_sz, [_i32, _i32, _i32, _i32]),
    "sc_attn_bwd": (C.c_int, [_p, _p, _p, _i64, _p, _i64, _p, _i64, _p, _p, _p, _i64, _i32, _p, _p, _i32, _i32, _i32,
                              _i32, _p, _i32, _f32, _i32, _p, _p, _p, _p, _i32, _i32, _i32, _p, _sz, _p]),
    "sc_embed": (C.c_int, [_p, _p, _p, _p, _p, _p, _i32, _i32, _p]),
    "sc_residual_layernorm": (C.c_int, [_p, _p, _i32, _p, _p, _p, _p, _p, _i32, _i32, _p]),
    "sc_residual_layernorm_ex": (C.c_int, [_p, _i32, _p, _i32, _p, _p, _p, _p, _p, _p, _i32, _i32, _p]),
    "sc_bias_gelu": (C.c_int, [_p, _p, _i32, _i64, _i32, _p]),
    "sc_gemm_bias_gelu": (C.c_int, [_p, _i64, _p, _i64, _p, _p, _i64, _i32, _i32, _i32, _p]),
    "sc_gemm_bias_gelu_pre": (C.c_int, [_p, _i64, _p, _i64, _p, _p, _i64, _p, _i64, _i32, _i32, _i32, _p]),
    "sc_gemm_residual_layernorm": (C.c_int, [_p, _i64, _p, _i64, _p, _p, _i64, _p, _p, _p, _i64, _p, _i64, _p,
                                             _i32, _i32, _i32, _p]),
    "sc_adamw_step": (C.c_int, [_p, _p, _p, _p, _p, _i64, C.c_double, C.c_double, C.c_double, C.c_double,
                                C.c_double, _i64, _p]),
    "sc_layernorm_fwd": (C.c_int, [_p, _i32, _p, _i32, _p, _p, _p, _p, _p, _p, _i32, _i32, _f32, _p]),
    "sc_layernorm_bwd": (C.c_int, [_p, _p, _p, _i32, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _i32, _i32, _p]),
    "sc_colsum": (C.c_int, [_p, _i32, _i64, _i32, _i32, _p, _p, _p]),
    "sc_ln_partials": (C.c_int, [_i32]),
    "sc_gelu_fwd": (C.c_int, [_p, _p, _i32, _i64, _p]),
    "sc_gelu_bwd": (C.c_int, [_p, _p, _p, _i32, _i32, _i32, _p, _p, _p]),
    "sc_cls_score": (C.c_int, [_p, _p, _i32, _i32, _p, _f32, _p, _p]),
    "sc_count_nonfinite": (C.c_int, [_p, _i64, _p, _p]),
    "sc_split_bf16x3": (C.c_int, [_p, _i64, _p, _i32, _p, _i64, _p, _i64, _i64, _i32, _p]),
    "sc_split_f16x2": (C.c_int, [_p, _i64, _p, _i32, _p, _i64, _p, _i64, _i64, _i32, _i32, _p, _p]),
    "sc_residual_layernorm_f16x2": (C.c_int, [_p, _p, _p, _p, _p, _p, _p, _i64, _i32, _p, _p, _i32, _i32, _p]),
    "sc_gemm_x3h_gelu_planes": (C.c_int, [_p, _i64, _p, _i64, _f32, _p, _p, _i64, _p, _i32, _i32, _i32, _p]),
    "sc_gemm_x3h": (C.c_int, [_p, _i64, _p, _i64, _f32, _p, _i64, _i32, _i32, _i32, _i32, _p]),
}

# Entry points that launch device work (counted for the bench's gpu_launches).
LAUNCHING = {n for n in SIGNATURES
             if n not in ("sc_last_error", "sc_version", "sc_kernel_launches", "sc_attn_workspace_bytes",
                          "sc_attn_workspace_bytes_qds", "sc_attn_bwd_workspace_bytes", "sc_ln_partials")}


def kernel_launches() -> int:
    """Kernels launched by the library in this process (the library's own counter)."""
    return int(load().sc_kernel_launches())


class LibraryNotBuiltError(RuntimeError):
    """The CUDA library is missing; there is deliberately no CPU fallback."""


class ScError(RuntimeError):
    def __init__(self, code, message):
        super().__init__(message)
        self.code = code


_lock = threading.Lock()
_lib = None
launch_calls = 0  # number of launching C-ABI calls made by this process


def load():
    """Load (once) and return the ctypes library handle."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryNotBuiltError(
                    f"{LIB_PATH} not found: build it with `python __graft_entry__.py build`"
                )
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    return load().sc_last_error().decode(errors="replace")


def call(name, *args, exc=ValueError):
    """Invoke an entry point; map a non-zero status to an exception.

    ``exc`` is the reference's exception class for SC_ERR_INVALID at this
    call site (AttentionError, BandShapeError, EncoderError ...).
    """
    global launch_calls
    fn = getattr(load(), name)
    rc = fn(*args)
    if name in LAUNCHING:
        launch_calls += 1
    if rc == SC_OK:
        return rc
    msg = last_error()
    if rc in (SC_ERR_INVALID, SC_ERR_NO_VALID_ROW):
        raise exc(msg)
    if rc == SC_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise ScError(rc, msg)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
