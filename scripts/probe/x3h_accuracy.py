"""Probe: fp16x3 (h0 g0 + h0 g1 + h1 g0) fp32-GEMM emulation vs split-bf16x6 and cuBLAS SGEMM (fp64 truth)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2312_17649_b200.encoder import split_planes, _split_weight_x6, _linear_x6

torch.backends.cuda.matmul.allow_tf32 = False
dev, F32 = "cuda", torch.float32

def h2(x):
    h0 = x.half(); h1 = (x - h0.float()).half()
    return h0, h1

def v_x3h(A, W, chunk=768, scale=1.0):
    K = A.shape[1]
    a0, a1 = h2(A * scale); w0, w1 = h2(W)
    a2 = torch.cat([a0, a1], 1).contiguous(); w2 = torch.cat([w1, w0], 1).contiguous()
    def run():
        c = torch.mm(a2, w2.t(), out_dtype=F32)
        for k0 in range(0, K, chunk):
            c = torch.addmm(c, a0[:, k0:k0 + chunk], w0[:, k0:k0 + chunk].t(), out_dtype=F32)
        return c / scale if scale != 1.0 else c
    return run

def v_x3h_ws(A, W, chunk=768):  # weights scaled by 2^e (max |W'| <= 2^14), output scaled back in the epilogue
    K = A.shape[1]
    e = int(torch.floor(torch.log2(16384.0 / W.abs().max())).item())
    a0, a1 = h2(A); w0, w1 = h2(W * 2.0 ** e)
    a2 = torch.cat([a0, a1], 1).contiguous(); w2 = torch.cat([w1, w0], 1).contiguous()
    s = 2.0 ** -e
    def run():
        c = torch.mm(a2, w2.t(), out_dtype=F32).mul_(s)
        for k0 in range(0, K, chunk):
            c = torch.addmm(c, a0[:, k0:k0 + chunk], w0[:, k0:k0 + chunk].t(), out_dtype=F32, alpha=s)
        return c
    return run

def v_x3h_one(A, W):  # all three products in one K' = 3K accumulation
    a0, a1 = h2(A); w0, w1 = h2(W)
    a3 = torch.cat([a0, a0, a1], 1).contiguous(); w3 = torch.cat([w0, w1, w0], 1).contiguous()
    return lambda: torch.mm(a3, w3.t(), out_dtype=F32)

def v_x6(A, W):
    p = split_planes(A); w5 = _split_weight_x6(W)
    return lambda: _linear_x6(p, w5)

def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

g = torch.Generator(device=dev).manual_seed(0)
for (M, N, K, amp) in ((131168, 768, 3072, 1.0), (131168, 3072, 768, 1.0), (131168, 2304, 768, 1.0), (131168, 768, 768, 30.0)):
    A = torch.randn((M, K), device=dev, generator=g) * amp
    W = torch.randn((N, K), device=dev, generator=g) * 0.02
    rows = torch.arange(0, M, 97, device=dev)
    exact = A[rows].double() @ W.double().t()
    for name, fn in (("sgemm", lambda: A @ W.t()), ("x6", v_x6(A, W)), ("x3h", v_x3h(A, W)),
                     ("x3h_chunk256", v_x3h(A, W, 256)), ("x3h_ws", v_x3h_ws(A, W)), ("x3h_ws384", v_x3h_ws(A, W, 384)), ("x3h_one", v_x3h_one(A, W))):
        out = fn()
        err = (out[rows].double() - exact).abs()
        rel = err.max().item() / exact.abs().max().item()
        print(f"M{M} N{N} K{K} amp{amp:g} {name:14s} max {err.max().item():.3e} (rel {rel:.1e}) mean {err.mean().item():.3e} "
              f"{timeit(fn):.3f} ms", flush=True)
