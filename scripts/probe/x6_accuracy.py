"""Probe: accuracy / speed of split-bf16 fp32 GEMM emulations vs cuBLAS SGEMM (fp64 truth)."""
import sys, os, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2312_17649_b200.encoder import split_planes, _split_weight_x6

torch.backends.cuda.matmul.allow_tf32 = False
dev = "cuda"
F32 = torch.float32

def planes3(x):
    x0 = x.bfloat16(); r = x - x0.float(); x1 = r.bfloat16(); x2 = (r - x1.float()).bfloat16()
    return x0, x1, x2

def mm(a, b):
    return torch.mm(a, b.t(), out_dtype=F32)

def v_cur(A, W):  # 3 GEMMs
    K = A.shape[1]
    a3 = split_planes(A); w6 = _split_weight_x6(W)
    def run():
        c = torch.mm(a3, w6[:, :3*K].t(), out_dtype=F32)
        c = torch.addmm(c, a3[:, :2*K], w6[:, 3*K:5*K].t(), out_dtype=F32)
        return torch.addmm(c, a3[:, :K], w6[:, 5*K:].t(), out_dtype=F32)
    return run

def v_main_corr(A, W, chunk=None):
    K = A.shape[1]
    a0, a1, a2 = planes3(A); w0, w1, w2 = planes3(W)
    a5 = torch.cat([a1, a2, a0, a1, a0], 1).contiguous()
    w5 = torch.cat([w0, w0, w1, w1, w2], 1).contiguous()
    a0v = a5[:, 2*K:3*K]
    w0v = w5[:, :K]
    def run():
        c = torch.mm(a5, w5.t(), out_dtype=F32)
        ck = chunk or K
        for k0 in range(0, K, ck):
            c = torch.addmm(c, a0v[:, k0:k0+ck], w0v[:, k0:k0+ck].t(), out_dtype=F32)
        return c
    return run

def v_tf32x3(A, W):
    def tf(x):  # round-to-nearest to tf32 (10 explicit mantissa bits)
        i = x.view(torch.int32)
        i = (i + 0x1000) & ~0x1FFF
        return i.view(F32)
    ah = tf(A); al = A - ah; wh = tf(W); wl = W - wh
    def run():
        torch.backends.cuda.matmul.allow_tf32 = True
        c = ah @ wh.t(); c += ah @ wl.t(); c += al @ wh.t()
        torch.backends.cuda.matmul.allow_tf32 = False
        return c
    return run

def v_sgemm(A, W):
    return lambda: A @ W.t()

def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

g = torch.Generator(device=dev).manual_seed(0)
for (M, N, K) in ((32792, 768, 3072), (32792, 3072, 768), (32792, 2304, 768)):
    A = torch.randn((M, K), device=dev, generator=g)
    W = torch.randn((N, K), device=dev, generator=g) / (K ** 0.5)
    # truth on a row subset in fp64
    rows = torch.arange(0, M, 37, device=dev)
    exact = A[rows].double() @ W.double().t()
    res = {}
    for name, mk in (("sgemm", v_sgemm), ("x6_3gemm", v_cur), ("x6_main_corr", v_main_corr),
                     ("x6_main_corr_chunk256", lambda a, w: v_main_corr(a, w, 256)), ("tf32x3", v_tf32x3)):
        fn = mk(A, W)
        out = fn()
        err = (out[rows].double() - exact).abs()
        ms = timeit(fn)
        print(f"M{M} N{N} K{K} {name:24s} max {err.max().item():.3e} mean {err.mean().item():.3e} bias {(out[rows].double()-exact).mean().item():+.2e} {ms:.3f} ms", flush=True)
