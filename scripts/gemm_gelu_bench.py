"""Fused tcgen05 W1 GEMM + bias + erf-GELU vs cuBLAS (F.linear) + the separate GELU pass, bench shape."""
import os
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_17649_b200 import _lib  # noqa: E402


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    M, N, K = 64 * 4099, 3072, 768
    x = torch.randn((M, K), device="cuda").to(torch.bfloat16)
    w = (torch.randn((N, K), device="cuda") / K ** 0.5).to(torch.bfloat16)
    b = torch.randn(N, device="cuda") * 0.1
    bh = b.to(torch.bfloat16)
    out = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    st = _lib.stream_handle()

    def cublas():
        f = F.linear(x, w, bh)
        _lib.call("sc_bias_gelu", f.data_ptr(), None, _lib.DTYPE_BF16, M, N, st)

    def fused():
        _lib.call("sc_gemm_bias_gelu", x.data_ptr(), K, w.data_ptr(), K, b.data_ptr(), out.data_ptr(), N, M, N, K, st)

    flops = 2.0 * M * N * K
    t_c, t_f = timeit(cublas), timeit(fused)
    lin = timeit(lambda: F.linear(x, w, bh))
    print(f"cuBLAS linear alone {lin:.3f} ms ({flops / lin / 1e9:.0f} TFLOP/s); cuBLAS + GELU pass {t_c:.3f} ms; "
          f"fused tcgen05 {t_f:.3f} ms ({flops / t_f / 1e9:.0f} TFLOP/s)")
    ref = F.gelu(F.linear(x, w, bh).float(), approximate="none")
    fused()
    torch.cuda.synchronize()
    print("max |fused - ref|", (out.float() - ref).abs().max().item())


if __name__ == "__main__":
    main()
