"""Fused Wo/W2 projection + residual + LayerNorm (cluster of 3) vs cuBLAS + the LayerNorm pass, bench shapes."""
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
    M, N = 64 * 4099, 768
    st = _lib.stream_handle()
    for K in (768, 3072):
        a = torch.randn((M, K), device="cuda").to(torch.bfloat16)
        w = (torch.randn((N, K), device="cuda") / K ** 0.5).to(torch.bfloat16)
        b = torch.randn(N, device="cuda") * 0.1
        bh = b.to(torch.bfloat16)
        resid = torch.randn((M, N), device="cuda").to(torch.bfloat16)
        gamma, beta = torch.ones(N, device="cuda"), torch.zeros(N, device="cuda")
        out = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)

        def cublas():
            y = F.linear(a, w, bh)
            _lib.call("sc_residual_layernorm_ex", resid.data_ptr(), 1, y.data_ptr(), 1, None, gamma.data_ptr(),
                      beta.data_ptr(), None, out.data_ptr(), None, M, N, st)

        def fused():
            _lib.call("sc_gemm_residual_layernorm", a.data_ptr(), K, w.data_ptr(), K, b.data_ptr(), resid.data_ptr(),
                      N, gamma.data_ptr(), beta.data_ptr(), out.data_ptr(), N, None, N, None, M, N, K, st)

        flops = 2.0 * M * N * K
        lin = timeit(lambda: F.linear(a, w, bh))
        t_c, t_f = timeit(cublas), timeit(fused)
        print(f"K={K}: cuBLAS linear {lin:.3f} ms ({flops / lin / 1e9:.0f} TFLOP/s); cuBLAS + LN pass {t_c:.3f} ms; "
              f"fused cluster-3 {t_f:.3f} ms ({flops / t_f / 1e9:.0f} TFLOP/s)", flush=True)


if __name__ == "__main__":
    main()
