"""GPU checks of the encoder-loop kernels against plain PyTorch fp32 references of the same ops."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2312_17649_b200 import _lib

    return _lib


def torch_gelu_erf(x):
    return 0.5 * x * (1.0 + torch.erf(x / math.sqrt(2.0)))


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("cols", [3072, 64, 37])
def test_bias_gelu(lib, dtype, cols):
    g = torch.Generator(device="cuda").manual_seed(0)
    x = (torch.randn((513, cols), device="cuda", generator=g) * 3).to(dtype)
    bias = torch.randn(cols, device="cuda", generator=g)
    ref = torch_gelu_erf(x.float() + bias)
    y = x.clone()
    lib.call("sc_bias_gelu", y.data_ptr(), bias.data_ptr(), 0 if dtype == torch.float32 else 1, 513, cols,
             lib.stream_handle())
    if dtype == torch.float32:
        torch.testing.assert_close(y, ref, atol=2e-6, rtol=1e-6)
    else:
        # bf16 output: one bf16 rounding (<= 2^-8 relative) of the exact-erf value,
        # plus the erf approximation's absolute error (< 3e-7 on erf => < 1e-6 on GELU here)
        excess = (y.float() - ref).abs() - 2 ** -8 * ref.abs()
        assert excess.max().item() <= 2e-6


@pytest.mark.parametrize("ydtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("h", [768, 32, 100, 2048])
def test_residual_layernorm(lib, ydtype, h):
    g = torch.Generator(device="cuda").manual_seed(1)
    rows = 1000
    resid = torch.randn((rows, h), device="cuda", generator=g)
    y = torch.randn((rows, h), device="cuda", generator=g).to(ydtype)
    gamma = torch.randn(h, device="cuda", generator=g)
    beta = torch.randn(h, device="cuda", generator=g)
    ref = torch.nn.functional.layer_norm(resid + y.float(), (h,), gamma, beta, eps=1e-12)
    out = torch.empty_like(resid)
    outh = torch.empty((rows, h), device="cuda", dtype=torch.bfloat16)
    lib.call("sc_residual_layernorm", resid.data_ptr(), y.data_ptr(), 0 if ydtype == torch.float32 else 1, None,
             gamma.data_ptr(), beta.data_ptr(), out.data_ptr(), outh.data_ptr(), rows, h, lib.stream_handle())
    torch.testing.assert_close(out, ref, atol=2e-5, rtol=1e-5)
    torch.testing.assert_close(outh, ref.to(torch.bfloat16), atol=0.02, rtol=0.01)


@pytest.mark.parametrize("h", [96, 768])
def test_embed_and_cls_score(lib, h):
    g = torch.Generator(device="cuda").manual_seed(2)
    V, P, T = 50, 30, 40
    tok = torch.randn((V, h), device="cuda", generator=g)
    pos = torch.randn((P, h), device="cuda", generator=g)
    ids = torch.randint(0, V, (T,), device="cuda", generator=g, dtype=torch.int32)
    tp = torch.cat([torch.arange(15), torch.arange(25)]).int().cuda()
    x = torch.empty((T, h), device="cuda")
    xh = torch.empty((T, h), device="cuda", dtype=torch.bfloat16)
    lib.call("sc_embed", ids.data_ptr(), tp.data_ptr(), tok.data_ptr(), pos.data_ptr(), x.data_ptr(), xh.data_ptr(),
             T, h, lib.stream_handle())
    ref = tok[ids.long()] + pos[tp.long()]
    torch.testing.assert_close(x, ref)
    torch.testing.assert_close(xh, ref.to(torch.bfloat16))
    cu = torch.tensor([0, 15, 40], dtype=torch.int32, device="cuda")
    w = torch.randn(h, device="cuda", generator=g)
    sc = torch.empty(2, device="cuda")
    lib.call("sc_cls_score", x.data_ptr(), cu.data_ptr(), 2, h, w.data_ptr(), 0.5, sc.data_ptr(), lib.stream_handle())
    torch.testing.assert_close(sc, torch.stack([x[0] @ w, x[15] @ w]) + 0.5, atol=1e-4, rtol=1e-5)


def test_kernel_launch_counter(lib):
    n0 = lib.kernel_launches()
    x = torch.zeros(10, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib.call("sc_count_nonfinite", x.data_ptr(), 10, cnt.data_ptr(), lib.stream_handle())
    assert lib.kernel_launches() == n0 + 1
    assert cnt.item() == 0
    x[3] = float("nan")
    lib.call("sc_count_nonfinite", x.data_ptr(), 10, cnt.data_ptr(), lib.stream_handle())
    assert cnt.item() > 0


@pytest.mark.parametrize("rdtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("h", [768, 100, 2048])
def test_residual_layernorm_ex(lib, rdtype, h):
    """bf16 / fp32 residual, each output optional, fused non-finite flag."""
    g = torch.Generator(device="cuda").manual_seed(3)
    rows = 777
    resid = torch.randn((rows, h), device="cuda", generator=g).to(rdtype)
    y = torch.randn((rows, h), device="cuda", generator=g).to(torch.bfloat16)
    gamma = torch.randn(h, device="cuda", generator=g)
    beta = torch.randn(h, device="cuda", generator=g)
    ref = torch.nn.functional.layer_norm(resid.float() + y.float(), (h,), gamma, beta, eps=1e-12)
    rd = 0 if rdtype == torch.float32 else 1
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.empty((rows, h), device="cuda")
    lib.call("sc_residual_layernorm_ex", resid.data_ptr(), rd, y.data_ptr(), 1, None, gamma.data_ptr(),
             beta.data_ptr(), out.data_ptr(), None, bad.data_ptr(), rows, h, lib.stream_handle())
    torch.testing.assert_close(out, ref, atol=2e-5, rtol=1e-5)
    assert bad.item() == 0
    # bf16-only output written in place over a bf16 residual
    if rdtype == torch.bfloat16:
        inplace = resid.clone()
        lib.call("sc_residual_layernorm_ex", inplace.data_ptr(), 1, y.data_ptr(), 1, None, gamma.data_ptr(),
                 beta.data_ptr(), None, inplace.data_ptr(), bad.data_ptr(), rows, h, lib.stream_handle())
        # identical arithmetic to the fp32-output call above: bitwise its bf16 rounding
        torch.testing.assert_close(inplace, out.to(torch.bfloat16), atol=0, rtol=0)
    # a NaN / Inf in one row is counted
    y2 = y.clone()
    y2[5, 3] = float("nan")
    y2[600, h - 1] = float("inf")
    lib.call("sc_residual_layernorm_ex", resid.data_ptr(), rd, y2.data_ptr(), 1, None, gamma.data_ptr(),
             beta.data_ptr(), out.data_ptr(), None, bad.data_ptr(), rows, h, lib.stream_handle())
    torch.cuda.synchronize()
    assert bad.item() >= 2
    with pytest.raises(ValueError):
        lib.call("sc_residual_layernorm_ex", resid.data_ptr(), rd, y.data_ptr(), 1, None, gamma.data_ptr(),
                 beta.data_ptr(), None, None, None, rows, h, lib.stream_handle())


@pytest.mark.parametrize("M,N,K", [(1000, 3072, 768), (128, 256, 64), (37, 512, 192)])
@pytest.mark.parametrize("with_bias", [True, False])
def test_gemm_bias_gelu_vs_torch(lib, M, N, K, with_bias):
    """Fused tcgen05 FFN up-projection: gelu_erf(x W^T + b) vs a plain PyTorch fp32 reference."""
    g = torch.Generator(device="cuda").manual_seed(5)
    x = (torch.randn((M, K), device="cuda", generator=g)).to(torch.bfloat16)
    w = (torch.randn((N, K), device="cuda", generator=g) / math.sqrt(K)).to(torch.bfloat16)
    b = torch.randn(N, device="cuda", generator=g) if with_bias else None
    ref = torch_gelu_erf(x.float() @ w.float().t() + (b if with_bias else 0.0))
    out = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    lib.call("sc_gemm_bias_gelu", x.data_ptr(), K, w.data_ptr(), K, None if b is None else b.data_ptr(),
             out.data_ptr(), N, M, N, K, lib.stream_handle())
    # one bf16 rounding of the output (fp32 accumulation order differs from torch's)
    excess = (out.float() - ref).abs() - 2 ** -8 * ref.abs()
    assert excess.max().item() <= 2e-3
    with pytest.raises(NotImplementedError):
        lib.call("sc_gemm_bias_gelu", x.data_ptr(), K, w.data_ptr(), K, None, out.data_ptr(), N, M, N - 8, K,
                 lib.stream_handle())


def test_gemm_bias_gelu_cta_pair_variant():
    """The opt-in cta_group::2 variant (SC_GEMM_2SM=1) gives the same result as the one-CTA kernel."""
    import subprocess
    import sys
    code = (
        "import math, torch, sys; sys.path.insert(0, '.');"
        "from paper_2312_17649_b200 import _lib;"
        "g = torch.Generator(device='cuda').manual_seed(7);"
        "x = torch.randn((700, 768), device='cuda', generator=g).to(torch.bfloat16);"
        "w = (torch.randn((1024, 768), device='cuda', generator=g) / 28).to(torch.bfloat16);"
        "b = torch.randn(1024, device='cuda', generator=g);"
        "o = torch.empty((700, 1024), device='cuda', dtype=torch.bfloat16);"
        "_lib.call('sc_gemm_bias_gelu', x.data_ptr(), 768, w.data_ptr(), 768, b.data_ptr(), o.data_ptr(), 1024, 700, 1024, 768, _lib.stream_handle());"
        "ref = torch.nn.functional.gelu(x.float() @ w.float().t() + b);"
        "err = ((o.float() - ref).abs() - 2 ** -8 * ref.abs()).max().item();"
        "assert err <= 2e-3, err; print('ok', err)")
    import os
    env = dict(os.environ, SC_GEMM_2SM="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("M,K", [(1000, 768), (37, 3072), (256, 192)])
def test_gemm_residual_layernorm_vs_torch(lib, M, K):
    """Cluster-of-3 fused projection + residual + LayerNorm vs a plain PyTorch fp32 reference."""
    N = 768
    g = torch.Generator(device="cuda").manual_seed(9)
    a = torch.randn((M, K), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((N, K), device="cuda", generator=g) / math.sqrt(K)).to(torch.bfloat16)
    b = torch.randn(N, device="cuda", generator=g) * 0.1
    resid = torch.randn((M, N), device="cuda", generator=g).to(torch.bfloat16)
    gamma = 1 + 0.1 * torch.randn(N, device="cuda", generator=g)
    beta = 0.1 * torch.randn(N, device="cuda", generator=g)
    ref = torch.nn.functional.layer_norm(resid.float() + a.float() @ w.float().t() + b, (N,), gamma, beta, eps=1e-12)
    out = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    out32 = torch.empty((M, N), device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib.call("sc_gemm_residual_layernorm", a.data_ptr(), K, w.data_ptr(), K, b.data_ptr(), resid.data_ptr(), N,
             gamma.data_ptr(), beta.data_ptr(), out.data_ptr(), N, out32.data_ptr(), N, bad.data_ptr(), M, N, K,
             lib.stream_handle())
    torch.testing.assert_close(out32, ref, atol=2e-3, rtol=1e-3)
    torch.testing.assert_close(out.float(), ref, atol=2e-2, rtol=1e-2)
    assert bad.item() == 0
    # bf16-only output, no bias; a NaN in one row is counted
    a2 = a.clone()
    a2[min(5, M - 1), 0] = float("nan")
    lib.call("sc_gemm_residual_layernorm", a2.data_ptr(), K, w.data_ptr(), K, None, resid.data_ptr(), N,
             gamma.data_ptr(), beta.data_ptr(), out.data_ptr(), N, None, N, bad.data_ptr(), M, N, K,
             lib.stream_handle())
    torch.cuda.synchronize()
    assert bad.item() >= 1
    with pytest.raises(NotImplementedError):
        lib.call("sc_gemm_residual_layernorm", a.data_ptr(), K, w.data_ptr(), K, None, resid.data_ptr(), N,
                 gamma.data_ptr(), beta.data_ptr(), out.data_ptr(), N, None, N, None, M, 512, K, lib.stream_handle())


def test_gemm_bias_gelu_pre_dual_output():
    """sc_gemm_bias_gelu_pre: the fused W1 GEMM also storing the pre-activation (fine-tuning)."""
    import paper_2312_17649_b200._lib as L

    torch.manual_seed(3)
    M, N, K = 1000, 512, 192
    a = torch.randn(M, K, device="cuda").bfloat16()
    w = (torch.randn(N, K, device="cuda") * 0.1).bfloat16()
    b = torch.randn(N, device="cuda")
    g = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    f = torch.empty_like(g)
    L.call("sc_gemm_bias_gelu_pre", a.data_ptr(), K, w.data_ptr(), K, b.data_ptr(), g.data_ptr(), N, f.data_ptr(),
           N, M, N, K, L.stream_handle())
    pre = a.float() @ w.float().t() + b
    torch.testing.assert_close(f.float(), pre, rtol=2e-2, atol=2e-2)
    torch.testing.assert_close(g.float(), torch.nn.functional.gelu(pre), rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("bias,gelu", [(False, False), (True, False), (True, True)])
@pytest.mark.parametrize("cols", [768, 3072, 13])
def test_split_bf16x3_planes(bias, gelu, cols):
    """sc_split_bf16x3: planes [p1 | p2 | p0 | p1 | p0]; p0 + p1 + p2 reproduces v = gelu?(x + bias) to
    2^-24 relative, each plane the round-to-nearest bf16 of the remaining residual; the fp32 copy
    matches an fp64 GELU."""
    from paper_2312_17649_b200.encoder import split_planes

    g = torch.Generator(device="cuda").manual_seed(cols)
    x = torch.randn((257, cols), device="cuda", generator=g) * 3
    b = torch.randn(cols, device="cuda", generator=g) if bias else None
    keep = torch.empty_like(x)
    pl = split_planes(x, bias=b, gelu=gelu, keep=keep)
    v = x.double() + (b.double() if bias else 0)
    if gelu:
        v = 0.5 * v * (1 + torch.special.erf(v / math.sqrt(2)))
    p1, p2, p0 = pl[:, :cols].double(), pl[:, cols:2 * cols].double(), pl[:, 2 * cols:3 * cols].double()
    assert torch.equal(pl[:, 2 * cols:3 * cols], keep.to(torch.bfloat16))
    assert torch.equal(pl[:, :cols], (keep - pl[:, 2 * cols:3 * cols].float()).to(torch.bfloat16))
    assert torch.equal(pl[:, 3 * cols:4 * cols], pl[:, :cols]) and torch.equal(pl[:, 4 * cols:], pl[:, 2 * cols:3 * cols])
    rel = ((p0 + p1 + p2 - keep.double()).abs() / keep.double().abs().clamp_min(1e-30)).max().item()
    assert rel <= 2.0 ** -24, rel
    assert (keep.double() - v).abs().max().item() < 1e-5


def test_linear_x6_matches_fp64():
    """_linear_x6 (six split products on the bf16 tensor cores) is at least as accurate as fp32 SGEMM
    (K = 768: one main accumulation; K = 3072: four chunks)."""
    from paper_2312_17649_b200.encoder import _linear_x6, _split_weight_x6, split_planes

    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn((1000, 3072), device="cuda", generator=g)
    w = torch.randn((768, 3072), device="cuda", generator=g) / 55
    exact = a.double() @ w.double().t()
    got = _linear_x6(split_planes(a), _split_weight_x6(w))
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        sg = a @ w.t()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    e6 = (got.double() - exact).abs().max().item()
    es = (sg.double() - exact).abs().max().item()
    print(f"x6 max err {e6:.3e}, sgemm {es:.3e}")
    assert e6 <= es * 1.25, (e6, es)


def test_split_f16x2_planes_and_range_flag():
    """sc_split_f16x2: [h0 | h1] with h0 = fp16_rn(v), h1 = fp16_rn(v - h0) (bias + GELU fused, fp32 kept);
    a value outside fp16 range raises the status flag."""
    from paper_2312_17649_b200.encoder import split_planes_h

    g = torch.Generator(device="cuda").manual_seed(9)
    for cols in (768, 13):
        x = torch.randn((333, cols), device="cuda", generator=g) * 7
        b = torch.randn(cols, device="cuda", generator=g)
        keep = torch.empty_like(x)
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        pl = split_planes_h(x, bias=b, gelu=True, keep=keep, status=st)
        v = torch.nn.functional.gelu((x + b).double())
        h0 = keep.to(torch.float16)
        assert torch.equal(pl[:, :cols], h0)
        assert torch.equal(pl[:, cols:], (keep - h0.float()).to(torch.float16))
        assert (keep.double() - v).abs().max().item() < 1e-4
        assert int(st.item()) == 0
    pl = split_planes_h(x, onehot=True)
    assert torch.equal(pl[:, :cols], x.to(torch.float16)) and torch.equal(pl[:, cols + 8:], (x - x.half().float()).half())
    assert (pl[:, cols] == 1).all() and (pl[:, cols + 1:cols + 8] == 0).all()
    x[5, 3] = 70000.0
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    split_planes_h(x, status=st)
    assert int(st.item()) == 1


@pytest.mark.parametrize("h", [768, 384])
@pytest.mark.parametrize("onehot", [False, True])
def test_residual_layernorm_f16x2_equals_ln_then_split(lib, h, onehot):
    """sc_residual_layernorm_f16x2 = sc_residual_layernorm_ex (fp32) followed by sc_split_f16x2 of its
    output, bit for bit (x_out and planes), and the range / non-finite flags."""
    from paper_2312_17649_b200.encoder import split_planes_h

    g = torch.Generator(device="cuda").manual_seed(h + onehot)
    M = 1031
    r = torch.randn((M, h), device="cuda", generator=g)
    y = torch.randn((M, h), device="cuda", generator=g) * 2
    b, gm, bt = (torch.randn(h, device="cuda", generator=g) for _ in range(3))
    ref = torch.empty_like(r)
    lib.call("sc_residual_layernorm_ex", r.data_ptr(), lib.DTYPE_F32, y.data_ptr(), lib.DTYPE_F32, b.data_ptr(),
             gm.data_ptr(), bt.data_ptr(), ref.data_ptr(), None, None, M, h, lib.stream_handle())
    ref_pl = split_planes_h(ref, onehot=onehot)
    out = torch.empty_like(r)
    pl = torch.empty((M, 2 * h + (8 if onehot else 0)), dtype=torch.float16, device="cuda")
    rng = torch.zeros(1, dtype=torch.int32, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib.call("sc_residual_layernorm_f16x2", r.data_ptr(), y.data_ptr(), b.data_ptr(), gm.data_ptr(), bt.data_ptr(),
             out.data_ptr(), pl.data_ptr(), pl.stride(0), int(onehot), rng.data_ptr(), bad.data_ptr(), M, h,
             lib.stream_handle())
    assert torch.equal(out, ref)
    assert torch.equal(pl, ref_pl)
    assert int(rng.item()) == 0 and int(bad.item()) == 0
    gm2 = gm.clone()
    gm2[7] = 1e6  # an output past fp16 range -> range flag
    lib.call("sc_residual_layernorm_f16x2", r.data_ptr(), y.data_ptr(), b.data_ptr(), gm2.data_ptr(), bt.data_ptr(),
             out.data_ptr(), pl.data_ptr(), pl.stride(0), int(onehot), rng.data_ptr(), bad.data_ptr(), M, h,
             lib.stream_handle())
    assert int(rng.item()) == 1 and int(bad.item()) == 0
    with pytest.raises(Exception):  # hidden outside the vectorised set: unsupported, reported
        lib.call("sc_residual_layernorm_f16x2", r.data_ptr(), y.data_ptr(), b.data_ptr(), gm.data_ptr(),
                 bt.data_ptr(), out.data_ptr(), pl.data_ptr(), pl.stride(0), int(onehot), None, None, M, 100,
                 lib.stream_handle())


def test_gemm_x3h_gelu_planes_matches_unfused(lib):
    """sc_gemm_x3h_gelu_planes (W1 as three fp16 products + bias + erff GELU + split, one tcgen05 GEMM)
    against the unfused f16x3 path (_linear_x3h on cuBLAS, then sc_split_f16x2 with bias + GELU) and
    fp64: the planes reconstruct gelu(x W^T + b) as accurately as the unfused path; ragged M; range flag."""
    from paper_2312_17649_b200.encoder import _linear_x3h, _split_weight_x3h, split_planes_h

    g = torch.Generator(device="cuda").manual_seed(11)
    M, K, N = 1031, 768, 3072
    x = torch.randn((M, K), device="cuda", generator=g)
    w = torch.randn((N, K), device="cuda", generator=g) * 0.03
    b = torch.randn(N, device="cuda", generator=g) * 0.5
    xs = split_planes_h(x)
    w2, sc = _split_weight_x3h(w)
    ref_pl = split_planes_h(_linear_x3h(xs, w2, sc), bias=b, gelu=True)
    out = torch.empty((M, 2 * N), dtype=torch.float16, device="cuda")
    rng = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib.call("sc_gemm_x3h_gelu_planes", xs.data_ptr(), xs.stride(0), w2.data_ptr(), w2.stride(0), float(sc),
             b.data_ptr(), out.data_ptr(), out.stride(0), rng.data_ptr(), M, N, K, lib.stream_handle())
    got = out[:, :N].double() + out[:, N:].double()
    ref = ref_pl[:, :N].double() + ref_pl[:, N:].double()
    pre = x.double() @ w.double().t() + b.double()
    exact = 0.5 * pre * (1 + torch.special.erf(pre / math.sqrt(2)))
    e_got = (got - exact).abs().max().item()
    e_ref = (ref - exact).abs().max().item()
    print(f"fused max err {e_got:.3e}, unfused {e_ref:.3e}, fused vs unfused {(got - ref).abs().max().item():.3e}")
    assert e_got <= 2 * e_ref + 1e-7, (e_got, e_ref)
    assert int(rng.item()) == 0
    big = torch.full((N,), 1e5, device="cuda")
    lib.call("sc_gemm_x3h_gelu_planes", xs.data_ptr(), xs.stride(0), w2.data_ptr(), w2.stride(0), float(sc),
             big.data_ptr(), out.data_ptr(), out.stride(0), rng.data_ptr(), M, N, K, lib.stream_handle())
    assert int(rng.item()) == 1
    with pytest.raises(NotImplementedError):
        lib.call("sc_gemm_x3h_gelu_planes", xs.data_ptr(), xs.stride(0), w2.data_ptr(), w2.stride(0), float(sc),
                 b.data_ptr(), out.data_ptr(), out.stride(0), None, M, 300, K, lib.stream_handle())


@pytest.mark.parametrize("bias", [False, True])
@pytest.mark.parametrize("N", [768, 2304])
def test_gemm_x3h_matches_cublas_path_and_fp64(lib, bias, N):
    """sc_gemm_x3h (the three fp16 products + the bias columns in one tcgen05 accumulation, fp32 out) vs
    _linear_x3h on cuBLAS and fp64 at K = 768: as accurate as the cuBLAS form; ragged M."""
    from paper_2312_17649_b200.encoder import _linear_x3h, _linear_x3h_tc, _split_weight_x3h, split_planes_h

    g = torch.Generator(device="cuda").manual_seed(N + bias)
    M, K = 1037, 768
    x = torch.randn((M, K), device="cuda", generator=g)
    w = torch.randn((N, K), device="cuda", generator=g) * 0.03
    b = torch.randn(N, device="cuda", generator=g) if bias else None
    xs = split_planes_h(x, onehot=bias)
    w2, sc = _split_weight_x3h(w, b)
    got = _linear_x3h_tc(xs, w2, sc)
    ref = _linear_x3h(xs, w2, sc)
    exact = x.double() @ w.double().t() + (b.double() if bias else 0)
    e_got = (got.double() - exact).abs().max().item()
    e_ref = (ref.double() - exact).abs().max().item()
    print(f"x3h tc max err {e_got:.3e}, cuBLAS form {e_ref:.3e}")
    assert e_got <= 1.5 * e_ref + 1e-7, (e_got, e_ref)


def test_linear_x3h_matches_fp64():
    """_linear_x3h (three split-fp16 products, weights scaled by 2^e) is about as accurate as fp32 SGEMM
    (K = 768: one main accumulation; K = 3072: four chunks); bias folded into the first GEMM."""
    from paper_2312_17649_b200.encoder import _linear_x3h, _split_weight_x3h, split_planes_h

    g = torch.Generator(device="cuda").manual_seed(5)
    for K in (768, 3072):
        a = torch.randn((1000, K), device="cuda", generator=g)
        w = torch.randn((768, K), device="cuda", generator=g) * 0.02
        b = torch.randn(768, device="cuda", generator=g)
        exact = a.double() @ w.double().t() + b.double()
        w2, s = _split_weight_x3h(w, b)
        got = _linear_x3h(split_planes_h(a, onehot=True), w2, s)
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        try:
            sg = a @ w.t() + b
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev
        e3 = (got.double() - exact).abs().max().item()
        es = (sg.double() - exact).abs().max().item()
        print(f"K={K} x3h max err {e3:.3e}, sgemm {es:.3e}")
        assert e3 <= es * 2.0, (K, e3, es)
