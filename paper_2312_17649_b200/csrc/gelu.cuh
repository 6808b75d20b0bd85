// Exact-erf GELU for the bf16 path (R/encoder.py:258-259), shared by the
// elementwise pass (encoder_ops.cu) and the fused W1 GEMM epilogue (gemm_gelu.cu).
#pragma once
#include "common.cuh"

namespace sc {

// erf for the bf16 path: Abramowitz & Stegun 7.1.26, |abs error| <= 1.5e-7
// (+ ~1e-7 from the approximate rcp/ex2), far below bf16 output resolution
// (2^-9 relative); one MUFU.RCP + one MUFU.EX2 + 8 FMA instead of erff's
// two-branch evaluation.  The fp32 parity path keeps erff.
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float gelu_bf16path(float x) {
  const float z = x * 0.70710678118654752440f;
  const float a = fabsf(z);
  const float t = rcp_approx(fmaf(0.3275911f, a, 1.f));
  float p = fmaf(1.061405429f, t, -1.453152027f);
  p = fmaf(p, t, 1.421413741f);
  p = fmaf(p, t, -0.284496736f);
  p = fmaf(p, t, 0.254829592f);
  p *= t;
  const float e = ex2_approx(-a * a * 1.4426950408889634f);
  const float erf_abs = fmaf(-p, e, 1.f);
  const float half_x = 0.5f * x;
  return fmaf(half_x, copysignf(erf_abs, z), half_x);
}

// Same formula on pairs with Blackwell's packed FP32 pipe (FFMA2/FMUL2): halves
// the FP instruction count of the issue-bound bf16 GELU pass.
__device__ __forceinline__ float2 gelu2_bf16path(float2 x) {
  const float2 z = __fmul2_rn(x, make_float2(0.70710678118654752440f, 0.70710678118654752440f));
  const float2 a = make_float2(fabsf(z.x), fabsf(z.y));
  const float2 d = __ffma2_rn(a, make_float2(0.3275911f, 0.3275911f), make_float2(1.f, 1.f));
  const float2 t = make_float2(rcp_approx(d.x), rcp_approx(d.y));
  float2 p = __ffma2_rn(make_float2(1.061405429f, 1.061405429f), t, make_float2(-1.453152027f, -1.453152027f));
  p = __ffma2_rn(p, t, make_float2(1.421413741f, 1.421413741f));
  p = __ffma2_rn(p, t, make_float2(-0.284496736f, -0.284496736f));
  p = __ffma2_rn(p, t, make_float2(0.254829592f, 0.254829592f));
  p = __fmul2_rn(p, t);
  const float2 g = __fmul2_rn(__fmul2_rn(a, a), make_float2(-1.4426950408889634f, -1.4426950408889634f));
  const float2 ne = make_float2(-ex2_approx(g.x), -ex2_approx(g.y));
  const float2 erf_abs = __ffma2_rn(p, ne, make_float2(1.f, 1.f));
  const float2 h = __fmul2_rn(x, make_float2(0.5f, 0.5f));
  return __ffma2_rn(h, make_float2(copysignf(erf_abs.x, x.x), copysignf(erf_abs.y, x.y)), h);
}

// GELU on pairs with one MUFU op per element: erfc(a) = exp(-a^2) R(a), R the
// degree-10 polynomial fit of erfcx on [0, 4] (|GELU error| <= 2e-6, far below
// bf16 resolution; a is clamped at 4, where exp(-a^2) < 1.2e-7).  Used by the
// fused GEMM epilogue, whose MUFU pipe the rcp of A&S 7.1.26 would saturate.
__device__ __forceinline__ float2 gelu2_bf16path_1mufu(float2 x) {
  const float2 z = __fmul2_rn(x, make_float2(0.70710678118654752440f, 0.70710678118654752440f));
  const float2 a = make_float2(fminf(fabsf(z.x), 4.f), fminf(fabsf(z.y), 4.f));
  float2 p = __ffma2_rn(make_float2(1.1544991139089689e-05f, 1.1544991139089689e-05f), a,
                        make_float2(-0.00027032289654016495f, -0.00027032289654016495f));
  p = __ffma2_rn(p, a, make_float2(0.0028087019454687834f, 0.0028087019454687834f));
  p = __ffma2_rn(p, a, make_float2(-0.017178276553750038f, -0.017178276553750038f));
  p = __ffma2_rn(p, a, make_float2(0.06945336610078812f, 0.06945336610078812f));
  p = __ffma2_rn(p, a, make_float2(-0.19890554249286652f, -0.19890554249286652f));
  p = __ffma2_rn(p, a, make_float2(0.4261739253997803f, 0.4261739253997803f));
  p = __ffma2_rn(p, a, make_float2(-0.7184767723083496f, -0.7184767723083496f));
  p = __ffma2_rn(p, a, make_float2(0.9914032816886902f, 0.9914032816886902f));
  p = __ffma2_rn(p, a, make_float2(-1.1274118423461914f, -1.1274118423461914f));
  p = __ffma2_rn(p, a, make_float2(0.9999727010726929f, 0.9999727010726929f));
  // half_erfc = 0.5 * exp(-z^2) * R(a)   (exp(-z^2) = ex2(-z^2 * log2 e))
  const float2 zz = __fmul2_rn(__fmul2_rn(z, z), make_float2(-1.4426950408889634f, -1.4426950408889634f));
  const float2 he = __fmul2_rn(__fmul2_rn(p, make_float2(ex2_approx(zz.x), ex2_approx(zz.y))), make_float2(0.5f, 0.5f));
  // x >= 0: x (1 - he);  x < 0: x he
  return make_float2(x.x >= 0.f ? fmaf(-x.x, he.x, x.x) : x.x * he.x, x.y >= 0.f ? fmaf(-x.y, he.y, x.y) : x.y * he.y);
}

}  // namespace sc
