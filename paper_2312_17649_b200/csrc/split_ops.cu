// fp32 GEMM operands as bf16 planes, for the ranking-exact fp32 mode.
//
// x = p0 + p1 + p2 with p0 = bf16_rn(x), p1 = bf16_rn(x - p0), p2 = bf16_rn(x - p0 - p1):
// 24 significant bits, |x - p0 - p1 - p2| <= 2^-27 |x|.  A product x*w is then
// sum_{i+j<=2} p_i(x) q_j(w) (six bf16 tensor-core products, fp32 accumulation;
// the dropped terms are <= 2^-27 relative), i.e. the reference's fp32 GEMMs
// (R/encoder.py:322-324, :345, :350, :352) on the bf16 tensor pipe.
//
// Layout per row: [p1 | p2 | p0 | p1 | p0] (five `cols`-wide planes).  The
// whole row times [q0 | q0 | q1 | q1 | q2] is the sum of the five correction
// products (magnitude 2^-8 of the result: their accumulation error is
// negligible); the main product p0 q0 is a separate GEMM on the middle plane,
// split over K so that no tensor-core accumulation runs long (the tensor
// pipe's fp32 accumulation is less exact than an FFMA chain; partial products
// are summed in the RN fp32 GEMM epilogue instead).  See encoder.py _linear_x6.
//
// Producers fuse the split into their pass: the optional bias and exact-erf
// GELU (R/encoder.py:258-259, erff as the fp32 path) are applied first and the
// fp32 result can be kept as well (y, may alias x).
#include <cuda_fp16.h>

#include "common.cuh"

namespace sc {

__device__ __forceinline__ void split3(float v, __nv_bfloat16& a, __nv_bfloat16& b, __nv_bfloat16& c) {
  a = __float2bfloat16_rn(v);
  const float r1 = v - __bfloat162float(a);  // exact in fp32
  b = __float2bfloat16_rn(r1);
  c = __float2bfloat16_rn(r1 - __bfloat162float(b));
}

__device__ __forceinline__ uint2 pack4(__nv_bfloat16 a, __nv_bfloat16 b, __nv_bfloat16 c, __nv_bfloat16 d) {
  __nv_bfloat162 lo = __halves2bfloat162(a, b), hi = __halves2bfloat162(c, d);
  return make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
}

// One float4 per thread-iteration (cols % 4 == 0, 16-byte aligned rows); rows walked last-to-first
// (the producing GEMM's most recent output is still in L2).
template <bool kBias, bool kGelu>
__global__ void __launch_bounds__(256) split3_vec_kernel(const float* __restrict__ x, int64_t ldx,
                                                         const float* __restrict__ bias, float* __restrict__ y,
                                                         int64_t ldy, __nv_bfloat16* __restrict__ p, int64_t ldp,
                                                         int64_t rows, int cols) {
  const int c4 = cols >> 2;
  const int64_t n = rows * c4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t j = n - 1 - i;
    const int64_t r = j / c4;
    const int c = (int)(j - r * c4) * 4;
    float4 v = *reinterpret_cast<const float4*>(x + r * ldx + c);
    if (kBias) {
      const float4 b = __ldg(reinterpret_cast<const float4*>(bias + c));
      v.x += b.x, v.y += b.y, v.z += b.z, v.w += b.w;
    }
    if (kGelu) {
      v.x = 0.5f * v.x * (1.f + erff(v.x * 0.70710678118654752440f));
      v.y = 0.5f * v.y * (1.f + erff(v.y * 0.70710678118654752440f));
      v.z = 0.5f * v.z * (1.f + erff(v.z * 0.70710678118654752440f));
      v.w = 0.5f * v.w * (1.f + erff(v.w * 0.70710678118654752440f));
    }
    if (y) *reinterpret_cast<float4*>(y + r * ldy + c) = v;
    __nv_bfloat16 a[4], b[4], d[4];
    split3(v.x, a[0], b[0], d[0]);
    split3(v.y, a[1], b[1], d[1]);
    split3(v.z, a[2], b[2], d[2]);
    split3(v.w, a[3], b[3], d[3]);
    __nv_bfloat16* pr = p + r * ldp + c;
    const uint2 v0 = pack4(a[0], a[1], a[2], a[3]), v1 = pack4(b[0], b[1], b[2], b[3]);
    *reinterpret_cast<uint2*>(pr) = v1;
    *reinterpret_cast<uint2*>(pr + cols) = pack4(d[0], d[1], d[2], d[3]);
    *reinterpret_cast<uint2*>(pr + 2 * cols) = v0;
    *reinterpret_cast<uint2*>(pr + 3 * cols) = v1;
    *reinterpret_cast<uint2*>(pr + 4 * cols) = v0;
  }
}

template <bool kBias, bool kGelu>
__global__ void split3_kernel(const float* __restrict__ x, int64_t ldx, const float* __restrict__ bias,
                              float* __restrict__ y, int64_t ldy, __nv_bfloat16* __restrict__ p, int64_t ldp,
                              int64_t rows, int cols) {
  const int64_t n = rows * cols;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t r = i / cols;
    const int c = (int)(i - r * cols);
    float v = x[r * ldx + c];
    if (kBias) v += __ldg(bias + c);
    if (kGelu) v = 0.5f * v * (1.f + erff(v * 0.70710678118654752440f));
    if (y) y[r * ldy + c] = v;
    __nv_bfloat16* pr = p + r * ldp + c;
    __nv_bfloat16 a, b, d;
    split3(v, a, b, d);
    pr[0] = b, pr[cols] = d, pr[2 * cols] = a, pr[3 * cols] = b, pr[4 * cols] = a;
  }
}

template <bool kBias, bool kGelu>
static void launch_split(bool vec, const float* x, int64_t ldx, const float* bias, float* y, int64_t ldy,
                         __nv_bfloat16* p, int64_t ldp, int64_t rows, int cols, cudaStream_t st) {
  const int64_t work = vec ? rows * (cols / 4) : rows * cols;
  int64_t blocks = (work + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (vec)
    split3_vec_kernel<kBias, kGelu><<<(unsigned)blocks, 256, 0, st>>>(x, ldx, bias, y, ldy, p, ldp, rows, cols);
  else
    split3_kernel<kBias, kGelu><<<(unsigned)blocks, 256, 0, st>>>(x, ldx, bias, y, ldy, p, ldp, rows, cols);
}


// ---- fp16 pair split (CrossEncoder(fp32_gemm="f16x3")) ---------------------
// v = h0 + h1 + O(2^-22 v) with h0 = fp16_rn(v), h1 = fp16_rn(v - h0): planes row = [h0 | h1].
// A product v*w is h0 g0 + (h0 g1 + h1 g0) + O(2^-22): three fp16 tensor-core products, half the
// work of the bf16 six-product form.  fp16's range (|v| < 65504) is checked: an out-of-range value
// sets *status (the encoder then raises, no silent inf).
template <bool kBias, bool kGelu>
__device__ __forceinline__ bool split2h_one(float4 v, const float* __restrict__ bias, float* __restrict__ y, int64_t ldy,
                                            __half* __restrict__ p, int64_t ldp, uint32_t r, int c, int cols, int h1_off,
                                            int onehot) {
  if (kBias) {
    const float4 b = __ldg(reinterpret_cast<const float4*>(bias + c));
    v.x += b.x, v.y += b.y, v.z += b.z, v.w += b.w;
  }
  if (kGelu) {
    v.x = 0.5f * v.x * (1.f + erff(v.x * 0.70710678118654752440f));
    v.y = 0.5f * v.y * (1.f + erff(v.y * 0.70710678118654752440f));
    v.z = 0.5f * v.z * (1.f + erff(v.z * 0.70710678118654752440f));
    v.w = 0.5f * v.w * (1.f + erff(v.w * 0.70710678118654752440f));
  }
  if (y) *reinterpret_cast<float4*>(y + (int64_t)r * ldy + c) = v;
  const __half2 a01 = __floats2half2_rn(v.x, v.y), a23 = __floats2half2_rn(v.z, v.w);
  const float2 f01 = __half22float2(a01), f23 = __half22float2(a23);
  const __half2 b01 = __floats2half2_rn(v.x - f01.x, v.y - f01.y), b23 = __floats2half2_rn(v.z - f23.x, v.w - f23.y);
  __half* pr = p + (int64_t)r * ldp + c;
  uint2 u;
  u.x = *reinterpret_cast<const uint32_t*>(&a01), u.y = *reinterpret_cast<const uint32_t*>(&a23);
  *reinterpret_cast<uint2*>(pr) = u;
  u.x = *reinterpret_cast<const uint32_t*>(&b01), u.y = *reinterpret_cast<const uint32_t*>(&b23);
  *reinterpret_cast<uint2*>(pr + h1_off) = u;
  if (onehot && c == 0) *reinterpret_cast<uint4*>(p + (int64_t)r * ldp + cols) = make_uint4(0x3c00u, 0u, 0u, 0u);  // [1, 0 x 7]
  return !(fabsf(v.x) < 65504.f && fabsf(v.y) < 65504.f && fabsf(v.z) < 65504.f && fabsf(v.w) < 65504.f);
}

// float4 items walked last-to-first (the producing GEMM's most recent output is still in L2), U
// loads in flight per thread before any math (one at a time left the pass at ~55-70% of HBM),
// 32-bit index arithmetic (rows * cols / 4 < 2^32; the caller falls back otherwise).
template <bool kBias, bool kGelu, int U>
__global__ void __launch_bounds__(256, 4) split2h_vec_kernel(const float* __restrict__ x, int64_t ldx,
                                                          const float* __restrict__ bias, float* __restrict__ y,
                                                          int64_t ldy, __half* __restrict__ p, int64_t ldp,
                                                          int64_t rows, int cols, int h1_off, int onehot,
                                                          int32_t* __restrict__ status) {
  const uint32_t c4 = (uint32_t)cols >> 2;
  const uint32_t n = (uint32_t)(rows * c4);
  const uint32_t stride = gridDim.x * blockDim.x;
  bool bad = false;
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  for (; i < n; i += U * stride) {
    float4 v[U];
    uint32_t rr[U];
    int cc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t k = i + u * stride;
      if (k < n) {
        const uint32_t j = n - 1 - k;
        rr[u] = j / c4;
        cc[u] = (int)(j - rr[u] * c4) * 4;
        v[u] = __ldcs(reinterpret_cast<const float4*>(x + (int64_t)rr[u] * ldx + cc[u]));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < n)
        bad |= split2h_one<kBias, kGelu>(v[u], bias, y, ldy, p, ldp, rr[u], cc[u], cols, h1_off, onehot);
  }
  if (bad && status) atomicExch(status, 1);
}

template <bool kBias, bool kGelu>
__global__ void split2h_kernel(const float* __restrict__ x, int64_t ldx, const float* __restrict__ bias,
                               float* __restrict__ y, int64_t ldy, __half* __restrict__ p, int64_t ldp, int64_t rows,
                               int cols, int h1_off, int onehot, int32_t* __restrict__ status) {
  const int64_t n = rows * cols;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t r = i / cols;
    const int c = (int)(i - r * cols);
    float v = x[r * ldx + c];
    if (kBias) v += __ldg(bias + c);
    if (kGelu) v = 0.5f * v * (1.f + erff(v * 0.70710678118654752440f));
    if (y) y[r * ldy + c] = v;
    bad |= !(fabsf(v) < 65504.f);
    const __half a = __float2half_rn(v);
    p[r * ldp + c] = a;
    p[r * ldp + h1_off + c] = __float2half_rn(v - __half2float(a));
    if (onehot && c < 8) p[r * ldp + cols + c] = __float2half_rn(c == 0 ? 1.f : 0.f);
  }
  if (bad && status) atomicExch(status, 1);
}

template <bool kBias, bool kGelu>
static void launch_split2h(bool vec, const float* x, int64_t ldx, const float* bias, float* y, int64_t ldy, __half* p,
                           int64_t ldp, int64_t rows, int cols, int h1_off, int onehot, int32_t* status,
                           cudaStream_t st) {
  vec = vec && rows * (cols / 4) < (int64_t)UINT32_MAX;
  if (vec) {
    // U float4 loads in flight per thread; one resident wave of CTAs (occupancy API).  The GELU form
    // is as much erff arithmetic as memory traffic: SC_SPLIT_GELU_U (measurement) picks its U.
    static int ug = -1;
    if (ug < 0) ug = getenv("SC_SPLIT_GELU_U") ? atoi(getenv("SC_SPLIT_GELU_U")) : 4;  // U = 1 / 2 / 4: 9.8 / 10.2 / 9.6 ms per 12 layers (erff-bound)
    const int U = kGelu ? ug : 4;
    auto kern = U == 1 ? split2h_vec_kernel<kBias, kGelu, 1>
              : U == 2 ? split2h_vec_kernel<kBias, kGelu, 2> : split2h_vec_kernel<kBias, kGelu, 4>;
    static int occ[3] = {0, 0, 0};
    const int ui = U == 1 ? 0 : (U == 2 ? 1 : 2);
    if (!occ[ui]) {
      int dev = 0, sms = 148, per = 4;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, 0);
      occ[ui] = sms * (per > 0 ? per : 1);
    }
    const int64_t work = (rows * (cols / 4) + U - 1) / U;
    int64_t blocks = (work + 255) / 256;
    if (blocks > occ[ui]) blocks = occ[ui];
    kern<<<(unsigned)blocks, 256, 0, st>>>(x, ldx, bias, y, ldy, p, ldp, rows, cols, h1_off, onehot, status);
    return;
  }
  int64_t blocks = (rows * cols + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  {
    split2h_kernel<kBias, kGelu><<<(unsigned)blocks, 256, 0, st>>>(x, ldx, bias, y, ldy, p, ldp, rows, cols, h1_off,
                                                                   onehot, status);
  }
}

}  // namespace sc

using namespace sc;

extern "C" int sc_split_bf16x3(const float* x, int64_t ldx, const float* bias, int32_t gelu, float* y, int64_t ldy,
                               void* planes, int64_t ldp, int64_t rows, int32_t cols, void* stream) {
  SC_CHECK_ARG(x && planes, "sc_split_bf16x3: null pointer");
  SC_CHECK_ARG(rows >= 0 && cols >= 1 && ldx >= cols && ldp >= 5LL * cols && (!y || ldy >= cols),
               "sc_split_bf16x3: bad shape");
  if (rows == 0) return SC_OK;
  const bool vec = cols % 4 == 0 && ldx % 4 == 0 && ldp % 4 == 0 && (!y || ldy % 4 == 0) &&
                   !(((uintptr_t)x | (uintptr_t)y | (uintptr_t)bias) & 15) && !((uintptr_t)planes & 7);
  cudaStream_t st = (cudaStream_t)stream;
  __nv_bfloat16* p = (__nv_bfloat16*)planes;
  if (bias && gelu)
    launch_split<true, true>(vec, x, ldx, bias, y, ldy, p, ldp, rows, cols, st);
  else if (bias)
    launch_split<true, false>(vec, x, ldx, bias, y, ldy, p, ldp, rows, cols, st);
  else if (gelu)
    launch_split<false, true>(vec, x, ldx, bias, y, ldy, p, ldp, rows, cols, st);
  else
    launch_split<false, false>(vec, x, ldx, bias, y, ldy, p, ldp, rows, cols, st);
  SC_CHECK_LAUNCH("split3_kernel");
  return SC_OK;
}

extern "C" int sc_split_f16x2(const float* x, int64_t ldx, const float* bias, int32_t gelu, float* y, int64_t ldy,
                              void* planes, int64_t ldp, int64_t rows, int32_t cols, int32_t onehot, int32_t* status,
                              void* stream) {
  SC_CHECK_ARG(x && planes, "sc_split_f16x2: null pointer");
  const int h1_off = cols + (onehot ? 8 : 0);
  SC_CHECK_ARG(rows >= 0 && cols >= 1 && ldx >= cols && ldp >= (int64_t)h1_off + cols && (!y || ldy >= cols),
               "sc_split_f16x2: bad shape");
  if (rows == 0) return SC_OK;
  const bool vec = cols % 4 == 0 && ldx % 4 == 0 && ldp % 8 == 0 && (!y || ldy % 4 == 0) &&
                   !(((uintptr_t)x | (uintptr_t)y | (uintptr_t)bias) & 15) && !((uintptr_t)planes & 15);
  cudaStream_t st = (cudaStream_t)stream;
  __half* p = (__half*)planes;
  const int oh = onehot ? 1 : 0;
  if (bias && gelu)
    launch_split2h<true, true>(vec, x, ldx, bias, y, ldy, p, ldp, rows, cols, h1_off, oh, status, st);
  else if (bias)
    launch_split2h<true, false>(vec, x, ldx, bias, y, ldy, p, ldp, rows, cols, h1_off, oh, status, st);
  else if (gelu)
    launch_split2h<false, true>(vec, x, ldx, bias, y, ldy, p, ldp, rows, cols, h1_off, oh, status, st);
  else
    launch_split2h<false, false>(vec, x, ldx, bias, y, ldy, p, ldp, rows, cols, h1_off, oh, status, st);
  SC_CHECK_LAUNCH("split2h_kernel");
  return SC_OK;
}
