// Encoder-loop kernels around the attention (R/encoder.py:306-371, :475-509):
// embedding gather + per-sequence positions, residual + LayerNorm (eps 1e-12),
// bias + exact-erf GELU, [CLS] relevance head, non-finite detection.
#include <cuda_fp16.h>

#include "common.cuh"
#include "gelu.cuh"

namespace sc {

constexpr float kLnEps = 1e-12f;  // R/encoder.py:41

// Elementwise passes walk their rows last-to-first (the producing GEMM's most
// recent output is still in L2); SC_ELT_REVERSE=0 restores forward order (A/B).
static bool elt_reverse() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SC_ELT_REVERSE");
    v = e ? (atoi(e) != 0) : 1;
  }
  return v != 0;
}

// Grid-stride launch size: enough CTAs for `per_sm` waves of 256 threads over 148 SMs.
static inline unsigned grid_cap(int64_t n, int per_sm) {
  int64_t b = (n + 255) / 256, cap = 148LL * per_sm;
  return (unsigned)(b < cap ? b : cap);
}

__global__ void embed_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ pos,
                             const float* __restrict__ tok, const float* __restrict__ pe,
                             float* __restrict__ x, __nv_bfloat16* __restrict__ xh, int T, int h) {
  int r = blockIdx.x;
  if (r >= T) return;
  const float* a = tok + (int64_t)__ldg(ids + r) * h;
  const float* b = pe + (int64_t)__ldg(pos + r) * h;
  for (int c = threadIdx.x; c < h; c += blockDim.x) {
    float v = __ldg(a + c) + __ldg(b + c);
    if (x) x[(int64_t)r * h + c] = v;
    if (xh) xh[(int64_t)r * h + c] = __float2bfloat16_rn(v);
  }
}

// Every LayerNorm variant: out = LN(resid + y (+ bias)) * gamma + beta with
// fp32 statistics.  resid is fp32 or bf16 (the bf16 inference path keeps its
// residual stream in bf16); `out` (fp32) and `out_h` (bf16) are each optional;
// `bad` (optional) counts warps that produced a non-finite value -- the
// reference's per-layer isfinite check (R/encoder.py:356-357) fused into the
// pass that writes the layer output.
__device__ __forceinline__ void flag_nonfinite(int32_t* bad, bool any_bad) {
  if (bad && __any_sync(0xffffffffu, any_bad) && (threadIdx.x & 31) == 0) atomicAdd(bad, 1);
}

// Vectorised embedding (h % 128 == 0, 16-byte aligned tables): one warp per
// token, float4 table reads, bf16x4 / float4 stores.
__global__ void __launch_bounds__(256) embed_vec_kernel(const int32_t* __restrict__ ids,
                                                        const int32_t* __restrict__ pos,
                                                        const float* __restrict__ tok,
                                                        const float* __restrict__ pe, float* __restrict__ x,
                                                        __nv_bfloat16* __restrict__ xh, int T, int h) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= T) return;
  const float4* a = reinterpret_cast<const float4*>(tok + (int64_t)__ldg(ids + r) * h);
  const float4* b = reinterpret_cast<const float4*>(pe + (int64_t)__ldg(pos + r) * h);
  for (int c = lane; c < h / 4; c += 32) {
    const float4 u = __ldg(a + c), v = __ldg(b + c);
    const float4 s = make_float4(u.x + v.x, u.y + v.y, u.z + v.z, u.w + v.w);
    if (x) reinterpret_cast<float4*>(x + (int64_t)r * h)[c] = s;
    if (xh) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(s.x, s.y), hi = __floats2bfloat162_rn(s.z, s.w);
      reinterpret_cast<uint2*>(xh + (int64_t)r * h)[c] =
          make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
    }
  }
}

// One warp per row, row cached in registers (h <= 32 * kPer).
template <typename R, typename Y, int kPer>
__global__ void residual_ln_kernel(const R* __restrict__ resid, const Y* __restrict__ y,
                                   const float* __restrict__ bias, const float* __restrict__ gamma,
                                   const float* __restrict__ beta, float* __restrict__ out,
                                   __nv_bfloat16* __restrict__ out_h, int32_t* __restrict__ bad,
                                   int rows, int h) {
  int lane = threadIdx.x & 31;
  int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const R* rr = resid + (int64_t)r * h;
  const Y* yr = y + (int64_t)r * h;
  float v[kPer];
  float sum = 0.f;
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    int c = lane + 32 * e;
    v[e] = 0.f;
    if (c < h) {
      float t = to_f32(yr[c]);
      if (bias) t += __ldg(bias + c);
      v[e] = to_f32(rr[c]) + t;
      sum += v[e];
    }
  }
  float mu = warp_sum(sum) / (float)h;
  float sq = 0.f;
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    int c = lane + 32 * e;
    if (c < h) {
      v[e] -= mu;
      sq = fmaf(v[e], v[e], sq);
    }
  }
  float var = warp_sum(sq) / (float)h;
  float inv = 1.f / sqrtf(var + kLnEps);
  bool nf = false;
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    int c = lane + 32 * e;
    if (c < h) {
      float o = __ldg(gamma + c) * (v[e] * inv) + __ldg(beta + c);
      nf |= !isfinite(o);
      if (out) out[(int64_t)r * h + c] = o;
      if (out_h) out_h[(int64_t)r * h + c] = __float2bfloat16_rn(o);
    }
  }
  flag_nonfinite(bad, nf);
}

// Vectorised variant for h % 128 == 0: lane covers 4 consecutive elements at
// 4*lane + 128*e (float4 / 8-byte bf16x4 accesses, fully coalesced).
__device__ __forceinline__ float4 load4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 load4(const __nv_bfloat16* p) {
  uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
  float2 a = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.x));
  float2 b = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ bool finite4(float4 o) {
  return isfinite(o.x) && isfinite(o.y) && isfinite(o.z) && isfinite(o.w);
}

template <typename R, typename Y, int kVec, bool kRev = true>
__global__ void __launch_bounds__(256, 3) residual_ln_vec_kernel(
    const R* __restrict__ resid, const Y* __restrict__ y, const float* __restrict__ bias,
    const float* __restrict__ gamma, const float* __restrict__ beta, float* __restrict__ out,
    __nv_bfloat16* __restrict__ out_h, int32_t* __restrict__ bad, int rows, int h,
    __half* __restrict__ planes = nullptr, int64_t ldp = 0, int onehot = 0, int32_t* __restrict__ range = nullptr) {
  const int lane = threadIdx.x & 31;
  // rows last-to-first: the producing GEMM's most recent output rows are still in L2
  const int r = (kRev ? gridDim.x - 1 - blockIdx.x : blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const R* rr = resid + (int64_t)r * h;
  const Y* yr = y + (int64_t)r * h;
  float4 v[kVec];
  float sum = 0.f;
#pragma unroll
  for (int e = 0; e < kVec; ++e) {
    const int c = 4 * lane + 128 * e;
    float4 a = load4(rr + c), b = load4(yr + c);
    if (bias) {
      float4 bb = load4(bias + c);
      b.x += bb.x; b.y += bb.y; b.z += bb.z; b.w += bb.w;
    }
    v[e] = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
    sum += (v[e].x + v[e].y) + (v[e].z + v[e].w);
  }
  const float mu = warp_sum(sum) / (float)h;
  float sq = 0.f;
#pragma unroll
  for (int e = 0; e < kVec; ++e) {
    v[e].x -= mu; v[e].y -= mu; v[e].z -= mu; v[e].w -= mu;
    sq = fmaf(v[e].x, v[e].x, sq); sq = fmaf(v[e].y, v[e].y, sq);
    sq = fmaf(v[e].z, v[e].z, sq); sq = fmaf(v[e].w, v[e].w, sq);
  }
  const float inv = 1.f / sqrtf(warp_sum(sq) / (float)h + kLnEps);
  bool nf = false;
#pragma unroll
  for (int e = 0; e < kVec; ++e) {
    const int c = 4 * lane + 128 * e;
    const float4 g = load4(gamma + c), bt = load4(beta + c);
    float4 o = make_float4(g.x * (v[e].x * inv) + bt.x, g.y * (v[e].y * inv) + bt.y,
                           g.z * (v[e].z * inv) + bt.z, g.w * (v[e].w * inv) + bt.w);
    nf |= !finite4(o);
    if (out) *reinterpret_cast<float4*>(out + (int64_t)r * h + c) = o;
    if (out_h) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(o.x, o.y), hi = __floats2bfloat162_rn(o.z, o.w);
      uint2 u = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
      *reinterpret_cast<uint2*>(out_h + (int64_t)r * h + c) = u;
    }
    if (planes) {  // f16x3 GEMM operand: [h0 | (1 0 .. 0) | h1], h0 = fp16_rn(o), h1 = fp16_rn(o - h0)
      const __half2 a01 = __floats2half2_rn(o.x, o.y), a23 = __floats2half2_rn(o.z, o.w);
      const float2 f01 = __half22float2(a01), f23 = __half22float2(a23);
      const __half2 b01 = __floats2half2_rn(o.x - f01.x, o.y - f01.y), b23 = __floats2half2_rn(o.z - f23.x, o.w - f23.y);
      __half* pr = planes + (int64_t)r * ldp + c;
      *reinterpret_cast<uint2*>(pr) = make_uint2(*reinterpret_cast<const uint32_t*>(&a01), *reinterpret_cast<const uint32_t*>(&a23));
      *reinterpret_cast<uint2*>(pr + h + (onehot ? 8 : 0)) =
          make_uint2(*reinterpret_cast<const uint32_t*>(&b01), *reinterpret_cast<const uint32_t*>(&b23));
      if (onehot && c == 0) *reinterpret_cast<uint4*>(planes + (int64_t)r * ldp + h) = make_uint4(0x3c00u, 0u, 0u, 0u);
      if (range && !(fabsf(o.x) < 65504.f && fabsf(o.y) < 65504.f && fabsf(o.z) < 65504.f && fabsf(o.w) < 65504.f))
        atomicExch(range, 1);
    }
  }
  flag_nonfinite(bad, nf);
}

// Large-h fallback: block per row, three passes through L1/L2.
template <typename R, typename Y>
__global__ void residual_ln_big_kernel(const R* __restrict__ resid, const Y* __restrict__ y,
                                       const float* __restrict__ bias, const float* __restrict__ gamma,
                                       const float* __restrict__ beta, float* __restrict__ out,
                                       __nv_bfloat16* __restrict__ out_h, int32_t* __restrict__ bad,
                                       int rows, int h) {
  __shared__ float red[32];
  int r = blockIdx.x;
  const R* rr = resid + (int64_t)r * h;
  const Y* yr = y + (int64_t)r * h;
  auto val = [&](int c) { return to_f32(rr[c]) + to_f32(yr[c]) + (bias ? bias[c] : 0.f); };
  auto block_sum = [&](float s) {
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    float t = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.f;
    t = warp_sum(t);
    __syncthreads();
    return t;
  };
  float s = 0.f;
  for (int c = threadIdx.x; c < h; c += blockDim.x) s += val(c);
  float mu = block_sum(s) / (float)h;
  float q = 0.f;
  for (int c = threadIdx.x; c < h; c += blockDim.x) { float t = val(c) - mu; q = fmaf(t, t, q); }
  float inv = 1.f / sqrtf(block_sum(q) / (float)h + kLnEps);
  __syncthreads();
  // (each column is read and written by the same thread, so resid may alias out / out_h)
  bool nf = false;
  for (int c = threadIdx.x; c < h; c += blockDim.x) {
    const float o = gamma[c] * ((val(c) - mu) * inv) + beta[c];
    nf |= !isfinite(o);
    if (out) out[(int64_t)r * h + c] = o;
    if (out_h) out_h[(int64_t)r * h + c] = __float2bfloat16_rn(o);
  }
  flag_nonfinite(bad, nf);
}

template <typename R, typename Y>
int launch_ln(const void* resid_v, const void* y, const float* bias, const float* gamma,
              const float* beta, float* out, void* out_h, int32_t* bad, int rows, int h, cudaStream_t st) {
  const R* resid = static_cast<const R*>(resid_v);
  const Y* yy = static_cast<const Y*>(y);
  __nv_bfloat16* oh = static_cast<__nv_bfloat16*>(out_h);
  unsigned blocks = (unsigned)((rows + 7) / 8);
  int per = (h + 31) / 32;
  const bool vec = (h % 128 == 0) && !(((uintptr_t)resid | (uintptr_t)y | (uintptr_t)out |
                                         (uintptr_t)out_h | (uintptr_t)gamma | (uintptr_t)beta |
                                         (uintptr_t)bias) & 15);
#define SC_LN_ARGS resid, yy, bias, gamma, beta, out, oh, bad, rows, h
  if (vec && h == 768 && !elt_reverse()) residual_ln_vec_kernel<R, Y, 6, false><<<blocks, 256, 0, st>>>(SC_LN_ARGS);
  else if (vec && h == 768) residual_ln_vec_kernel<R, Y, 6><<<blocks, 256, 0, st>>>(SC_LN_ARGS);
  else if (vec && h == 384) residual_ln_vec_kernel<R, Y, 3><<<blocks, 256, 0, st>>>(SC_LN_ARGS);
  else if (vec && h == 1024) residual_ln_vec_kernel<R, Y, 8><<<blocks, 256, 0, st>>>(SC_LN_ARGS);
  else if (vec && h == 512) residual_ln_vec_kernel<R, Y, 4><<<blocks, 256, 0, st>>>(SC_LN_ARGS);
  else if (vec && h == 256) residual_ln_vec_kernel<R, Y, 2><<<blocks, 256, 0, st>>>(SC_LN_ARGS);
  else if (vec && h == 128) residual_ln_vec_kernel<R, Y, 1><<<blocks, 256, 0, st>>>(SC_LN_ARGS);
  else if (per <= 1) residual_ln_kernel<R, Y, 1><<<blocks, 256, 0, st>>>(SC_LN_ARGS);
  else if (per <= 4) residual_ln_kernel<R, Y, 4><<<blocks, 256, 0, st>>>(SC_LN_ARGS);
  else if (per <= 8) residual_ln_kernel<R, Y, 8><<<blocks, 256, 0, st>>>(SC_LN_ARGS);
  else if (per <= 24) residual_ln_kernel<R, Y, 24><<<blocks, 256, 0, st>>>(SC_LN_ARGS);
  else if (per <= 32) residual_ln_kernel<R, Y, 32><<<blocks, 256, 0, st>>>(SC_LN_ARGS);
  else residual_ln_big_kernel<R, Y><<<rows, 256, 0, st>>>(SC_LN_ARGS);
#undef SC_LN_ARGS
  SC_CHECK_LAUNCH("residual_ln_kernel");
  return SC_OK;
}

__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.f + erff(x * 0.70710678118654752440f));
}

template <typename T>
__global__ void bias_gelu_kernel(T* __restrict__ x, const float* __restrict__ bias, int64_t n,
                                 int cols) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float v = to_f32(x[i]);
    if (bias) v += __ldg(bias + (int)(i % cols));
    x[i] = from_f32<T>(gelu_erf(v));
  }
}

// bf16, 8 elements per thread, cols % 8 == 0.
template <bool kBias>
__device__ __forceinline__ void gelu_bf16x8(uint4& u, const float* __restrict__ bias, int64_t i, int cols) {
  __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&u);
  const int c0 = kBias ? (int)((i * 8) % cols) : 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    float2 f = __bfloat1622float2(b[e]);
    if constexpr (kBias) { f.x += __ldg(bias + c0 + 2 * e); f.y += __ldg(bias + c0 + 2 * e + 1); }
    b[e] = __float22bfloat162_rn(gelu2_bf16path(f));
  }
}

// Four 16-byte vectors per thread per iteration, all loads issued before any
// math: ~48 KB of loads in flight per SM at 4 CTAs x 256 threads, enough to
// cover HBM latency (2 vectors/thread at 3 CTAs/SM measured 74% of copy BW,
// stalled on long scoreboard).
template <bool kBias, bool kRev = true>
__global__ void __launch_bounds__(256, 4) bias_gelu_bf16x8_kernel(__nv_bfloat16* __restrict__ x,
                                                                 const float* __restrict__ bias, int64_t n8,
                                                                 int cols) {
  constexpr int U = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  uint4* xv = reinterpret_cast<uint4*>(x);
  // walked last-to-first (vector n8-1-i): the W1 GEMM's most recent output is still in L2
  const int64_t last = n8 - 1;
  auto at = [&](int64_t k) { return kRev ? last - k : k; };
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n8; i += U * stride) {
    uint4 u[U];
#pragma unroll
    for (int k = 0; k < U; ++k) u[k] = __ldcs(xv + at(i + k * stride));
#pragma unroll
    for (int k = 0; k < U; ++k) gelu_bf16x8<kBias>(u[k], bias, at(i + k * stride), cols);
#pragma unroll
    for (int k = 0; k < U; ++k) __stcs(xv + at(i + k * stride), u[k]);
  }
  for (; i < n8; i += stride) {
    uint4 v = xv[at(i)];
    gelu_bf16x8<kBias>(v, bias, at(i), cols);
    xv[at(i)] = v;
  }
}

__global__ void cls_score_kernel(const float* __restrict__ x, const int32_t* __restrict__ cu, int nseq,
                                 int h, const float* __restrict__ w, float b, float* __restrict__ out) {
  int lane = threadIdx.x & 31;
  int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= nseq) return;
  const float* xr = x + (int64_t)cu[j] * h;
  float s = 0.f;
  for (int c = lane; c < h; c += 32) s = fmaf(xr[c], w[c], s);
  s = warp_sum(s);
  if (lane == 0) out[j] = s + b;
}

__global__ void nonfinite_kernel(const float* __restrict__ x, int64_t n, int32_t* __restrict__ count) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    bad |= !isfinite(x[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicAdd(count, 1);
}

}  // namespace sc

using namespace sc;

extern "C" int sc_embed(const int32_t* ids, const int32_t* tok_pos, const float* tok_emb,
                        const float* pos_emb, float* x, void* xh, int32_t total_tokens,
                        int32_t hidden, void* stream) {
  SC_CHECK_ARG(ids && tok_pos && tok_emb && pos_emb && (x || xh), "sc_embed: null pointer");
  SC_CHECK_ARG(total_tokens >= 0 && hidden >= 1, "sc_embed: bad shape");
  if (total_tokens == 0) return SC_OK;
  const bool vec = hidden % 128 == 0 && !(((uintptr_t)tok_emb | (uintptr_t)pos_emb | (uintptr_t)x | (uintptr_t)xh) & 15);
  if (vec) {
    embed_vec_kernel<<<(total_tokens + 7) / 8, 256, 0, (cudaStream_t)stream>>>(
        ids, tok_pos, tok_emb, pos_emb, x, (__nv_bfloat16*)xh, total_tokens, hidden);
  } else {
    int threads = hidden >= 256 ? 256 : 32 * ((hidden + 31) / 32);
    embed_kernel<<<total_tokens, threads, 0, (cudaStream_t)stream>>>(
        ids, tok_pos, tok_emb, pos_emb, x, (__nv_bfloat16*)xh, total_tokens, hidden);
  }
  SC_CHECK_LAUNCH("embed_kernel");
  return SC_OK;
}

extern "C" int sc_residual_layernorm_ex(const void* resid, int32_t resid_dtype, const void* y,
                                        int32_t y_dtype, const float* bias, const float* gamma,
                                        const float* beta, float* x_out, void* out_h,
                                        int32_t* nonfinite_count, int32_t rows, int32_t hidden,
                                        void* stream) {
  SC_CHECK_ARG(resid && y && gamma && beta && (x_out || out_h), "sc_residual_layernorm: null pointer");
  SC_CHECK_ARG(rows >= 0 && hidden >= 1, "sc_residual_layernorm: bad shape");
  SC_CHECK_ARG(resid_dtype == SC_DTYPE_F32 || resid_dtype == SC_DTYPE_BF16, "sc_residual_layernorm: bad resid dtype %d", resid_dtype);
  SC_CHECK_ARG(y_dtype == SC_DTYPE_F32 || y_dtype == SC_DTYPE_BF16, "sc_residual_layernorm: bad dtype %d", y_dtype);
  if (rows == 0) return SC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const float* b = bias;
  if (resid_dtype == SC_DTYPE_F32) {
    if (y_dtype == SC_DTYPE_F32) return launch_ln<float, float>(resid, y, b, gamma, beta, x_out, out_h, nonfinite_count, rows, hidden, st);
    return launch_ln<float, __nv_bfloat16>(resid, y, b, gamma, beta, x_out, out_h, nonfinite_count, rows, hidden, st);
  }
  if (y_dtype == SC_DTYPE_F32) return launch_ln<__nv_bfloat16, float>(resid, y, b, gamma, beta, x_out, out_h, nonfinite_count, rows, hidden, st);
  return launch_ln<__nv_bfloat16, __nv_bfloat16>(resid, y, b, gamma, beta, x_out, out_h, nonfinite_count, rows, hidden, st);
}

extern "C" int sc_residual_layernorm(const float* resid, const void* y, int32_t y_dtype,
                                     const float* bias, const float* gamma, const float* beta,
                                     float* x_out, void* out_h, int32_t rows, int32_t hidden,
                                     void* stream) {
  SC_CHECK_ARG(x_out, "sc_residual_layernorm: null pointer");
  return sc_residual_layernorm_ex(resid, SC_DTYPE_F32, y, y_dtype, bias, gamma, beta, x_out, out_h, nullptr,
                                  rows, hidden, stream);
}

// fp32 residual LayerNorm that also writes the f16x3 GEMM operand planes of its output (the split
// pass of the ranking-exact fp32 mode fused into the producer; encoder.py split_planes_h).
extern "C" int sc_residual_layernorm_f16x2(const float* resid, const float* y, const float* bias, const float* gamma,
                                           const float* beta, float* x_out, void* planes, int64_t ldp, int32_t onehot,
                                           int32_t* range_status, int32_t* nonfinite_count, int32_t rows,
                                           int32_t hidden, void* stream) {
  SC_CHECK_ARG(resid && y && gamma && beta && x_out && planes, "sc_residual_layernorm_f16x2: null pointer");
  SC_CHECK_ARG(rows >= 0 && hidden >= 1 && ldp >= 2LL * hidden + (onehot ? 8 : 0),
               "sc_residual_layernorm_f16x2: bad shape");
  if (rows == 0) return SC_OK;
  const bool vec = (hidden == 128 || hidden == 256 || hidden == 384 || hidden == 512 || hidden == 768 ||
                    hidden == 1024) && ldp % 8 == 0 &&
                   !(((uintptr_t)resid | (uintptr_t)y | (uintptr_t)x_out | (uintptr_t)gamma | (uintptr_t)beta |
                      (uintptr_t)bias | (uintptr_t)planes) & 15);
  if (!vec) {
    set_error("sc_residual_layernorm_f16x2: needs hidden in {128,256,384,512,768,1024} and 16-byte alignment");
    return SC_ERR_UNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned blocks = (unsigned)((rows + 7) / 8);
  __half* pl = static_cast<__half*>(planes);
#define SC_LNP_ARGS resid, y, bias, gamma, beta, x_out, nullptr, nonfinite_count, rows, hidden, pl, ldp, onehot ? 1 : 0, range_status
  switch (hidden) {
    case 128: residual_ln_vec_kernel<float, float, 1><<<blocks, 256, 0, st>>>(SC_LNP_ARGS); break;
    case 256: residual_ln_vec_kernel<float, float, 2><<<blocks, 256, 0, st>>>(SC_LNP_ARGS); break;
    case 384: residual_ln_vec_kernel<float, float, 3><<<blocks, 256, 0, st>>>(SC_LNP_ARGS); break;
    case 512: residual_ln_vec_kernel<float, float, 4><<<blocks, 256, 0, st>>>(SC_LNP_ARGS); break;
    case 768: residual_ln_vec_kernel<float, float, 6><<<blocks, 256, 0, st>>>(SC_LNP_ARGS); break;
    default: residual_ln_vec_kernel<float, float, 8><<<blocks, 256, 0, st>>>(SC_LNP_ARGS); break;
  }
#undef SC_LNP_ARGS
  SC_CHECK_LAUNCH("residual_ln_vec_kernel (planes)");
  return SC_OK;
}

extern "C" int sc_bias_gelu(void* x, const float* bias, int32_t dtype, int64_t rows, int32_t cols,
                            void* stream) {
  SC_CHECK_ARG(x && rows >= 0 && cols >= 1, "sc_bias_gelu: bad arguments");
  int64_t n = rows * cols;
  if (n == 0) return SC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SC_DTYPE_BF16 && cols % 8 == 0 && ((uintptr_t)x & 15) == 0) {
    int64_t n8 = n / 8;
    unsigned blocks = grid_cap((n8 + 3) / 4, 4);
    if (bias)
      bias_gelu_bf16x8_kernel<true><<<blocks, 256, 0, st>>>((__nv_bfloat16*)x, bias, n8, cols);
    else if (elt_reverse())
      bias_gelu_bf16x8_kernel<false><<<blocks, 256, 0, st>>>((__nv_bfloat16*)x, bias, n8, cols);
    else
      bias_gelu_bf16x8_kernel<false, false><<<blocks, 256, 0, st>>>((__nv_bfloat16*)x, bias, n8, cols);
  } else if (dtype == SC_DTYPE_BF16) {
    unsigned blocks = grid_cap(n, 16);
    bias_gelu_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>((__nv_bfloat16*)x, bias, n, cols);
  } else if (dtype == SC_DTYPE_F32) {
    unsigned blocks = grid_cap(n, 16);
    bias_gelu_kernel<float><<<blocks, 256, 0, st>>>((float*)x, bias, n, cols);
  } else {
    set_error("sc_bias_gelu: bad dtype %d", dtype);
    return SC_ERR_INVALID;
  }
  SC_CHECK_LAUNCH("bias_gelu_kernel");
  return SC_OK;
}

extern "C" int sc_cls_score(const float* x, const int32_t* cu_seqlens, int32_t nseq, int32_t hidden,
                            const float* head_w, float head_b, float* scores, void* stream) {
  SC_CHECK_ARG(x && cu_seqlens && head_w && scores && nseq >= 0 && hidden >= 1,
               "sc_cls_score: bad arguments");
  if (nseq == 0) return SC_OK;
  cls_score_kernel<<<(nseq + 7) / 8, 256, 0, (cudaStream_t)stream>>>(x, cu_seqlens, nseq, hidden,
                                                                      head_w, head_b, scores);
  SC_CHECK_LAUNCH("cls_score_kernel");
  return SC_OK;
}

extern "C" int sc_count_nonfinite(const float* x, int64_t n, int32_t* count, void* stream) {
  SC_CHECK_ARG(x && count && n >= 0, "sc_count_nonfinite: bad arguments");
  if (n == 0) return SC_OK;
  unsigned blocks = grid_cap(n, 8);
  nonfinite_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(x, n, count);
  SC_CHECK_LAUNCH("nonfinite_kernel");
  return SC_OK;
}
