// Dense-layer kernels of the fine-tuning step, replacing the
// reference's layer_norm / layer_norm_backward (R/encoder.py:267-285) and the
// bias sums of layer_backward (R/encoder.py:398-443):
//   * ln_fwd_kernel:  y = LN(a + b) with per-row mean / rstd kept for the
//     backward (residual add fused; a, b fp32 or bf16);
//   * ln_bwd_kernel:  dx = rstd (g dy - mean(g dy) - xhat mean(g dy xhat)),
//     recomputing xhat from a + b, plus per-CTA partial column sums of
//     dy * xhat and dy (dgamma, dbeta);
//   * colsum_kernel:  per-CTA partial column sums of a [rows x cols] matrix
//     (bias gradients);
//   * colsum_reduce_kernel: the partials summed in CTA order.
// Warp per row, lane holds columns lane + 32e; every reduction has a fixed
// order, so the gradients are bit-reproducible.
#include "common.cuh"

namespace sc {

constexpr int kLnMaxV = 32;  // columns per lane -> cols <= 1024
constexpr int kLnWarps = 8;

// 4 consecutive columns as float4 (fp32 rows: 16-byte loads; bf16 rows: 8-byte loads).
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ld4(const __nv_bfloat16* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
  const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }

// Lane owns column groups q = lane + 32k (k < KV), columns 4q .. 4q+3; cols % 4 == 0.
template <typename TA, typename TB, int KV>
__global__ void __launch_bounds__(kLnWarps * 32, 4) ln_fwd_kernel(const TA* __restrict__ a, const TB* __restrict__ b,
                                                                  const float* __restrict__ gamma,
                                                                  const float* __restrict__ beta,
                                                                  float* __restrict__ y, float* __restrict__ mean,
                                                                  float* __restrict__ rstd, int rows, int cols,
                                                                  float eps, __nv_bfloat16* __restrict__ y16) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * kLnWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int64_t base = (int64_t)row * cols;
  const int ng = cols >> 2;
  float4 x[KV];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    const int q = lane + 32 * k;
    x[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (q < ng) {
      x[k] = ld4(a + base + 4 * q);
      if (b) x[k] = add4(x[k], ld4(b + base + 4 * q));
    }
    s += (x[k].x + x[k].y) + (x[k].z + x[k].w);
  }
  const float mu = warp_sum(s) / cols;
  float v = 0.f;
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    if (lane + 32 * k < ng) {
      const float d0 = x[k].x - mu, d1 = x[k].y - mu, d2 = x[k].z - mu, d3 = x[k].w - mu;
      v = fmaf(d0, d0, fmaf(d1, d1, fmaf(d2, d2, fmaf(d3, d3, v))));
    }
  }
  const float rs = rsqrtf(warp_sum(v) / cols + eps);
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    const int q = lane + 32 * k;
    if (q < ng) {
      const float4 g = ld4(gamma + 4 * q), bb = ld4(beta + 4 * q);
      const float4 o = make_float4((x[k].x - mu) * rs * g.x + bb.x, (x[k].y - mu) * rs * g.y + bb.y,
                                   (x[k].z - mu) * rs * g.z + bb.z, (x[k].w - mu) * rs * g.w + bb.w);
      *reinterpret_cast<float4*>(y + base + 4 * q) = o;
      if (y16) {  // bf16 copy for the next GEMM
        __nv_bfloat162 lo = __floats2bfloat162_rn(o.x, o.y), hi = __floats2bfloat162_rn(o.z, o.w);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&lo);
        u.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(y16 + base + 4 * q) = u;
      }
    }
  }
  if (lane == 0) { mean[row] = mu; rstd[row] = rs; }
}

// Grid: a fixed number of CTAs; warp w of CTA k handles rows (k * kLnWarps + w) + i * stride.
// dgamma / dbeta accumulate in the warp's own shared-memory row (no atomics), then the CTA sums
// its warps in order into one partial row.
template <typename TA, typename TB, int KV>
__global__ void __launch_bounds__(kLnWarps * 32, 2) ln_bwd_kernel(const float* __restrict__ dy,
                                                                  const TA* __restrict__ a, const TB* __restrict__ b,
                                                                  const float* __restrict__ gamma,
                                                                  const float* __restrict__ mean,
                                                                  const float* __restrict__ rstd,
                                                                  float* __restrict__ dx, float* __restrict__ part_g,
                                                                  float* __restrict__ part_b, int rows, int cols,
                                                                  const __nv_bfloat16* __restrict__ dy16,
                                                                  __nv_bfloat16* __restrict__ dx16) {
  extern __shared__ float4 lnsm[];  // [2][kLnWarps][ng] float4
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ng = cols >> 2;
  float4* accg = lnsm + warp * ng;
  float4* accb = lnsm + (kLnWarps + warp) * ng;
  for (int q = lane; q < ng; q += 32) accg[q] = accb[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  const float inv_cols = 1.f / cols;
  const int stride = gridDim.x * kLnWarps;
  for (int row = blockIdx.x * kLnWarps + warp; row < rows; row += stride) {
    const int64_t base = (int64_t)row * cols;
    const float mu = mean[row], rs = rstd[row];
    float4 xh[KV], gd[KV];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int q = lane + 32 * k;
      xh[k] = gd[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (q < ng) {
        float4 xv = ld4(a + base + 4 * q);
        if (b) xv = add4(xv, ld4(b + base + 4 * q));
        float4 d = ld4(dy + base + 4 * q);
        if (dy16) d = add4(d, ld4(dy16 + base + 4 * q));  // gradient of the bf16 copy of y
        const float4 g = ld4(gamma + 4 * q);
        xh[k] = make_float4((xv.x - mu) * rs, (xv.y - mu) * rs, (xv.z - mu) * rs, (xv.w - mu) * rs);
        gd[k] = make_float4(d.x * g.x, d.y * g.y, d.z * g.z, d.w * g.w);
        float4 ag = accg[q], ab = accb[q];
        ag.x = fmaf(d.x, xh[k].x, ag.x); ag.y = fmaf(d.y, xh[k].y, ag.y);
        ag.z = fmaf(d.z, xh[k].z, ag.z); ag.w = fmaf(d.w, xh[k].w, ag.w);
        accg[q] = ag;
        accb[q] = add4(ab, d);
        s1 += (gd[k].x + gd[k].y) + (gd[k].z + gd[k].w);
        s2 = fmaf(gd[k].x, xh[k].x, fmaf(gd[k].y, xh[k].y, fmaf(gd[k].z, xh[k].z, fmaf(gd[k].w, xh[k].w, s2))));
      }
    }
    const float m1 = warp_sum(s1) * inv_cols, m2 = warp_sum(s2) * inv_cols;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int q = lane + 32 * k;
      if (q < ng) {
        const float4 o = make_float4(rs * (gd[k].x - m1 - xh[k].x * m2), rs * (gd[k].y - m1 - xh[k].y * m2),
                                     rs * (gd[k].z - m1 - xh[k].z * m2), rs * (gd[k].w - m1 - xh[k].w * m2));
        if (dx) *reinterpret_cast<float4*>(dx + base + 4 * q) = o;
        if (dx16) {  // bf16 copy: the gradient of a bf16 input
          __nv_bfloat162 lo = __floats2bfloat162_rn(o.x, o.y), hi = __floats2bfloat162_rn(o.z, o.w);
          uint2 u;
          u.x = *reinterpret_cast<uint32_t*>(&lo);
          u.y = *reinterpret_cast<uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(dx16 + base + 4 * q) = u;
        }
      }
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < ng; q += blockDim.x) {
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f), bb = g;
    for (int w = 0; w < kLnWarps; ++w) {
      g = add4(g, lnsm[w * ng + q]);
      bb = add4(bb, lnsm[(kLnWarps + w) * ng + q]);
    }
    *reinterpret_cast<float4*>(part_g + (int64_t)blockIdx.x * cols + 4 * q) = g;
    *reinterpret_cast<float4*>(part_b + (int64_t)blockIdx.x * cols + 4 * q) = bb;
  }
}

// CTA k sums rows [k * rpc, (k+1) * rpc) of x; thread t owns columns 8t .. 8t+7 (+ 8 * blockDim
// per pass), 16-byte loads for bf16 (two for fp32), rows summed in order in registers.
template <typename T>
__global__ void __launch_bounds__(256) colsum_kernel(const T* __restrict__ x, int64_t ld, int rows, int cols, int rpc,
                                                     float* __restrict__ part) {
  const int r0 = blockIdx.x * rpc, r1 = min(rows, r0 + rpc);
  const bool vec = (cols % 8) == 0 && ((ld * sizeof(T)) % 16) == 0 && (reinterpret_cast<uintptr_t>(x) % 16) == 0;
  for (int c0 = 8 * threadIdx.x; c0 < cols; c0 += 8 * blockDim.x) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const T* p = x + (int64_t)r0 * ld + c0;
    for (int r = r0; r < r1; ++r, p += ld) {
      if (vec) {
        if constexpr (sizeof(T) == 2) {
          const uint4 u = *reinterpret_cast<const uint4*>(p);
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(h[e]);
            acc[2 * e] += f.x;
            acc[2 * e + 1] += f.y;
          }
        } else {
          const float4 u0 = *reinterpret_cast<const float4*>(p), u1 = *reinterpret_cast<const float4*>(p + 4);
          acc[0] += u0.x; acc[1] += u0.y; acc[2] += u0.z; acc[3] += u0.w;
          acc[4] += u1.x; acc[5] += u1.y; acc[6] += u1.z; acc[7] += u1.w;
        }
      } else {
        for (int e = 0; e < 8 && c0 + e < cols; ++e) acc[e] += to_f32(p[e]);
      }
    }
    if (vec) {
      float4* o = reinterpret_cast<float4*>(part + (int64_t)blockIdx.x * cols + c0);
      o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
      o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    } else {
      for (int e = 0; e < 8 && c0 + e < cols; ++e) part[(int64_t)blockIdx.x * cols + c0 + e] = acc[e];
    }
  }
}

// out[c] = sum over partial rows k of part[k][c]: block = 32 columns x 8 warps, warp w sums rows
// k = w (mod 8) (four loads in flight), the 8 warp sums are added in warp order (deterministic).
constexpr int kRedWarps = 8;
// blockIdx.y = 1 reduces a second (part, out) pair in the same launch (LayerNorm dgamma + dbeta).
__global__ void __launch_bounds__(kRedWarps * 32) colsum_reduce_kernel(const float* __restrict__ part, int nparts,
                                                                       int cols, float* __restrict__ out,
                                                                       const float* __restrict__ part1 = nullptr,
                                                                       float* __restrict__ out1 = nullptr) {
  if (blockIdx.y == 1) part = part1, out = out1;
  __shared__ float red[kRedWarps][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float acc = 0.f;
  if (c < cols) {
#pragma unroll 4
    for (int k = warp; k < nparts; k += kRedWarps) acc += __ldg(part + (int64_t)k * cols + c);
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && c < cols) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < kRedWarps; ++w) t += red[w][lane];
    out[c] = t;
  }
}

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  return sms;
}

template <typename TA, typename TB, int KV>
void ln_launch(bool fwd, const void* a, const void* b, const float* gamma, const float* beta, const float* dy,
               float* y, float* mean, float* rstd, float* dx, float* pg, float* pb, int rows, int cols, float eps,
               unsigned blocks, cudaStream_t st, void* aux, void* aux2) {
  if (fwd) {
    ln_fwd_kernel<TA, TB, KV><<<blocks, kLnWarps * 32, 0, st>>>((const TA*)a, (const TB*)b, gamma, beta, y, mean,
                                                                 rstd, rows, cols, eps, (__nv_bfloat16*)aux);
  } else {
    const size_t sm = (size_t)2 * kLnWarps * cols * sizeof(float);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(ln_bwd_kernel<TA, TB, KV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           2 * kLnWarps * kLnMaxV * 32 * (int)sizeof(float));
      attr = true;
    }
    ln_bwd_kernel<TA, TB, KV><<<blocks, kLnWarps * 32, sm, st>>>(dy, (const TA*)a, (const TB*)b, gamma, mean, rstd,
                                                                  dx, pg, pb, rows, cols, (const __nv_bfloat16*)aux,
                                                                  (__nv_bfloat16*)aux2);
  }
}

template <int KV>
void ln_dispatch_types(bool af, bool bf, bool fwd, const void* a, const void* b, const float* gamma,
                       const float* beta, const float* dy, float* y, float* mean, float* rstd, float* dx, float* pg,
                       float* pb, int rows, int cols, float eps, unsigned blocks, cudaStream_t st, void* aux,
                       void* aux2) {
  using B16 = __nv_bfloat16;
  if (af && bf) ln_launch<float, float, KV>(fwd, a, b, gamma, beta, dy, y, mean, rstd, dx, pg, pb, rows, cols, eps, blocks, st, aux, aux2);
  else if (af) ln_launch<float, B16, KV>(fwd, a, b, gamma, beta, dy, y, mean, rstd, dx, pg, pb, rows, cols, eps, blocks, st, aux, aux2);
  else if (bf) ln_launch<B16, float, KV>(fwd, a, b, gamma, beta, dy, y, mean, rstd, dx, pg, pb, rows, cols, eps, blocks, st, aux, aux2);
  else ln_launch<B16, B16, KV>(fwd, a, b, gamma, beta, dy, y, mean, rstd, dx, pg, pb, rows, cols, eps, blocks, st, aux, aux2);
}

// Column groups (of 4) per lane rounded up to an instantiated width.
void ln_dispatch(bool af, bool bf, bool fwd, const void* a, const void* b, const float* gamma, const float* beta,
                 const float* dy, float* y, float* mean, float* rstd, float* dx, float* pg, float* pb, int rows,
                 int cols, float eps, unsigned blocks, cudaStream_t st, void* aux, void* aux2) {
  const int kv = (cols / 4 + 31) / 32;
#define SC_LN_CASE(W) \
  if (kv <= W) return ln_dispatch_types<W>(af, bf, fwd, a, b, gamma, beta, dy, y, mean, rstd, dx, pg, pb, rows, cols, eps, blocks, st, aux, aux2);
  SC_LN_CASE(1) SC_LN_CASE(2) SC_LN_CASE(4) SC_LN_CASE(6) SC_LN_CASE(8)
#undef SC_LN_CASE
}

}  // namespace sc

using namespace sc;

extern "C" int sc_ln_partials(int32_t rows) {
  const int cap = num_sms() * 4;
  return rows < cap ? (rows > 0 ? rows : 1) : cap;
}

extern "C" int sc_layernorm_fwd(const void* a, int32_t a_dtype, const void* b, int32_t b_dtype, const float* gamma,
                                const float* beta, float* y, void* y_bf16, float* mean, float* rstd, int32_t rows,
                                int32_t cols, float eps, void* stream) {
  SC_CHECK_ARG(a && gamma && beta && y && mean && rstd, "sc_layernorm_fwd: null pointer");
  SC_CHECK_ARG(rows >= 0 && cols >= 1, "sc_layernorm_fwd: bad shape");
  if (cols > kLnMaxV * 32 || cols % 4 ||
      ((uintptr_t)a | (uintptr_t)b | (uintptr_t)y | (uintptr_t)y_bf16 | (uintptr_t)gamma | (uintptr_t)beta) % 8) {
    set_error("sc_layernorm_fwd: needs cols %% 4 == 0, cols <= %d and 8-byte aligned rows", kLnMaxV * 32);
    return SC_ERR_UNSUPPORTED;
  }
  SC_CHECK_ARG((a_dtype == SC_DTYPE_F32 || a_dtype == SC_DTYPE_BF16) &&
               (!b || b_dtype == SC_DTYPE_F32 || b_dtype == SC_DTYPE_BF16), "sc_layernorm_fwd: bad dtype");
  if (rows == 0) return SC_OK;
  const unsigned blocks = (unsigned)((rows + kLnWarps - 1) / kLnWarps);
  ln_dispatch(a_dtype == SC_DTYPE_F32, !b || b_dtype == SC_DTYPE_F32, true, a, b, gamma, beta, nullptr, y, mean, rstd,
              nullptr, nullptr, nullptr, rows, cols, eps, blocks, (cudaStream_t)stream, y_bf16, nullptr);
  SC_CHECK_LAUNCH("ln_fwd_kernel");
  return SC_OK;
}

extern "C" int sc_layernorm_bwd(const float* dy, const void* dy_bf16, const void* a, int32_t a_dtype, const void* b,
                                int32_t b_dtype,
                                const float* gamma, const float* mean, const float* rstd, float* dx, void* dx_bf16, float* dgamma,
                                float* dbeta, float* partials, int32_t rows, int32_t cols, void* stream) {
  SC_CHECK_ARG(dy && a && gamma && mean && rstd && (dx || dx_bf16) && dgamma && dbeta && partials,
               "sc_layernorm_bwd: null pointer");
  SC_CHECK_ARG(rows >= 0 && cols >= 1, "sc_layernorm_bwd: bad shape");
  if (cols > kLnMaxV * 32 || cols % 4 ||
      ((uintptr_t)a | (uintptr_t)b | (uintptr_t)dy | (uintptr_t)dy_bf16 | (uintptr_t)dx | (uintptr_t)dx_bf16 |
       (uintptr_t)gamma) % 8) {
    set_error("sc_layernorm_bwd: needs cols %% 4 == 0, cols <= %d and 8-byte aligned rows", kLnMaxV * 32);
    return SC_ERR_UNSUPPORTED;
  }
  SC_CHECK_ARG((a_dtype == SC_DTYPE_F32 || a_dtype == SC_DTYPE_BF16) &&
               (!b || b_dtype == SC_DTYPE_F32 || b_dtype == SC_DTYPE_BF16), "sc_layernorm_bwd: bad dtype");
  const int nparts = sc_ln_partials(rows);
  cudaStream_t st = (cudaStream_t)stream;
  float* pg = partials;
  float* pb = partials + (int64_t)nparts * cols;
  if (rows == 0) {  // no partial rows to reduce: the parameter gradients are exactly zero
    if (cudaMemsetAsync(dgamma, 0, sizeof(float) * cols, st) != cudaSuccess ||
        cudaMemsetAsync(dbeta, 0, sizeof(float) * cols, st) != cudaSuccess) {
      set_error("sc_layernorm_bwd: cudaMemsetAsync failed");
      return SC_ERR_CUDA;
    }
    return SC_OK;
  }
  ln_dispatch(a_dtype == SC_DTYPE_F32, !b || b_dtype == SC_DTYPE_F32, false, a, b, gamma, nullptr, dy, nullptr,
                (float*)mean, (float*)rstd, dx, pg, pb, rows, cols, 0.f, (unsigned)nparts, st, (void*)dy_bf16,
                dx_bf16);
  SC_CHECK_LAUNCH("ln_bwd_kernel");
  colsum_reduce_kernel<<<dim3((cols + 31) / 32, 2), kRedWarps * 32, 0, st>>>(pg, nparts, cols, dgamma, pb, dbeta);
  SC_CHECK_LAUNCH("colsum_reduce_kernel");
  return SC_OK;
}

extern "C" int sc_colsum(const void* x, int32_t dtype, int64_t ld, int32_t rows, int32_t cols, float* out,
                         float* partials, void* stream) {
  SC_CHECK_ARG(x && out && partials, "sc_colsum: null pointer");
  SC_CHECK_ARG(rows >= 0 && cols >= 1 && ld >= cols, "sc_colsum: bad shape");
  SC_CHECK_ARG(dtype == SC_DTYPE_F32 || dtype == SC_DTYPE_BF16, "sc_colsum: bad dtype");
  const int nparts = sc_ln_partials(rows);
  const int rpc = (rows + nparts - 1) / nparts;
  cudaStream_t st = (cudaStream_t)stream;
  const int threads = min(256, max(32, ((cols + 7) / 8 + 31) / 32 * 32));
  if (dtype == SC_DTYPE_F32)
    colsum_kernel<float><<<nparts, threads, 0, st>>>((const float*)x, ld, rows, cols, rpc, partials);
  else
    colsum_kernel<__nv_bfloat16><<<nparts, threads, 0, st>>>((const __nv_bfloat16*)x, ld, rows, cols, rpc, partials);
  SC_CHECK_LAUNCH("colsum_kernel");
  colsum_reduce_kernel<<<(cols + 31) / 32, kRedWarps * 32, 0, st>>>(partials, nparts, cols, out);
  SC_CHECK_LAUNCH("colsum_reduce_kernel");
  return SC_OK;
}

// ---- exact-erf GELU forward / backward (R/encoder.py:258-264) -------------------------------
//   gelu(x)  = 0.5 x (1 + erf(x / sqrt 2))
//   gelu'(x) = 0.5 (1 + erf(x / sqrt 2)) + x exp(-x^2 / 2) / sqrt(2 pi)
// The backward also reduces the column sums of dx (the bias gradient of the GEMM that produced x),
// per-CTA partials like colsum_kernel.

namespace sc {

// fp32 (parity) path: erff / expf.
__device__ __forceinline__ float gelu_f(float x) { return 0.5f * x * (1.f + erff(x * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_grad_f(float x) {
  return 0.5f * (1.f + erff(x * 0.70710678118654752f)) + x * expf(-0.5f * x * x) * 0.3989422804014327f;
}

// bf16 path: one MUFU op per element.  With z = x / sqrt 2, e = exp(-z^2):
//   Phi(x) = 1 - 0.5 e R(|z|) (x >= 0) or 0.5 e R(|z|) (x < 0), R the degree-10 erfcx fit of
//   gelu.cuh (|z| clamped at 4), and phi(x) = e / sqrt(2 pi); gelu = x Phi, gelu' = Phi + x phi.
__device__ __forceinline__ void gelu_parts_fast(float x, float& Phi, float& phi) {
  const float z = x * 0.70710678118654752f;
  const float a = fminf(fabsf(z), 4.f);
  float p = fmaf(1.1544991139089689e-05f, a, -0.00027032289654016495f);
  p = fmaf(p, a, 0.0028087019454687834f);
  p = fmaf(p, a, -0.017178276553750038f);
  p = fmaf(p, a, 0.06945336610078812f);
  p = fmaf(p, a, -0.19890554249286652f);
  p = fmaf(p, a, 0.4261739253997803f);
  p = fmaf(p, a, -0.7184767723083496f);
  p = fmaf(p, a, 0.9914032816886902f);
  p = fmaf(p, a, -1.1274118423461914f);
  p = fmaf(p, a, 0.9999727010726929f);
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-z * z * 1.4426950408889634f));
  const float he = 0.5f * e * p;
  Phi = x >= 0.f ? 1.f - he : he;
  phi = e * 0.3989422804014327f;
}
template <typename T>
__device__ __forceinline__ float gelu_t(float x) {
  if constexpr (sizeof(T) == 2) {
    float Phi, phi;
    gelu_parts_fast(x, Phi, phi);
    return x * Phi;
  } else {
    return gelu_f(x);
  }
}
template <typename T>
__device__ __forceinline__ float gelu_grad_t(float x) {
  if constexpr (sizeof(T) == 2) {
    float Phi, phi;
    gelu_parts_fast(x, Phi, phi);
    return fmaf(x, phi, Phi);
  } else {
    return gelu_grad_f(x);
  }
}

template <typename T>
__device__ __forceinline__ void ld8(const T* p, float (&v)[8]) {
  if constexpr (sizeof(T) == 2) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(h[e]);
      v[2 * e] = f.x;
      v[2 * e + 1] = f.y;
    }
  } else {
    const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
}
template <typename T>
__device__ __forceinline__ void st8(T* p, const float (&v)[8]) {
  if constexpr (sizeof(T) == 2) {
    uint4 u;
    uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
      w[e] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(p) = u;
  } else {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) gelu_fwd_kernel(const T* __restrict__ x, T* __restrict__ y, int64_t n8) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    float v[8];
    ld8(x + 8 * i, v);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = gelu_t<T>(v[e]);
    st8(y + 8 * i, v);
  }
}

// CTA k: rows [k * rpc, (k+1) * rpc); thread t: columns 8t .. 8t+7 (+ 8 * blockDim per pass).
template <typename T>
__global__ void __launch_bounds__(256) gelu_bwd_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                                                       T* __restrict__ dx, int rows, int cols, int rpc,
                                                       float* __restrict__ part) {
  const int r0 = blockIdx.x * rpc, r1 = min(rows, r0 + rpc);
  for (int c0 = 8 * threadIdx.x; c0 < cols; c0 += 8 * blockDim.x) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int r = r0;
    for (; r + 1 < r1; r += 2) {  // two rows in flight
      const int64_t off0 = (int64_t)r * cols + c0, off1 = off0 + cols;
      float x0[8], g0[8], x1[8], g1[8];
      ld8(x + off0, x0);
      ld8(dy + off0, g0);
      ld8(x + off1, x1);
      ld8(dy + off1, g1);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        x0[e] = g0[e] * gelu_grad_t<T>(x0[e]);
        x1[e] = g1[e] * gelu_grad_t<T>(x1[e]);
        acc[e] += x0[e];
        acc[e] += x1[e];
      }
      st8(dx + off0, x0);
      st8(dx + off1, x1);
    }
    for (; r < r1; ++r) {
      const int64_t off = (int64_t)r * cols + c0;
      float xv[8], gv[8];
      ld8(x + off, xv);
      ld8(dy + off, gv);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        xv[e] = gv[e] * gelu_grad_t<T>(xv[e]);
        acc[e] += xv[e];
      }
      st8(dx + off, xv);
    }
    if (part) {
      float4* o = reinterpret_cast<float4*>(part + (int64_t)blockIdx.x * cols + c0);
      o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
      o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
  }
}

}  // namespace sc

extern "C" int sc_gelu_fwd(const void* x, void* y, int32_t dtype, int64_t n, void* stream) {
  SC_CHECK_ARG(x && y, "sc_gelu_fwd: null pointer");
  SC_CHECK_ARG(dtype == SC_DTYPE_F32 || dtype == SC_DTYPE_BF16, "sc_gelu_fwd: bad dtype");
  if (n % 8 || ((uintptr_t)x | (uintptr_t)y) % 16) {
    set_error("sc_gelu_fwd: needs n %% 8 == 0 and 16-byte aligned buffers");
    return SC_ERR_UNSUPPORTED;
  }
  if (n == 0) return SC_OK;
  const int64_t n8 = n / 8;
  const int64_t want = (n8 + 255) / 256, cap = (int64_t)num_sms() * 16;
  const unsigned blocks = (unsigned)(want < cap ? want : cap);
  if (dtype == SC_DTYPE_F32) gelu_fwd_kernel<float><<<blocks, 256, 0, (cudaStream_t)stream>>>((const float*)x, (float*)y, n8);
  else gelu_fwd_kernel<__nv_bfloat16><<<blocks, 256, 0, (cudaStream_t)stream>>>((const __nv_bfloat16*)x, (__nv_bfloat16*)y, n8);
  SC_CHECK_LAUNCH("gelu_fwd_kernel");
  return SC_OK;
}

extern "C" int sc_gelu_bwd(const void* x, const void* dy, void* dx, int32_t dtype, int32_t rows, int32_t cols,
                           float* dbias, float* partials, void* stream) {
  SC_CHECK_ARG(x && dy && dx, "sc_gelu_bwd: null pointer");
  SC_CHECK_ARG(dtype == SC_DTYPE_F32 || dtype == SC_DTYPE_BF16, "sc_gelu_bwd: bad dtype");
  SC_CHECK_ARG(rows >= 0 && cols >= 1 && (!dbias || partials), "sc_gelu_bwd: bad shape / missing partials");
  if (cols % 8 || ((uintptr_t)x | (uintptr_t)dy | (uintptr_t)dx) % 16) {
    set_error("sc_gelu_bwd: needs cols %% 8 == 0 and 16-byte aligned rows");
    return SC_ERR_UNSUPPORTED;
  }
  if (rows == 0) return SC_OK;
  const int nparts = sc_ln_partials(rows);
  const int rpc = (rows + nparts - 1) / nparts;
  const int threads = min(256, max(32, (cols / 8 + 31) / 32 * 32));
  cudaStream_t st = (cudaStream_t)stream;
  float* part = dbias ? partials : nullptr;
  if (dtype == SC_DTYPE_F32)
    gelu_bwd_kernel<float><<<nparts, threads, 0, st>>>((const float*)x, (const float*)dy, (float*)dx, rows, cols, rpc, part);
  else
    gelu_bwd_kernel<__nv_bfloat16><<<nparts, threads, 0, st>>>((const __nv_bfloat16*)x, (const __nv_bfloat16*)dy,
                                                               (__nv_bfloat16*)dx, rows, cols, rpc, part);
  SC_CHECK_LAUNCH("gelu_bwd_kernel");
  if (dbias) {
    colsum_reduce_kernel<<<(cols + 31) / 32, kRedWarps * 32, 0, st>>>(partials, nparts, cols, dbias);
    SC_CHECK_LAUNCH("colsum_reduce_kernel");
  }
  return SC_OK;
}
