// L1 band kernels ⊡_w / ⊙_w (R/band.py:154-236) on device.
//   band_scores: out[b,i,j] = q[b,i,:] . k[b,i+j-w,:]  (0 when i+j-w is out of range)
//   band_apply:  out[b,i,:] = sum_{valid j} p[b,i,j] v[b,i+j-w,:]
// One warp per (batch, row); fp32 accumulation in ascending feature / slot
// order.  These are standalone array kernels for the band API; the encoder
// path never materialises a band (the fused attention kernels do not).
#include "common.cuh"

namespace sc {

template <typename T>
__global__ void band_scores_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                   T* __restrict__ out, int64_t rows_total, int s, int t, int d,
                                   int w) {
  int lane = threadIdx.x & 31;
  int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows_total) return;
  int64_t b = r / s;
  int i = (int)(r % s);
  int width = 2 * w + 1;
  const T* qr = q + r * d;
  const T* kb = k + b * (int64_t)t * d;
  for (int j = lane; j < width; j += 32) {
    int tg = i + j - w;
    float acc = 0.f;
    if (tg >= 0 && tg < t) {
      const T* kr = kb + (int64_t)tg * d;
      for (int c = 0; c < d; ++c) acc = fmaf(to_f32(qr[c]), to_f32(kr[c]), acc);
    }
    out[r * width + j] = from_f32<T>(acc);
  }
}

template <typename T>
__global__ void band_apply_kernel(const T* __restrict__ p, const T* __restrict__ v,
                                  T* __restrict__ out, int64_t rows_total, int s, int t, int d,
                                  int w) {
  int lane = threadIdx.x & 31;
  int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows_total) return;
  int64_t b = r / s;
  int i = (int)(r % s);
  int width = 2 * w + 1;
  const T* pr = p + r * width;
  const T* vb = v + b * (int64_t)t * d;
  int jlo = max(0, w - i), jhi = min(width, t + w - i);  // valid slot range
  for (int c = lane; c < d; c += 32) {
    float acc = 0.f;
    for (int j = jlo; j < jhi; ++j) acc = fmaf(to_f32(pr[j]), to_f32(vb[(int64_t)(i + j - w) * d + c]), acc);
    out[r * d + c] = from_f32<T>(acc);
  }
}

// Adjoints (R/band.py:239-274), gather form (no atomics): one warp per output row.
//   grad_q[b,i,:] = sum_j g[b,i,j] k[b,i+j-w,:]      grad_k[b,r,:] = sum_j g[b,r-j+w,j] q[b,r-j+w,:]
//   grad_p[b,i,j] = go[b,i,:] . v[b,i+j-w,:] (0 invalid)   grad_v[b,r,:] = sum_j p[b,r-j+w,j] go[b,r-j+w,:]
template <typename T>
__global__ void band_rows_adjoint_kernel(const T* __restrict__ g, const T* __restrict__ x,
                                         T* __restrict__ out, int64_t rows_total, int s, int t, int d, int w) {
  // out[b,i,:] = sum_{valid j} g[b,i,j] x[b,i+j-w,:]   (grad_q of scores; same shape as band_apply)
  int lane = threadIdx.x & 31;
  int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows_total) return;
  int64_t b = r / s;
  int i = (int)(r % s);
  int width = 2 * w + 1;
  const T* gr = g + r * width;
  const T* xb = x + b * (int64_t)t * d;
  int jlo = max(0, w - i), jhi = min(width, t + w - i);
  for (int c = lane; c < d; c += 32) {
    float acc = 0.f;
    for (int j = jlo; j < jhi; ++j) acc = fmaf(to_f32(gr[j]), to_f32(xb[(int64_t)(i + j - w) * d + c]), acc);
    out[r * d + c] = from_f32<T>(acc);
  }
}

template <typename T>
__global__ void band_cols_adjoint_kernel(const T* __restrict__ g, const T* __restrict__ x,
                                         T* __restrict__ out, int64_t rows_total, int s, int t, int d, int w) {
  // out[b,r,:] = sum_j g[b,r-j+w,j] x[b,r-j+w,:] over source rows in [0,s)   (grad_k / grad_v)
  int lane = threadIdx.x & 31;
  int64_t rr = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (rr >= rows_total) return;
  int64_t b = rr / t;
  int r = (int)(rr % t);
  int width = 2 * w + 1;
  const T* gb = g + b * (int64_t)s * width;
  const T* xb = x + b * (int64_t)s * d;
  int jlo = max(0, r + w - (s - 1)), jhi = min(width, r + w + 1);
  for (int c = lane; c < d; c += 32) {
    float acc = 0.f;
    for (int j = jlo; j < jhi; ++j) {
      int i = r - j + w;
      acc = fmaf(to_f32(gb[(int64_t)i * width + j]), to_f32(xb[(int64_t)i * d + c]), acc);
    }
    out[rr * d + c] = from_f32<T>(acc);
  }
}

}  // namespace sc

using namespace sc;

static int band_check(const void* a, const void* b, const void* out, int64_t batch, int32_t s, int32_t t,
                      int32_t d, int32_t window, int32_t dtype) {
  SC_CHECK_ARG(window >= 0, "window must be a non-negative integer, got %d", window);
  SC_CHECK_ARG(a && b && out, "band kernel: null pointer");
  SC_CHECK_ARG(batch >= 0 && s >= 0 && t >= 1 && d >= 1, "band kernel: bad shape");
  SC_CHECK_ARG(dtype == SC_DTYPE_F32 || dtype == SC_DTYPE_BF16, "band kernel: bad dtype");
  return SC_OK;
}

extern "C" int sc_band_scores(const void* q, const void* k, void* out, int64_t batch, int32_t s,
                              int32_t t, int32_t d, int32_t window, int32_t dtype, void* stream) {
  int rc = band_check(q, k, out, batch, s, t, d, window, dtype);
  if (rc) return rc;
  int64_t rows = batch * s;
  if (rows == 0) return SC_OK;
  unsigned blocks = (unsigned)((rows + 7) / 8);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SC_DTYPE_F32)
    band_scores_kernel<float><<<blocks, 256, 0, st>>>((const float*)q, (const float*)k, (float*)out,
                                                      rows, s, t, d, window);
  else
    band_scores_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
        (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (__nv_bfloat16*)out, rows, s, t, d, window);
  SC_CHECK_LAUNCH("band_scores_kernel");
  return SC_OK;
}

extern "C" int sc_band_apply(const void* p, const void* v, void* out, int64_t batch, int32_t s,
                             int32_t t, int32_t d, int32_t window, int32_t dtype, void* stream) {
  int rc = band_check(p, v, out, batch, s, t, d, window, dtype);
  if (rc) return rc;
  int64_t rows = batch * s;
  if (rows == 0) return SC_OK;
  unsigned blocks = (unsigned)((rows + 7) / 8);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SC_DTYPE_F32)
    band_apply_kernel<float><<<blocks, 256, 0, st>>>((const float*)p, (const float*)v, (float*)out,
                                                     rows, s, t, d, window);
  else
    band_apply_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
        (const __nv_bfloat16*)p, (const __nv_bfloat16*)v, (__nv_bfloat16*)out, rows, s, t, d, window);
  SC_CHECK_LAUNCH("band_apply_kernel");
  return SC_OK;
}


extern "C" int sc_band_scores_backward(const void* grad_band, const void* q, const void* k, void* grad_q,
                                       void* grad_k, int64_t batch, int32_t s, int32_t t, int32_t d,
                                       int32_t window, int32_t dtype, void* stream) {
  int rc = band_check(q, k, grad_band, batch, s, t, d, window, dtype);
  if (rc) return rc;
  SC_CHECK_ARG(grad_q && grad_k, "band backward: null gradient pointer");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rq = batch * s, rk = batch * t;
  const unsigned bq = (unsigned)((rq + 7) / 8), bk = (unsigned)((rk + 7) / 8);
  if (dtype == SC_DTYPE_F32) {
    if (rq) band_rows_adjoint_kernel<float><<<bq, 256, 0, st>>>((const float*)grad_band, (const float*)k,
                                                               (float*)grad_q, rq, s, t, d, window);
    if (rk) band_cols_adjoint_kernel<float><<<bk, 256, 0, st>>>((const float*)grad_band, (const float*)q,
                                                               (float*)grad_k, rk, s, t, d, window);
  } else {
    using B = __nv_bfloat16;
    if (rq) band_rows_adjoint_kernel<B><<<bq, 256, 0, st>>>((const B*)grad_band, (const B*)k, (B*)grad_q, rq, s,
                                                           t, d, window);
    if (rk) band_cols_adjoint_kernel<B><<<bk, 256, 0, st>>>((const B*)grad_band, (const B*)q, (B*)grad_k, rk, s,
                                                           t, d, window);
  }
  SC_CHECK_LAUNCH("band_scores_backward");
  return SC_OK;
}

extern "C" int sc_band_apply_backward(const void* grad_out, const void* p, const void* v, void* grad_p,
                                      void* grad_v, int64_t batch, int32_t s, int32_t t, int32_t d, int32_t window,
                                      int32_t dtype, void* stream) {
  int rc = band_check(p, v, grad_out, batch, s, t, d, window, dtype);
  if (rc) return rc;
  SC_CHECK_ARG(grad_p && grad_v, "band backward: null gradient pointer");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rp = batch * s, rv = batch * t;
  const unsigned bp = (unsigned)((rp + 7) / 8), bv = (unsigned)((rv + 7) / 8);
  // grad_p = band_scores(grad_out, v); grad_v = cols-adjoint of (p, grad_out)
  if (dtype == SC_DTYPE_F32) {
    if (rp) band_scores_kernel<float><<<bp, 256, 0, st>>>((const float*)grad_out, (const float*)v, (float*)grad_p,
                                                         rp, s, t, d, window);
    if (rv) band_cols_adjoint_kernel<float><<<bv, 256, 0, st>>>((const float*)p, (const float*)grad_out,
                                                               (float*)grad_v, rv, s, t, d, window);
  } else {
    using B = __nv_bfloat16;
    if (rp) band_scores_kernel<B><<<bp, 256, 0, st>>>((const B*)grad_out, (const B*)v, (B*)grad_p, rp, s, t, d,
                                                     window);
    if (rv) band_cols_adjoint_kernel<B><<<bv, 256, 0, st>>>((const B*)p, (const B*)grad_out, (B*)grad_v, rv, s, t,
                                                           d, window);
  }
  SC_CHECK_LAUNCH("band_apply_backward");
  return SC_OK;
}
