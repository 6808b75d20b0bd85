// Fused AdamW step over one flat fp32 parameter buffer (R/training.py:114-137):
//   m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2
//   w -= lr_t * ((m / bc1) / (sqrt(v / bc2) + eps) + weight_decay * w)
// One pass: reads w, g, m, v and writes w, m, v (28 bytes per parameter; + 2 for the optional bf16
// shadow copy the bf16 forward reads), float4 vectors, the update arithmetic in fp64 like the
// reference (moments stored in fp32).
#include "common.cuh"

namespace sc {

struct AdamCoef {
  double lr, b1, b2, eps, wd, ibc1, ibc2;
};

__device__ __forceinline__ void adam_one(float& w, float g, float& m, float& v, const AdamCoef& c) {
  const double md = c.b1 * (double)m + (1.0 - c.b1) * (double)g;
  const double vd = c.b2 * (double)v + (1.0 - c.b2) * (double)g * (double)g;
  const double upd = (md * c.ibc1) / (sqrt(vd * c.ibc2) + c.eps);
  w = (float)((double)w - c.lr * (upd + c.wd * (double)w));
  m = (float)md;
  v = (float)vd;
}

__global__ void __launch_bounds__(256) adamw_kernel(float* __restrict__ w, const float* __restrict__ g,
                                                    float* __restrict__ m, float* __restrict__ v,
                                                    __nv_bfloat16* __restrict__ w16, int64_t n, AdamCoef c) {
  const int64_t n4 = n >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 wv = reinterpret_cast<float4*>(w)[i];
    const float4 gv = reinterpret_cast<const float4*>(g)[i];
    float4 mv = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    adam_one(wv.x, gv.x, mv.x, vv.x, c);
    adam_one(wv.y, gv.y, mv.y, vv.y, c);
    adam_one(wv.z, gv.z, mv.z, vv.z, c);
    adam_one(wv.w, gv.w, mv.w, vv.w, c);
    reinterpret_cast<float4*>(w)[i] = wv;
    reinterpret_cast<float4*>(m)[i] = mv;
    reinterpret_cast<float4*>(v)[i] = vv;
    if (w16) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(wv.x, wv.y), hi = __floats2bfloat162_rn(wv.z, wv.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&lo);
      u.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(w16)[i] = u;
    }
  }
  for (int64_t i = (n4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    adam_one(w[i], g[i], m[i], v[i], c);
    if (w16) w16[i] = __float2bfloat16_rn(w[i]);
  }
}

}  // namespace sc

using namespace sc;

extern "C" int sc_adamw_step(float* w, const float* g, float* m, float* v, void* w_bf16, int64_t n, double lr,
                             double beta1, double beta2, double eps, double weight_decay, int64_t step, void* stream) {
  SC_CHECK_ARG(w && g && m && v, "sc_adamw_step: null pointer");
  SC_CHECK_ARG(n >= 0 && step >= 1, "sc_adamw_step: bad size or step");
  SC_CHECK_ARG(((uintptr_t)w | (uintptr_t)g | (uintptr_t)m | (uintptr_t)v | (uintptr_t)w_bf16) % 16 == 0,
               "sc_adamw_step: buffers must be 16-byte aligned");
  if (n == 0) return SC_OK;
  AdamCoef c;
  c.lr = lr; c.b1 = beta1; c.b2 = beta2; c.eps = eps; c.wd = weight_decay;
  c.ibc1 = 1.0 / (1.0 - pow(beta1, (double)step));
  c.ibc2 = 1.0 / (1.0 - pow(beta2, (double)step));
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = ((n >> 2) + 255) / 256;
  const unsigned blocks = (unsigned)(want < (int64_t)sms * 8 ? (want > 0 ? want : 1) : (int64_t)sms * 8);
  adamw_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(w, g, m, v, (__nv_bfloat16*)w_bf16, n, c);
  SC_CHECK_LAUNCH("adamw_kernel");
  return SC_OK;
}
