// Fused FFN up-projection for the ranking-exact fp32 mode (CrossEncoder(fp32_gemm="f16x3")):
//   planes(gelu_erf(x1 W1^T + b1))     (R/encoder.py:350-351, :258-259)
// with x1 W1^T as three fp16 tensor-core products from the operand planes (encoder.py _linear_x3h):
//   A = [h0 | h1]  (x1 = h0 + h1, fp16 hi / residual)        [M, 2K]
//   W = [g1 | g0]  (W1 * 2^e = g0 + g1, scaled into fp16)     [N, 2K]
//   acc = [h0 h1] . [g1 g0]  (the two correction products, K' = 2K, magnitude 2^-11)
//       + h0 . g0            (the main product, K)
//   v = acc * s + b1  (s = 2^-e, exact),  g = 0.5 v (1 + erff(v / sqrt 2))  (erff as the fp32 path),
// and the epilogue writes g straight as the W2 GEMM's operand planes [M, 2N] = [fp16_rn(g) | fp16_rn(g -
// fp16_rn(g))] -- the fp32 [M, 3072] activation (written by cuBLAS, read and re-written by the split
// pass, 0.8 ms per layer) never exists.  A value outside fp16 range sets *range (the encoder raises).
//
// Same warp roles as gemm_bias_gelu_kernel (gemm_gelu.cu): warp 0 TMA producer (3-stage ring of
// A [128 x 64] + W [256 x 64] fp16 boxes), warp 1 TMEM owner + single-thread tcgen05.mma (kind::f16,
// fp16 operands, fp32 accumulation, D[128 x 256] double-buffered across tiles), warps 2-5 epilogue
// (tcgen05.ld 64-column chunks, two staging chunks per chunk -- hi and lo planes -- TMA stores).
#include <cuda_fp16.h>

#include "gemm_common.cuh"

namespace sc {
namespace gx {
using namespace tcx;
using gg::BM;
using gg::BN;
using gg::BK;
using gg::ROWB;
using gg::NTHREADS;
using gg::A_BYTES;
using gg::STAGE;
using gg::STG_BYTES;
using gg::epi_sync;
using gg::tma_store_2d;

constexpr int NS = 3;  // stages: 3 x 48 KB + 2 x 2 staging chunks of 16 KB
constexpr int SMEM_STG = NS * STAGE;
constexpr int SMEM_BAR = SMEM_STG + 4 * STG_BYTES;
constexpr int SMEM_BIAS = SMEM_BAR + (2 * NS + 4) * 8 + 16;
constexpr int SMEM_TOTAL = SMEM_BIAS + BN * 4;

// fp16 A and B (a_format = b_format = 0), fp32 D, both K-major.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// kGelu: epilogue = bias + erff GELU + fp16 hi/lo planes (tmO: fp16 [M, 2N], 64-column boxes);
// else fp32 out = acc * scale (+ bias) (tmO: fp32 [M, N], 32-column boxes).  kb = 0, or 8 when the
// planes carry a constant column / bias columns (sc_split_f16x2 onehot, the QKV weight planes): the
// correction k-blocks then span 2K + 8 columns and the main product's W block starts at K + 8; the
// maps' widths make TMA zero-fill whatever a 64-column box reads past them.
template <bool kGelu>
__global__ void __launch_bounds__(NTHREADS, 1) gemm_x3h_kernel(
    const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
    const __grid_constant__ CUtensorMap tmO, const float* __restrict__ bias, float scale, int32_t* __restrict__ range,
    int M, int N, int K, int kb8) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sm0 = smem_u32(smem);
  const uint32_t bar0 = sm0 + SMEM_BAR;
  const uint32_t full_bar = bar0, empty_bar = bar0 + 8 * NS, acc_full = bar0 + 16 * NS, acc_empty = acc_full + 16;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + SMEM_BAR + (2 * NS + 4) * 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_n = N / BN, tiles = ((M + BM - 1) / BM) * tiles_n;
  const int nk_c = (2 * K + kb8 + BK - 1) / BK, nk = nk_c + (K + kb8 + BK - 1) / BK;  // corrections, then main

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      mbar_init(empty_bar + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full + 8 * b, 1);
      mbar_init(acc_empty + 8 * b, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------------------- TMA producer
    if (lane == 0) {
      prefetch_map(&tmA);
      prefetch_map(&tmB);
      int it = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % NS;
          if (it >= NS) mbar_wait(empty_bar + 8 * s, ((it / NS) & 1) ^ 1);
          // corrections: A[:, kb*64] x W[:, kb*64] over [h0 | h1] x [g1 | g0]; main: h0 x g0
          const int ca = kb < nk_c ? kb * BK : (kb - nk_c) * BK;
          const int cb = kb < nk_c ? kb * BK : K + kb8 + (kb - nk_c) * BK;
          mbar_expect_tx(full_bar + 8 * s, STAGE);
          tma_load_2d(sm0 + s * STAGE, &tmA, ca, m0, full_bar + 8 * s);
          tma_load_2d(sm0 + s * STAGE + A_BYTES, &tmB, cb, n0, full_bar + 8 * s);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_f16(BM, BN);
      int it = 0, i = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
        const int buf = i & 1;
        if (i >= 2) mbar_wait(acc_empty + 8 * buf, ((i >> 1) & 1) ^ 1);  // epilogue drained this buffer
        tc_fence_after();
        const uint32_t tD = tmem + buf * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % NS;
          mbar_wait(full_bar + 8 * s, (it / NS) & 1);
          tc_fence_after();
          const uint64_t ad = sw128_desc(sm0 + s * STAGE), bd = sw128_desc(sm0 + s * STAGE + A_BYTES);
#pragma unroll
          for (int ks = 0; ks < BK / 16; ++ks) mma_ss(tD, ad + 2 * ks, bd + 2 * ks, idesc, (kb > 0 || ks > 0));
          tc_commit(empty_bar + 8 * s);
        }
        tc_commit(acc_full + 8 * buf);
      }
    }
  } else {
    // ------------------------------------------------------------- epilogue
    const int q = warp & 3;       // TMEM lane quadrant of this warp
    const int r = q * 32 + lane;  // row within the tile
    const int et = threadIdx.x - 64;
    bool bad = false;
    int i = 0, chunk = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
      const int buf = i & 1;
      const int m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
      float* sb = reinterpret_cast<float*>(smem + SMEM_BIAS);
      for (int c = et; c < BN; c += 128) sb[c] = bias ? __ldg(bias + n0 + c) : 0.f;
      epi_sync();
      mbar_wait(acc_full + 8 * buf, (i >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + buf * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 64; ++c, ++chunk) {
        uint32_t v[64];
        TC_LD32(taddr + c * 64, v);
        TC_LD32(taddr + c * 64 + 32, (&v[32]));
        tc_wait_ld();
        if (c == BN / 64 - 1) {  // accumulator fully read: hand the TMEM buffer back
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(acc_empty + 8 * buf);
        }
        const float* bc = sb + c * 64;
        uint32_t hi[32], lo[32];  // kGelu: fp16 hi / lo pairs; else the two 32-column fp32 halves
        if constexpr (kGelu) {
#pragma unroll
          for (int e = 0; e < 64; e += 2) {
            float x0 = fmaf(__uint_as_float(v[e]), scale, bc[e]);
            float x1 = fmaf(__uint_as_float(v[e + 1]), scale, bc[e + 1]);
            x0 = 0.5f * x0 * (1.f + erff(x0 * 0.70710678118654752440f));
            x1 = 0.5f * x1 * (1.f + erff(x1 * 0.70710678118654752440f));
            bad |= !(fabsf(x0) < 65504.f && fabsf(x1) < 65504.f);
            const __half2 h = __floats2half2_rn(x0, x1);
            const float2 hf = __half22float2(h);
            const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
            hi[e / 2] = *reinterpret_cast<const uint32_t*>(&h);
            lo[e / 2] = *reinterpret_cast<const uint32_t*>(&l);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            hi[e] = __float_as_uint(fmaf(__uint_as_float(v[e]), scale, bc[e]));
            lo[e] = __float_as_uint(fmaf(__uint_as_float(v[32 + e]), scale, bc[32 + e]));
          }
        }
        // staging pair (chunk & 1) is free once the stores issued two chunks ago (two groups per chunk)
        // have read it
        const uint32_t stg = sm0 + SMEM_STG + (chunk & 1) * 2 * STG_BYTES;
        if (et == 0) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
        epi_sync();
#pragma unroll
        for (int p16 = 0; p16 < 8; ++p16) {
          const uint32_t addr = stg + r * ROWB + ((p16 ^ (r & 7)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(hi[4 * p16]), "r"(hi[4 * p16 + 1]),
                       "r"(hi[4 * p16 + 2]), "r"(hi[4 * p16 + 3])
                       : "memory");
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr + STG_BYTES), "r"(lo[4 * p16]),
                       "r"(lo[4 * p16 + 1]), "r"(lo[4 * p16 + 2]), "r"(lo[4 * p16 + 3])
                       : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        epi_sync();
        if (et == 0) {
          if constexpr (kGelu) {
            tma_store_2d(&tmO, stg, n0 + c * 64, m0);                  // hi plane: columns [0, N)
            tma_store_2d(&tmO, stg + STG_BYTES, N + n0 + c * 64, m0);  // lo plane: columns [N, 2N)
          } else {
            tma_store_2d(&tmO, stg, n0 + c * 64, m0);                  // fp32 columns c*64 .. +31
            tma_store_2d(&tmO, stg + STG_BYTES, n0 + c * 64 + 32, m0); //              c*64+32 .. +63
          }
        }
      }
    }
    if (et == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (bad && range) atomicExch(range, 1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

}  // namespace gx
}  // namespace sc

using namespace sc;

namespace sc {
namespace gx {
// fp32 [rows][cols] as a 2-D map with 32-column (128 B) x box_rows boxes, 128B swizzle.
static bool make_map_f32(CUtensorMap* m, const void* base, int64_t cols, int64_t rows, int64_t ld, int box_rows) {
  static tcx::EncodeFn enc = nullptr;
  if (!enc) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    enc = reinterpret_cast<tcx::EncodeFn>(ptr);
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {32u, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool kGelu>
static int launch_x3h(const CUtensorMap& mA, const CUtensorMap& mB, const CUtensorMap& mO, const float* bias,
                      float scale, int32_t* range, int M, int N, int K, int kb8, cudaStream_t st, const char* name) {
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (num_sms <= 0) num_sms = 148;
  }
  static bool attr = false;
  const size_t smem = SMEM_TOTAL + 1024;
  if (!attr) {
    if (cudaFuncSetAttribute(gemm_x3h_kernel<kGelu>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess) {
      set_error("%s: shared memory request of %zu bytes failed", name, smem);
      return SC_ERR_UNSUPPORTED;
    }
    attr = true;
  }
  const int tiles = ((M + BM - 1) / BM) * (N / BN);
  gemm_x3h_kernel<kGelu><<<tiles < num_sms ? tiles : num_sms, NTHREADS, smem, st>>>(mA, mB, mO, bias, scale, range,
                                                                                    M, N, K, kb8);
  SC_CHECK_LAUNCH("gemm_x3h_kernel");
  return SC_OK;
}
}  // namespace gx
}  // namespace sc

extern "C" int sc_gemm_x3h_gelu_planes(const void* a_planes, int64_t lda, const void* w_planes, int64_t ldw,
                                       float w_scale, const float* bias, void* out_planes, int64_t ldo,
                                       int32_t* range_status, int32_t M, int32_t N, int32_t K, void* stream) {
  using namespace gx;
  SC_CHECK_ARG(a_planes && w_planes && out_planes && M >= 0 && N >= 1 && K >= 1,
               "sc_gemm_x3h_gelu_planes: bad arguments");
  if (M == 0) return SC_OK;
  if (N % BN || K % BK || lda < 2LL * K || ldw < 2LL * K || ldo < 2LL * N || (lda * 2) % 16 || (ldw * 2) % 16 ||
      (ldo * 2) % 16 || (((uintptr_t)a_planes | (uintptr_t)w_planes | (uintptr_t)out_planes) & 15) ||
      (bias && ((uintptr_t)bias & 7))) {
    set_error("sc_gemm_x3h_gelu_planes: needs N %% 256 == 0, K %% 64 == 0 and 16-byte aligned rows");
    return SC_ERR_UNSUPPORTED;
  }
  // fp16 planes through the 2-byte maps (TMA copies bytes; the MMA kind reads them as fp16)
  CUtensorMap mA, mB, mO;
  if (!make_map(&mA, a_planes, 2LL * K, M, lda, BM) || !make_map(&mB, w_planes, 2LL * K, N, ldw, BN) ||
      !make_map(&mO, out_planes, 2LL * N, M, ldo, BM)) {
    set_error("sc_gemm_x3h_gelu_planes: cuTensorMapEncodeTiled failed");
    return SC_ERR_UNSUPPORTED;
  }
  return launch_x3h<true>(mA, mB, mO, bias, w_scale, range_status, M, N, K, 0, (cudaStream_t)stream,
                         "sc_gemm_x3h_gelu_planes");
}

extern "C" int sc_gemm_x3h(const void* a_planes, int64_t lda, const void* w_planes, int64_t ldw, float w_scale,
                           float* out, int64_t ldo, int32_t M, int32_t N, int32_t K, int32_t bias_cols, void* stream) {
  using namespace gx;
  SC_CHECK_ARG(a_planes && w_planes && out && M >= 0 && N >= 1 && K >= 1 && (bias_cols == 0 || bias_cols == 8),
               "sc_gemm_x3h: bad arguments");
  if (M == 0) return SC_OK;
  const int64_t acols = 2LL * K + bias_cols, wcols = 2LL * K + 2 * bias_cols;
  if (N % BN || K % BK || lda < acols || ldw < wcols || ldo < N || (lda * 2) % 16 || (ldw * 2) % 16 ||
      (ldo * 4) % 16 || (((uintptr_t)a_planes | (uintptr_t)w_planes | (uintptr_t)out) & 15)) {
    set_error("sc_gemm_x3h: needs N %% 256 == 0, K %% 64 == 0 and 16-byte aligned rows");
    return SC_ERR_UNSUPPORTED;
  }
  CUtensorMap mA, mB, mO;
  if (!make_map(&mA, a_planes, acols, M, lda, BM) || !make_map(&mB, w_planes, wcols, N, ldw, BN) ||
      !make_map_f32(&mO, out, N, M, ldo, BM)) {
    set_error("sc_gemm_x3h: cuTensorMapEncodeTiled failed");
    return SC_ERR_UNSUPPORTED;
  }
  return launch_x3h<false>(mA, mB, mO, nullptr, w_scale, nullptr, M, N, K, bias_cols, (cudaStream_t)stream,
                           "sc_gemm_x3h");
}
