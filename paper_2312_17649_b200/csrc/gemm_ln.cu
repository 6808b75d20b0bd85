// Fused output projection + residual + LayerNorm for the bf16 encoder
// (R/encoder.py:345-347 and :352-354, LN eps 1e-12 at :41):
//   out = LN(resid + A W^T + b) * gamma + beta,   W: [768, K]
// in one tcgen05 GEMM.  A LayerNorm row spans all 768 output columns, more than
// one CTA's TMEM holds at M = 128, so a cluster of three CTAs (one per 256-column
// slice, same 128 rows) computes a row block: each CTA drains its slice into
// per-row (mean, M2) partials, pushes them into its two peers' shared memory
// (st.shared::cluster + a remote mbarrier arrive), combines the three partials
// (Chan et al.) and normalises its own columns.  The separate residual +
// LayerNorm pass (read y and resid, write out: 6 B/element, 11% of the step)
// disappears; the epilogue reads resid (2 B, TMA-staged) and writes out (2 B).
//
// Roles per CTA as in gemm_gelu.cu (warp 0 TMA, warp 1 MMA, warps 2-5
// epilogue); TMEM double-buffered.  The epilogue makes two passes over its
// 128 x 256 accumulator: y = acc + bias + resid written back into TMEM with
// shifted row sums, then (after the exchange) normalise + store.
#include "gemm_common.cuh"

namespace sc {
namespace gl {
using namespace tcx;
using namespace gg;

constexpr int NS = 3, NCL = 3;  // stages (smem: 3 x 48 KB + staging + stats), CTAs per cluster (3 x 256 = 768 columns)
constexpr int SMEM_STG = NS * STAGE;
constexpr int SMEM_RES = SMEM_STG + 2 * STG_BYTES;            // 2 x 16 KB residual chunks (columns 0-127)
constexpr int SMEM_STATS = SMEM_RES + 2 * STG_BYTES;          // [2 bufs][3 ranks][128 rows] float2 (mean, M2)
constexpr int STATS_BYTES = 2 * NCL * BM * 8;
constexpr int SMEM_VEC = SMEM_STATS + STATS_BYTES;             // bias, gamma, beta slices (3 x 256 fp32)
constexpr int SMEM_BAR = SMEM_VEC + 3 * BN * 4;
constexpr int SMEM_TOTAL = SMEM_BAR + (2 * NS + 8) * 8 + 16;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_peer(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f2(uint32_t addr, float a, float b) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}
__global__ void __cluster_dims__(NCL, 1, 1) __launch_bounds__(NTHREADS, 1) gemm_res_ln_kernel(
    const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
    const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmR, const float* __restrict__ bias,
    const float* __restrict__ gamma,
    const float* __restrict__ beta, float* __restrict__ out_f32, int64_t ldf, int32_t* __restrict__ bad,
    int M, int K) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sm0 = smem_u32(smem);
  const uint32_t bar0 = sm0 + SMEM_BAR;
  const uint32_t full_bar = bar0, empty_bar = bar0 + 8 * NS, acc_full = bar0 + 16 * NS, acc_empty = acc_full + 16,
                 stats_bar = acc_full + 32;
  const uint32_t res_bar = stats_bar + 16;  // [2]: residual columns 0-127 / 128-255 landed
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + SMEM_BAR + (2 * NS + 8) * 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cl = blockIdx.x / NCL, ncl = gridDim.x / NCL;
  const int n0 = (int)rank * BN;
  const int tiles = (M + BM - 1) / BM, nk = K / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      mbar_init(empty_bar + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full + 8 * b, 1);
      mbar_init(acc_empty + 8 * b, 4);
      mbar_init(stats_bar + 8 * b, BM * (NCL - 1));  // every epilogue thread of both peers
      mbar_init(res_bar + 8 * b, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers of every CTA initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      prefetch_map(&tmA);
      prefetch_map(&tmB);
      int it = 0;
      for (int t = cl; t < tiles; t += ncl) {
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % NS;
          if (it >= NS) mbar_wait(empty_bar + 8 * s, ((it / NS) & 1) ^ 1);
          mbar_expect_tx(full_bar + 8 * s, STAGE);
          tma_load_2d(sm0 + s * STAGE, &tmA, kb * BK, t * BM, full_bar + 8 * s);
          tma_load_2d(sm0 + s * STAGE + A_BYTES, &tmB, kb * BK, n0, full_bar + 8 * s);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(BM, BN, 0);
      int it = 0, i = 0;
      for (int t = cl; t < tiles; t += ncl, ++i) {
        const int buf = i & 1;
        if (i >= 2) mbar_wait(acc_empty + 8 * buf, ((i >> 1) & 1) ^ 1);
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
    const int q = warp & 3, r = q * 32 + lane, et = threadIdx.x - 64;
    float* vb = reinterpret_cast<float*>(smem + SMEM_VEC);  // bias | gamma | beta of this slice
    for (int c = et; c < BN; c += 128) {
      vb[c] = bias ? __ldg(bias + n0 + c) : 0.f;
      vb[BN + c] = __ldg(gamma + n0 + c);
      vb[2 * BN + c] = __ldg(beta + n0 + c);
    }
    epi_sync();
    const float inv_n = 1.f / (float)(NCL * BN);
    int i = 0, chunk = 0;
    for (int t = cl; t < tiles; t += ncl, ++i) {
      const int buf = i & 1;
      const int m0 = t * BM, row = m0 + r;
      const bool live = row < M;
      // residual tile by TMA (four 64-column chunks, 128B swizzle): columns 0-127 into
      // the dedicated buffers, 128-255 into the output staging buffers once the
      // previous tile's stores have read them; both land while the mainloop runs
      if (et == 0) {
        if (i == 0) {  // later tiles' columns 0-127 were prefetched after the previous pass 1
          mbar_expect_tx(res_bar, 2 * STG_BYTES);
          tma_load_2d(sm0 + SMEM_RES, &tmR, n0, m0, res_bar);
          tma_load_2d(sm0 + SMEM_RES + STG_BYTES, &tmR, n0 + 64, m0, res_bar);
        }
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        mbar_expect_tx(res_bar + 8, 2 * STG_BYTES);
        tma_load_2d(sm0 + SMEM_STG, &tmR, n0 + 128, m0, res_bar + 8);
        tma_load_2d(sm0 + SMEM_STG + STG_BYTES, &tmR, n0 + 192, m0, res_bar + 8);
      }
      mbar_wait(acc_full + 8 * buf, (i >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + buf * BN;
      // pass 1: y = acc + bias + resid, written back over the accumulator in TMEM;
      // shifted sums around the row's first value give the slice mean and
      // centred M2 in one sweep.
      float piv = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        if (c0 == 0 || c0 == 128) mbar_wait(res_bar + (c0 ? 8 : 0), i & 1);
        const int ch = c0 >> 6;  // 64-column residual chunk
        const uint8_t* rbase = smem + (ch < 2 ? SMEM_RES + ch * STG_BYTES : SMEM_STG + (ch - 2) * STG_BYTES);
        uint32_t v[32];
        TC_LD32(taddr + c0, v);
        uint4 rw[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int p16 = ((c0 & 63) >> 3) + k;
          rw[k] = *reinterpret_cast<const uint4*>(rbase + r * ROWB + ((p16 ^ (r & 7)) << 4));
        }
        tc_wait_ld();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&rw[k]);
#pragma unroll
          for (int e2 = 0; e2 < 4; ++e2) {
            const int e = 8 * k + 2 * e2;
            const float2 rf = __bfloat1622float2(h[e2]);
            const float2 bb = *reinterpret_cast<const float2*>(vb + c0 + e);
            const float y0 = __uint_as_float(v[e]) + bb.x + rf.x, y1 = __uint_as_float(v[e + 1]) + bb.y + rf.y;
            if (c0 == 0 && e == 0) piv = y0;
            const float d0 = y0 - piv, d1 = y1 - piv;
            s1 += d0 + d1;
            s2 = fmaf(d0, d0, fmaf(d1, d1, s2));
            v[e] = __float_as_uint(y0);
            v[e + 1] = __float_as_uint(y1);
          }
        }
        TC_ST32(taddr + c0, v);
      }
      tc_wait_st();
      epi_sync();  // residual chunks read: staging free for the output, dedicated buffers for the next tile
      if (et == 0 && t + ncl < tiles) {
        mbar_expect_tx(res_bar, 2 * STG_BYTES);
        tma_load_2d(sm0 + SMEM_RES, &tmR, n0, (t + ncl) * BM, res_bar);
        tma_load_2d(sm0 + SMEM_RES + STG_BYTES, &tmR, n0 + 64, (t + ncl) * BM, res_bar);
      }
      const float mean_s = piv + s1 * (1.f / BN);
      const float m2 = fmaxf(s2 - s1 * s1 * (1.f / BN), 0.f);
      // exchange (mean, M2) of the three 256-column slices through distributed shared memory
      const uint32_t slot = sm0 + SMEM_STATS + (buf * NCL * BM) * 8;
      *reinterpret_cast<float2*>(smem + SMEM_STATS + ((buf * NCL + rank) * BM + r) * 8) = make_float2(mean_s, m2);
#pragma unroll
      for (int pr = 1; pr < NCL; ++pr) {
        const uint32_t peer = (rank + pr) % NCL;
        st_cluster_f2(map_peer(slot + (rank * BM + r) * 8, peer), mean_s, m2);
      }
      // each thread's remote arrive releases its own stores (no cluster-wide fence)
#pragma unroll
      for (int pr = 1; pr < NCL; ++pr) arrive_remote(map_peer(stats_bar + 8 * buf, (rank + pr) % NCL));
      wait_cluster(stats_bar + 8 * buf, (i >> 1) & 1);
      float mean = 0.f;
      float2 st[NCL];
#pragma unroll
      for (int k = 0; k < NCL; ++k) {
        st[k] = *reinterpret_cast<const float2*>(smem + SMEM_STATS + ((buf * NCL + k) * BM + r) * 8);
        mean += st[k].x;
      }
      mean *= 1.f / NCL;
      float M2 = 0.f;
#pragma unroll
      for (int k = 0; k < NCL; ++k) {
        const float d = st[k].x - mean;
        M2 += st[k].y + BN * d * d;
      }
      const float rstd = rsqrtf(M2 * inv_n + 1e-12f);
      // pass 2: normalise y (re-read from TMEM), bf16 -> staging -> TMA store;
      // optional fp32 copy; non-finite flag
      bool nf = false;
#pragma unroll 1
      for (int c = 0; c < BN / 64; ++c, ++chunk) {
        uint32_t pk[32];
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t v[32];
          TC_LD32(taddr + c * 64 + half * 32, v);
          tc_wait_ld();
          if (c == BN / 64 - 1 && half == 1) {  // accumulator fully read: hand the TMEM buffer back
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty + 8 * buf);
          }
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const int cc = c * 64 + half * 32 + e;
            const float2 gg2 = *reinterpret_cast<const float2*>(vb + BN + cc);
            const float2 bt2 = *reinterpret_cast<const float2*>(vb + 2 * BN + cc);
            const float o0 = fmaf((__uint_as_float(v[e]) - mean) * rstd, gg2.x, bt2.x);
            const float o1 = fmaf((__uint_as_float(v[e + 1]) - mean) * rstd, gg2.y, bt2.y);
            nf |= !(isfinite(o0) && isfinite(o1));
            if (out_f32 && live)
              *reinterpret_cast<float2*>(out_f32 + (int64_t)row * ldf + n0 + cc) = make_float2(o0, o1);
            __nv_bfloat162 h2 = __floats2bfloat162_rn(o0, o1);
            pk[half * 16 + e / 2] = *reinterpret_cast<uint32_t*>(&h2);
          }
        }
        const uint32_t stg = sm0 + SMEM_STG + (chunk & 1) * STG_BYTES;
        if (et == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        epi_sync();
#pragma unroll
        for (int p16 = 0; p16 < 8; ++p16) {
          const uint32_t addr = stg + r * ROWB + ((p16 ^ (r & 7)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pk[4 * p16]),
                       "r"(pk[4 * p16 + 1]), "r"(pk[4 * p16 + 2]), "r"(pk[4 * p16 + 3])
                       : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        epi_sync();
        if (et == 0) tma_store_2d(&tmO, stg, n0 + c * 64, m0);
      }
      if (bad && __any_sync(0xffffffffu, nf && live) && lane == 0) atomicAdd(bad, 1);
    }
    if (et == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // no CTA leaves while a peer may still write into its shared memory
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

}  // namespace gl
}  // namespace sc

using namespace sc;

extern "C" int sc_gemm_residual_layernorm(const void* a, int64_t lda, const void* w, int64_t ldw, const float* bias,
                                          const void* resid, int64_t ldr, const float* gamma, const float* beta,
                                          void* out, int64_t ldo, float* out_f32, int64_t ldf,
                                          int32_t* nonfinite_count, int32_t M, int32_t N, int32_t K, void* stream) {
  using namespace gl;
  SC_CHECK_ARG(a && w && resid && gamma && beta && out && M >= 0 && K >= 1, "sc_gemm_residual_layernorm: bad arguments");
  if (M == 0) return SC_OK;
  if (N != NCL * BN || K % BK || lda < K || ldw < K || ldo < N || ldr < N || (lda * 2) % 16 || (ldw * 2) % 16 ||
      (ldo * 2) % 16 || (ldr * 2) % 16 || (out_f32 && (ldf < N || ldf % 2)) ||
      (((uintptr_t)a | (uintptr_t)w | (uintptr_t)out | (uintptr_t)resid) & 15) ||
      (((uintptr_t)gamma | (uintptr_t)beta | (uintptr_t)(bias ? bias : gamma) | (uintptr_t)(out_f32 ? out_f32 : gamma)) & 7)) {
    set_error("sc_gemm_residual_layernorm: needs N == 768, K %% 64 == 0 and 16-byte aligned rows");
    return SC_ERR_UNSUPPORTED;
  }
  CUtensorMap mA, mB, mO, mR;
  if (!make_map(&mA, a, K, M, lda, BM) || !make_map(&mB, w, K, N, ldw, BN) || !make_map(&mO, out, N, M, ldo, BM) ||
      !make_map(&mR, resid, N, M, ldr, BM)) {
    set_error("sc_gemm_residual_layernorm: cuTensorMapEncodeTiled failed");
    return SC_ERR_UNSUPPORTED;
  }
  static bool attr = false;
  const size_t smem = SMEM_TOTAL + 1024;
  if (!attr) {
    if (cudaFuncSetAttribute(gemm_res_ln_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess) {
      set_error("sc_gemm_residual_layernorm: shared memory request of %zu bytes failed", smem);
      return SC_ERR_UNSUPPORTED;
    }
    attr = true;
  }
  static int clusters = 0;
  if (!clusters) {
    // as many 3-CTA clusters as can be co-resident (1 CTA per SM)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(3 * 64);
    cfg.blockDim = dim3(NTHREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = NCL;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, gemm_res_ln_kernel, &cfg) != cudaSuccess || n <= 0) n = 148 / NCL;
    clusters = n;
  }
  const int tiles = (M + BM - 1) / BM;
  const int ncl = tiles < clusters ? tiles : clusters;
  gemm_res_ln_kernel<<<NCL * ncl, NTHREADS, smem, (cudaStream_t)stream>>>(
      mA, mB, mO, mR, bias, gamma, beta, out_f32, ldf, nonfinite_count, M, K);
  SC_CHECK_LAUNCH("gemm_res_ln_kernel");
  return SC_OK;
}
