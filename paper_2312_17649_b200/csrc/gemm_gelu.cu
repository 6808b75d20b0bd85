// Fused FFN up-projection for the bf16 encoder: out = gelu_erf(A W^T + b)
// (R/encoder.py:350-351, :258-259) in one tcgen05 GEMM whose epilogue applies
// the bias and the exact-erf GELU before the single bf16 store -- the separate
// GELU pass (read + write of the [T, 3072] activation, 14% of the encoder step
// after cuBLAS) disappears.
//
// Persistent, warp-specialised, 1 CTA per SM:
//   warp 0    TMA producer: A [128 x 64] and W [256 x 64] boxes (128B swizzle)
//             into a 4-stage mbarrier ring
//   warp 1    TMEM owner + single-thread tcgen05.mma issuer: D[128 x 256] fp32
//             in TMEM, double-buffered across tiles (2 x 256 columns)
//   warps 2-5 epilogue: tcgen05.ld of a 64-column chunk, + bias (shared-memory
//             broadcast), GELU with one MUFU op per element, bf16,
//             swizzled st.shared into a staging buffer, TMA store; the next
//             tile's mainloop runs into the other TMEM buffer meanwhile.
// A is [M, K] row-major (K-major), W is [N, K] row-major (nn.Linear layout),
// both UMMA operands K-major; requires N % 256 == 0, K % 64 == 0.
#include "gelu.cuh"
#include "gemm_common.cuh"

namespace sc {
namespace gg {
using namespace tcx;

// Shared-memory layout of one instantiation: NSV pipeline stages, then 2 staging chunks per output
// (kPre: a second output holding the pre-activation A W^T + b, for the fine-tuning backward).
template <int NSV, bool kPre>
struct Lay {
  static constexpr int NOUT = kPre ? 2 : 1;
  static constexpr int STG = NSV * STAGE;
  static constexpr int BAR = STG + 2 * NOUT * STG_BYTES;
  static constexpr int BIAS = BAR + (2 * NSV + 4) * 8 + 16;  // BN fp32 bias slice of the current tile
  static constexpr int TOTAL = BIAS + BN * 4;
};
constexpr int NS = 4;
constexpr int SMEM_STG = Lay<NS, false>::STG;
constexpr int SMEM_BAR = Lay<NS, false>::BAR;
constexpr int SMEM_BIAS = Lay<NS, false>::BIAS;
constexpr int SMEM_TOTAL = Lay<NS, false>::TOTAL;
constexpr int NS_PRE = 3;  // the dual-output variant trades a stage for the extra staging chunks


template <bool kGelu = true, bool kPre = false, int NSV = NS>
__global__ void __launch_bounds__(NTHREADS, 1) gemm_bias_gelu_kernel(
    const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
    const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmP,
    const float* __restrict__ bias, int M, int N, int K) {
  constexpr int NS = NSV;
  using L = Lay<NS, kPre>;
  constexpr int SMEM_STG = L::STG, SMEM_BAR = L::BAR, SMEM_BIAS = L::BIAS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sm0 = smem_u32(smem);
  const uint32_t bar0 = sm0 + SMEM_BAR;
  const uint32_t full_bar = bar0, empty_bar = bar0 + 8 * NS, acc_full = bar0 + 16 * NS, acc_empty = acc_full + 16;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + SMEM_BAR + (2 * NS + 4) * 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_n = N / BN, tiles = ((M + BM - 1) / BM) * tiles_n, nk = K / BK;

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
          mbar_expect_tx(full_bar + 8 * s, STAGE);
          tma_load_2d(sm0 + s * STAGE, &tmA, kb * BK, m0, full_bar + 8 * s);
          tma_load_2d(sm0 + s * STAGE + A_BYTES, &tmB, kb * BK, n0, full_bar + 8 * s);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(BM, BN, 0);
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
    const int q = warp & 3;               // TMEM lane quadrant of this warp
    const int r = q * 32 + lane;          // row within the tile
    const int et = threadIdx.x - 64;      // epilogue thread 0..127
    int i = 0, chunk = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++i) {
      const int buf = i & 1;
      const int m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
      // this tile's bias slice -> shared memory (read back as broadcasts); every
      // epilogue thread finished reading the previous tile's slice before the first
      // barrier of that tile's last chunk
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
        uint32_t pk[32], pp[kPre ? 32 : 1];
#pragma unroll
        for (int e = 0; e < 64; e += 2) {
          const float2 x = __fadd2_rn(make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])),
                                      *reinterpret_cast<const float2*>(bc + e));
          const float2 g = kGelu ? gelu2_bf16path_1mufu(x) : x;
          __nv_bfloat162 h2 = __floats2bfloat162_rn(g.x, g.y);
          pk[e / 2] = *reinterpret_cast<uint32_t*>(&h2);
          if constexpr (kPre) {
            __nv_bfloat162 x2 = __floats2bfloat162_rn(x.x, x.y);
            pp[e / 2] = *reinterpret_cast<uint32_t*>(&x2);
          }
        }
        // staging chunk(s) (chunk & 1) are free once the TMA stores issued two chunks ago have read
        // them (one store group per output per chunk)
        const uint32_t stg = sm0 + SMEM_STG + (chunk & 1) * L::NOUT * STG_BYTES;
        if (et == 0) {
          if constexpr (kPre) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
          else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
        epi_sync();
#pragma unroll
        for (int p16 = 0; p16 < 8; ++p16) {
          const uint32_t addr = stg + r * ROWB + ((p16 ^ (r & 7)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pk[4 * p16]),
                       "r"(pk[4 * p16 + 1]), "r"(pk[4 * p16 + 2]), "r"(pk[4 * p16 + 3])
                       : "memory");
          if constexpr (kPre)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr + STG_BYTES), "r"(pp[4 * p16]),
                         "r"(pp[4 * p16 + 1]), "r"(pp[4 * p16 + 2]), "r"(pp[4 * p16 + 3])
                         : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        epi_sync();
        if (et == 0) {
          tma_store_2d(&tmO, stg, n0 + c * 64, m0);
          if constexpr (kPre) tma_store_2d(&tmP, stg + STG_BYTES, n0 + c * 64, m0);
        }
      }
    }
    if (et == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}


// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs on one TPC computes a
// 256 x 256 tile with M=256 UMMAs issued by the even CTA.  Each CTA stages its
// own 128 rows of A and half (128 rows) of the W tile, so per SM a k-block moves
// 32 KB through shared memory instead of 48 KB -- the one-CTA kernel is bound
// by shared-memory bandwidth (TMA write + UMMA read of 96 KB per 512 tensor
// cycles), this one fits 6 stages.  The epilogue of each CTA drains its own
// TMEM rows; the odd CTA's epilogue signals the even CTA's TMEM-empty barrier
// remotely, the even CTA's MMA commits multicast to both CTAs.  Correct, but
// measured 10% slower than the one-CTA kernel at the encoder shape (the W1 GEMM
// is power-capped rather than shared-memory bound), so it is opt-in
// (SC_GEMM_2SM=1).
constexpr int NS2 = 6, B2_BYTES = (BN / 2) * ROWB, STAGE2 = A_BYTES + B2_BYTES;
constexpr int SMEM2_STG = NS2 * STAGE2;
constexpr int SMEM2_BAR = SMEM2_STG + 2 * STG_BYTES;
constexpr int SMEM2_BIAS = SMEM2_BAR + (2 * NS2 + 4) * 8 + 16;
constexpr int SMEM2_TOTAL = SMEM2_BIAS + BN * 4;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
// TMA load into this CTA's smem, transaction bytes counted on CTA 0's barrier.
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void mma_ss_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p; }"
      ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// Commit: arrive on the barrier at this offset in both CTAs of the pair.
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {
  asm volatile(
      "{ .reg .b16 m; mov.b16 m, 3; "
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m; }"
      ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cta0(uint32_t bar) {
  asm volatile(
      "{ .reg .b32 ra; mapa.shared::cluster.u32 ra, %0, 0; mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra]; }"
      ::"r"(bar)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1) gemm_bias_gelu_2sm_kernel(
    const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
    const __grid_constant__ CUtensorMap tmO, const float* __restrict__ bias, int M, int N, int K) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sm0 = smem_u32(smem);
  const uint32_t bar0 = sm0 + SMEM2_BAR;
  const uint32_t full_bar = bar0, empty_bar = bar0 + 8 * NS2, acc_full = bar0 + 16 * NS2, acc_empty = acc_full + 16;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + SMEM2_BAR + (2 * NS2 + 4) * 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int tiles_n = N / BN, tiles = ((M + 2 * BM - 1) / (2 * BM)) * tiles_n, nk = K / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS2; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      mbar_init(empty_bar + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full + 8 * b, 1);
      mbar_init(acc_empty + 8 * b, 8);  // 4 epilogue warps x 2 CTAs (used in CTA 0)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------------------- TMA producer (both CTAs)
    if (lane == 0) {
      prefetch_map(&tmA);
      prefetch_map(&tmB);
      int it = 0;
      for (int tile = pair; tile < tiles; tile += npairs) {
        const int m0 = (tile / tiles_n) * 2 * BM + rank * BM, n0 = (tile % tiles_n) * BN + rank * (BN / 2);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % NS2;
          if (it >= NS2) mbar_wait(empty_bar + 8 * s, ((it / NS2) & 1) ^ 1);
          if (rank == 0) mbar_expect_tx(full_bar + 8 * s, 2 * STAGE2);  // both CTAs' bytes land on CTA 0's barrier
          tma_load_2d_pair(sm0 + s * STAGE2, &tmA, kb * BK, m0, full_bar + 8 * s);
          tma_load_2d_pair(sm0 + s * STAGE2 + A_BYTES, &tmB, kb * BK, n0, full_bar + 8 * s);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer (CTA 0 only)
    if (lane == 0 && rank == 0) {
      const uint32_t idesc = idesc_bf16(2 * BM, BN, 0);
      int it = 0, i = 0;
      for (int tile = pair; tile < tiles; tile += npairs, ++i) {
        const int buf = i & 1;
        if (i >= 2) mbar_wait(acc_empty + 8 * buf, ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tD = tmem + buf * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % NS2;
          mbar_wait(full_bar + 8 * s, (it / NS2) & 1);
          tc_fence_after();
          const uint64_t ad = sw128_desc(sm0 + s * STAGE2), bd = sw128_desc(sm0 + s * STAGE2 + A_BYTES);
#pragma unroll
          for (int ks = 0; ks < BK / 16; ++ks) mma_ss_pair(tD, ad + 2 * ks, bd + 2 * ks, idesc, (kb > 0 || ks > 0));
          tc_commit_pair(empty_bar + 8 * s);
        }
        tc_commit_pair(acc_full + 8 * buf);
      }
    }
  } else {
    // ------------------------------------------------------------- epilogue (both CTAs, own rows)
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int et = threadIdx.x - 64;
    int i = 0, chunk = 0;
    for (int tile = pair; tile < tiles; tile += npairs, ++i) {
      const int buf = i & 1;
      const int m0 = (tile / tiles_n) * 2 * BM + rank * BM, n0 = (tile % tiles_n) * BN;
      float* sb = reinterpret_cast<float*>(smem + SMEM2_BIAS);
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
        if (c == BN / 64 - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (rank == 0) mbar_arrive(acc_empty + 8 * buf);
            else mbar_arrive_cta0(acc_empty + 8 * buf);
          }
        }
        const float* bc = sb + c * 64;
        uint32_t pk[32];
#pragma unroll
        for (int e = 0; e < 64; e += 2) {
          const float2 x = __fadd2_rn(make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])),
                                      *reinterpret_cast<const float2*>(bc + e));
          const float2 g = gelu2_bf16path_1mufu(x);
          __nv_bfloat162 h2 = __floats2bfloat162_rn(g.x, g.y);
          pk[e / 2] = *reinterpret_cast<uint32_t*>(&h2);
        }
        const uint32_t stg = sm0 + SMEM2_STG + (chunk & 1) * STG_BYTES;
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
    }
    if (et == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}
}  // namespace gg
}  // namespace sc

using namespace sc;

static int gemm_bias_gelu_impl(const void* a, int64_t lda, const void* w, int64_t ldw, const float* bias,
                               void* out, int64_t ldo, void* pre, int64_t ldp, int32_t M, int32_t N, int32_t K,
                               void* stream) {
  using namespace gg;
  if (pre && (ldp < N || (ldp * 2) % 16 || ((uintptr_t)pre & 15))) {
    set_error("sc_gemm_bias_gelu_pre: the pre-activation rows must be 16-byte aligned");
    return SC_ERR_UNSUPPORTED;
  }
  SC_CHECK_ARG(a && w && out && M >= 0 && N >= 1 && K >= 1, "sc_gemm_bias_gelu: bad arguments");
  if (M == 0) return SC_OK;
  if (N % BN || K % BK || lda < K || ldw < K || ldo < N || (lda * 2) % 16 || (ldw * 2) % 16 || (ldo * 2) % 16 ||
      (((uintptr_t)a | (uintptr_t)w | (uintptr_t)out) & 15) || (bias && ((uintptr_t)bias & 7))) {
    set_error("sc_gemm_bias_gelu: needs N %% 256 == 0, K %% 64 == 0 and 16-byte aligned rows");
    return SC_ERR_UNSUPPORTED;
  }
  CUtensorMap mA, mB, mO, mA2, mB2;
  if (!make_map(&mA, a, K, M, lda, BM) || !make_map(&mB, w, K, N, ldw, BN) || !make_map(&mO, out, N, M, ldo, BM) ||
      !make_map(&mA2, a, K, M, lda, BM) || !make_map(&mB2, w, K, N, ldw, BN / 2)) {
    set_error("sc_gemm_bias_gelu: cuTensorMapEncodeTiled failed");
    return SC_ERR_UNSUPPORTED;
  }
  static int pair_mode = -1;
  if (pair_mode < 0) {
    const char* e = getenv("SC_GEMM_2SM");
    pair_mode = e ? (atoi(e) != 0) : 0;  // measured: pair 1.232 ms vs one-CTA 1.118 ms (M=262k, N=3072, K=768)
  }
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (num_sms <= 0) num_sms = 148;
  }
  if (pair_mode) {
    static bool attr2 = false;
    const size_t smem2 = SMEM2_TOTAL + 1024;
    if (!attr2) {
      if (cudaFuncSetAttribute(gemm_bias_gelu_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2) !=
          cudaSuccess) {
        set_error("sc_gemm_bias_gelu: shared memory request of %zu bytes failed", smem2);
        return SC_ERR_UNSUPPORTED;
      }
      attr2 = true;
    }
    const int ptiles = ((M + 2 * BM - 1) / (2 * BM)) * (N / BN);
    const int pairs = ptiles < num_sms / 2 ? ptiles : num_sms / 2;
    gemm_bias_gelu_2sm_kernel<<<2 * pairs, NTHREADS, smem2, (cudaStream_t)stream>>>(mA2, mB2, mO, bias, M, N, K);
    SC_CHECK_LAUNCH("gemm_bias_gelu_2sm_kernel");
    return SC_OK;
  }
  static bool attr = false;
  const size_t smem = SMEM_TOTAL + 1024;
  if (!attr) {
    if (cudaFuncSetAttribute(gemm_bias_gelu_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(gemm_bias_gelu_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess) {
      set_error("sc_gemm_bias_gelu: shared memory request of %zu bytes failed", smem);
      return SC_ERR_UNSUPPORTED;
    }
    attr = true;
  }
  if (pre) {  // dual output: gelu(x) and the pre-activation x = A W^T + b
    static bool attr_pre = false;
    const size_t smem_pre = Lay<NS_PRE, true>::TOTAL + 1024;
    if (!attr_pre) {
      if (cudaFuncSetAttribute(gemm_bias_gelu_kernel<true, true, NS_PRE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem_pre) != cudaSuccess) {
        set_error("sc_gemm_bias_gelu: shared memory request of %zu bytes failed", smem_pre);
        return SC_ERR_UNSUPPORTED;
      }
      attr_pre = true;
    }
    CUtensorMap mP;
    if (!make_map(&mP, pre, N, M, ldp, BM)) {
      set_error("sc_gemm_bias_gelu: cuTensorMapEncodeTiled failed");
      return SC_ERR_UNSUPPORTED;
    }
    const int tiles_p = ((M + BM - 1) / BM) * (N / BN);
    gemm_bias_gelu_kernel<true, true, NS_PRE><<<tiles_p < num_sms ? tiles_p : num_sms, NTHREADS, smem_pre,
                                                (cudaStream_t)stream>>>(mA, mB, mO, mP, bias, M, N, K);
    SC_CHECK_LAUNCH("gemm_bias_gelu_kernel");
    return SC_OK;
  }
  const int tiles = ((M + BM - 1) / BM) * (N / BN);
  static int no_gelu = -1;  // SC_GEMM_NO_GELU=1: bias-only epilogue (measurement of the mainloop alone)
  if (no_gelu < 0) {
    const char* e = getenv("SC_GEMM_NO_GELU");
    no_gelu = e ? (atoi(e) != 0) : 0;
  }
  if (no_gelu)
    gemm_bias_gelu_kernel<false><<<tiles < num_sms ? tiles : num_sms, NTHREADS, smem, (cudaStream_t)stream>>>(
        mA, mB, mO, mO, bias, M, N, K);
  else
    gemm_bias_gelu_kernel<true><<<tiles < num_sms ? tiles : num_sms, NTHREADS, smem, (cudaStream_t)stream>>>(
        mA, mB, mO, mO, bias, M, N, K);
  SC_CHECK_LAUNCH("gemm_bias_gelu_kernel");
  return SC_OK;
}

extern "C" int sc_gemm_bias_gelu(const void* a, int64_t lda, const void* w, int64_t ldw, const float* bias,
                                 void* out, int64_t ldo, int32_t M, int32_t N, int32_t K, void* stream) {
  return gemm_bias_gelu_impl(a, lda, w, ldw, bias, out, ldo, nullptr, 0, M, N, K, stream);
}

extern "C" int sc_gemm_bias_gelu_pre(const void* a, int64_t lda, const void* w, int64_t ldw, const float* bias,
                                     void* out, int64_t ldo, void* pre, int64_t ldp, int32_t M, int32_t N, int32_t K,
                                     void* stream) {
  SC_CHECK_ARG(pre, "sc_gemm_bias_gelu_pre: null pre-activation output");
  return gemm_bias_gelu_impl(a, lda, w, ldw, bias, out, ldo, pre, ldp, M, N, K, stream);
}
