// Shared pieces of the warp-specialised tcgen05 GEMMs with fused epilogues
// (gemm_gelu.cu: W1 + bias + GELU; gemm_ln.cu: Wo / W2 + bias + residual + LayerNorm).
#pragma once
#include "tc_common.cuh"

namespace sc {
namespace gg {

// 128 x 256 output tile per CTA, 64-deep k-blocks (one 128B swizzle atom per row).
constexpr int BM = 128, BN = 256, BK = 64, ROWB = 128;
// warp 0: TMA producer, warp 1: TMEM owner + MMA issuer, warps 2-5: epilogue.
constexpr int NTHREADS = 192;
constexpr int A_BYTES = BM * ROWB, B_BYTES = BN * ROWB, STAGE = A_BYTES + B_BYTES;
constexpr int STG_BYTES = BM * ROWB;  // one 128-row x 64-column bf16 staging chunk

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(src)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// Named barrier of the 128 epilogue threads.
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

}  // namespace gg
}  // namespace sc
