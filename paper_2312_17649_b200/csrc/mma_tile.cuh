// mma.sync tile helpers shared by the tiled attention kernels that stage
// 64-dim bf16 rows in 128B-swizzled shared memory (attn_bwd_band.cu,
// attn_qds.cu): ldmatrix / mma.sync m16n8k16 fragments, cp.async staging.
#pragma once
#include "common.cuh"

namespace sc {
namespace mmat {

constexpr int ROWB = 128;  // bytes per 64-dim bf16 row

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t swz(uint32_t base, int row, int chunk) {
  return base + row * ROWB + ((chunk ^ (row & 7)) << 4);
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// 8x8 b16 transpose across the warp (movmatrix): a C-fragment row pair -> a B-fragment column pair.
__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t r;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}
// 16-byte async copy; src_bytes = 0 zero-fills the destination.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// A fragments (16 rows x 64 dims) of the block starting at smem row `row0`.
__device__ __forceinline__ void load_a(uint32_t buf, int row0, int lane, uint32_t (&a)[4][4]) {
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) ldsm_x4(swz(buf, row0 + (lane & 15), ks * 2 + (lane >> 4)), a[ks]);
}
// C[2 n8 tiles] += A(16x64) . B[row0 .. row0+15]^T  (B rows = the n index, 64 dims = k)
__device__ __forceinline__ void mm_nt16(uint32_t bbuf, int row0, int lane, const uint32_t (&a)[4][4],
                                        float (&c0)[4], float (&c1)[4]) {
  const int brow = row0 + (lane & 7) + ((lane >> 4) << 3);
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    uint32_t b[4];
    ldsm_x4(swz(bbuf, brow, ks * 2 + ((lane >> 3) & 1)), b);
    mma16816(c0, a[ks], b[0], b[1]);
    mma16816(c1, a[ks], b[2], b[3]);
  }
}
// O(16x64) += P(16 x 16, as two C-layout n8 tiles) . B[row0 .. row0+15]  (B rows = the k index)
__device__ __forceinline__ void mm_nn16(uint32_t bbuf, int row0, int lane, const float (&p0)[4],
                                        const float (&p1)[4], float (&o)[8][4]) {
  uint32_t a[4] = {pack_bf16(p0[0], p0[1]), pack_bf16(p0[2], p0[3]), pack_bf16(p1[0], p1[1]),
                   pack_bf16(p1[2], p1[3])};
  const int brow = row0 + (lane & 7) + (((lane >> 3) & 1) << 3);
#pragma unroll
  for (int np = 0; np < 4; ++np) {
    uint32_t b[4];
    ldsm_x4_t(swz(bbuf, brow, np * 2 + (lane >> 4)), b);
    mma16816(o[2 * np], a, b[0], b[1]);
    mma16816(o[2 * np + 1], a, b[2], b[3]);
  }
}

// Online-softmax update over NB n8 blocks of RAW logits (masked to -inf) for the two rows (g, g+8)
// of an m16n8 C fragment; m in raw-logit units, c2 = log2(e)/scale.  Overwrites s with P.
// kFresh: o is still zero (first update of a row block) -> no O rescale.
template <int NB, bool kFresh = false>
__device__ __forceinline__ void softmax_update(float (&s)[NB][4], float c2, float& m0, float& m1, float& l0,
                                               float& l1, float (&o)[8][4]) {
  float x0 = -INFINITY, x1 = -INFINITY;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    x0 = fmaxf(x0, fmaxf(s[b][0], s[b][1]));
    x1 = fmaxf(x1, fmaxf(s[b][2], s[b][3]));
  }
  x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, 1));
  x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, 2));
  x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, 1));
  x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, 2));
  const float n0 = fmaxf(m0, x0), n1 = fmaxf(m1, x1);
  const float b0 = n0 == -INFINITY ? 0.f : n0 * c2, b1 = n1 == -INFINITY ? 0.f : n1 * c2;
  const float a0 = ex2(fmaf(m0, c2, -b0)), a1 = ex2(fmaf(m1, c2, -b1));
  float r0 = 0.f, r1 = 0.f;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    s[b][0] = ex2(fmaf(s[b][0], c2, -b0));
    s[b][1] = ex2(fmaf(s[b][1], c2, -b0));
    s[b][2] = ex2(fmaf(s[b][2], c2, -b1));
    s[b][3] = ex2(fmaf(s[b][3], c2, -b1));
    r0 += s[b][0] + s[b][1];
    r1 += s[b][2] + s[b][3];
  }
  l0 = fmaf(l0, a0, r0);
  l1 = fmaf(l1, a1, r1);
  if constexpr (!kFresh) {
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
      o[nb][0] *= a0;
      o[nb][1] *= a0;
      o[nb][2] *= a1;
      o[nb][3] *= a1;
    }
  }
  m0 = n0;
  m1 = n1;
}

// Stage `nrows` rows (64 bf16 each) into a swizzled smem buffer; rowptr(i) == nullptr zero-fills.
template <typename F>
__device__ __forceinline__ void stage_rows(uint32_t buf, int nrows, const __nv_bfloat16* any, F&& rowptr) {
  for (int idx = threadIdx.x; idx < nrows * 8; idx += blockDim.x) {
    const int r = idx >> 3, c = idx & 7;
    const __nv_bfloat16* p = rowptr(r);
    cp_async16(swz(buf, r, c), p ? p + c * 8 : any, p ? 16 : 0);
  }
}

}  // namespace mmat
}  // namespace sc
