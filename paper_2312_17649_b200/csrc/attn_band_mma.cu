// Tiled band attention for doc rows (the HBM-bound hot path of the sparse
// cross-encoder, arXiv 2312.17649 Eqs. 1-3), bf16 I/O, fp32 softmax/accum.
//
// One CTA = one tile of BM=64 doc rows of one sequence, looping over heads.
// Per head a 2-3 stage TMA pipeline (128B-swizzled boxes, mbarrier complete_tx)
// stages in shared memory:
//   Q   [64 x 64]        doc rows r0..r0+63
//   Kb/Vb [64+2w x 64]   doc rows r0-w .. r0+63+w  (the band halo)
//   Kg/Vg [GR x 64]      the sequence's cls + query-group rows (global keys)
//   Qf  [GR x 64]        the same rows as queries ("full rows": CLS, and query
//                        rows under longformer/full, that attend the whole doc)
// Warps 0-3 each own 16 doc rows: S = Q K^T over {global keys} U {band keys}
// with mma.sync m16n8k16 (bf16 -> fp32), static band mask, online softmax in
// the exp2 domain, O += P V, bf16 stores.  The producer warp, one item behind
// its loads, emits the split-softmax records (m, l, acc) of the "full rows"
// over the tile's 64 doc keys (keys as the MMA's M dimension: 8 full rows per
// n8 column block), so the CLS row never re-reads K/V from HBM.  The first
// tile of a sequence also computes the head rows (cls, query group) over the
// global keys -- final for rows without a doc link (sparse query rows), a
// record for the others -- and merge_full_rows_kernel (one warp per sequence,
// head and row) folds the records into the CLS (and longformer query) rows.
// Warp 4 is the TMA producer (and the full-row records).
//
// Semantics: doc row r attends cls (if linked), query group (if linked) and
// doc keys t with |t - r| <= w, 0 <= t < n_doc (R/band.py:48-52,
// R/attention.py:125-139); zero-logit padding adds (2w+1 - #in-range) logit-0
// slots (R/attention.py:244-247).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "attn.cuh"

namespace sc {
namespace bandk {

constexpr int BM = 64;
constexpr int D = 64;
constexpr int ROWB = 128;  // bytes per smem row
constexpr int NDOCW = 4;
constexpr int PRODW = 4;
constexpr int NTHREADS = 160;
constexpr int MAX_W = 96;  // Kb box rows 64 + 2w <= 256 (TMA box limit)
constexpr int REC = D + 4; // split-softmax record: m, l, pad, pad, acc[D] (16B-aligned acc)
// Resident CTAs per SM the register/smem budget targets (measured on B200,
// s=4099 H=12: 3 CTAs / 2 stages is best for w <= 8, 2 CTAs / 3 stages above).
#ifndef SC_BAND_L2PROMO
#define SC_BAND_L2PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
#ifndef SC_BAND_CTAS1
#define SC_BAND_CTAS1 3  // resident CTAs per SM of the single-chunk (w <= 8) variant
#endif
#ifndef SC_BAND_PF
// L2 prefetch (cp.async.bulk.prefetch.tensor) of the boxes SC_BAND_PF x NS items ahead; 0 = none.
// Measured on B200: off 4.35 us vs on 4.83 us per sequence-layer at w=4 (88% vs 79% of HBM): the
// stage loads are already in flight NS items ahead and the extra L2 fills only compete with them.
#define SC_BAND_PF 0
#endif
__host__ __device__ constexpr int min_ctas(int nbc, int qfg = 0) { return nbc == 1 || qfg ? SC_BAND_CTAS1 : 2; }

struct Params {
  int nseq, H, w, kb_rows, fneed, fmax, padding;
  int reverse;  // visit tiles last-to-first: the producing GEMM's most recent output rows are still in L2
  int link_cls, link_query;
  int doc_rows;  // 0: head rows only (doc rows computed by the tcgen05 kernel)
  int dout;      // head_dim (32 or 64; smem rows are always 64 dims, zero-padded)
  int Ht;        // heads of the layout (records / outputs); H counts items per tile (H / 2 in pair mode)
  // head rows (cls = group 0, query = group 1): links to cls / query keys, doc FULL
  int hl[2][2], hdoc[2];
  int ntiles_max;      // record index of sequence j's global-key record = ntiles_max + j
  int cls_skip;        // measurement only (SC_BAND_CLS_SKIP=1): no full-row records (wrong CLS rows)
  float c2;  // log2(e) / scale: raw logit -> exp2 domain
  const int32_t* cu;
  const int32_t* qlen;
  const int32_t* tile_base;
  const __nv_bfloat16* q;  // QFG variants: the cls + query rows' q read from global memory
  int64_t ld_q;
  int T;
  __nv_bfloat16* out;
  int64_t ld_out;
  float* partials;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// One lane of a converged warp (elect.sync; the lowest active lane): TMA issue / bulk-store waits
// under it keep their operands warp-uniform.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0, 1, 0, P; }" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}
// Tensor maps are 3-D [rows][heads][head_dim] with 64-element boxes along head_dim: a
// 32-dim head lands zero-padded in a 64-dim (128 B) smem row (the out-of-bounds half of the
// box is zero-filled; no extra HBM bytes), so one kernel serves head_dim 32 and 64.
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int head, int row, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(head), "r"(row), "r"(bar)
      : "memory");
}
// Pull a box into L2 only (no smem, no barrier): the producer runs one
// pipeline round ahead so the next round's TMA loads are served from L2.
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int head, int row) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(head), "r"(row)
               : "memory");
}
// Shared -> global TMA store of a box (bulk-group completion); the padded half of a
// 32-dim head is clipped.
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int head, int row) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(head), "r"(row), "r"(src)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// Wait until every committed bulk store has finished READING shared memory.
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void stsm_x4(uint32_t addr, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
  asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1,%2,%3,%4};"
               ::"r"(addr), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
               : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// 128B-swizzled address of (row, 16-byte chunk) in a 1024B-aligned buffer.
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

// A fragments of a 16-row x 64-dim Q block starting at smem row `row0`.
__device__ __forceinline__ void load_q(uint32_t buf, int row0, int lane, uint32_t (&qa)[4][4]) {
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) ldsm_x4(swz(buf, row0 + (lane & 15), ks * 2 + (lane >> 4)), qa[ks]);
}

// S[2 n8 blocks] = Q(16x64) . K[key0 .. key0+15]^T
__device__ __forceinline__ void qk16(uint32_t kbuf, int key0, int lane, const uint32_t (&qa)[4][4],
                                     float (&s0)[4], float (&s1)[4]) {
  const int krow = key0 + (lane & 7) + ((lane >> 4) << 3);
#pragma unroll
  for (int e = 0; e < 4; ++e) s0[e] = s1[e] = 0.f;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    uint32_t b[4];
    ldsm_x4(swz(kbuf, krow, ks * 2 + ((lane >> 3) & 1)), b);
    mma16816(s0, qa[ks], b[0], b[1]);
    mma16816(s1, qa[ks], b[2], b[3]);
  }
}

// O(16x64) += P(16 x 16 keys) . V[key0 .. key0+15]
__device__ __forceinline__ void pv16(uint32_t vbuf, int key0, int lane, const float (&p0)[4],
                                     const float (&p1)[4], float (&o)[8][4]) {
  uint32_t a[4] = {pack_bf16(p0[0], p0[1]), pack_bf16(p0[2], p0[3]), pack_bf16(p1[0], p1[1]),
                   pack_bf16(p1[2], p1[3])};
  const int vrow = key0 + (lane & 7) + (((lane >> 3) & 1) << 3);
#pragma unroll
  for (int np = 0; np < 4; ++np) {
    uint32_t b[4];
    ldsm_x4_t(swz(vbuf, vrow, np * 2 + (lane >> 4)), b);
    mma16816(o[2 * np], a, b[0], b[1]);
    mma16816(o[2 * np + 1], a, b[2], b[3]);
  }
}

// Per-lane byte offsets of the ldmatrix / stmatrix row addresses inside a
// 16-row block whose first row is a multiple of 8 (then the 128B swizzle term
// depends on the lane only): q = A fragments of Q, k = B fragments of K
// (non-transposed), v = B fragments of V (transposed) and the stmatrix layout.
struct LaneOff {
  uint32_t q[4], k[4], v[4];
};
__device__ __forceinline__ LaneOff lane_offsets(int lane) {
  LaneOff o;
  const int l7 = lane & 7;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o.q[i] = (lane & 15) * ROWB + (((2 * i + (lane >> 4)) ^ l7) << 4);
    o.k[i] = (l7 + ((lane >> 4) << 3)) * ROWB + (((2 * i + ((lane >> 3) & 1)) ^ l7) << 4);
    o.v[i] = (l7 + (((lane >> 3) & 1) << 3)) * ROWB + (((2 * i + (lane >> 4)) ^ l7) << 4);
  }
  return o;
}
// Aligned variants (row0 / key0 multiples of 8): one add per ldmatrix.
__device__ __forceinline__ void load_q(uint32_t buf, int row0, const LaneOff& lo, uint32_t (&qa)[4][4]) {
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) ldsm_x4(buf + row0 * ROWB + lo.q[ks], qa[ks]);
}
__device__ __forceinline__ void qk16(uint32_t kbuf, int key0, const LaneOff& lo, const uint32_t (&qa)[4][4],
                                     float (&s0)[4], float (&s1)[4]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) s0[e] = s1[e] = 0.f;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    uint32_t b[4];
    ldsm_x4(kbuf + key0 * ROWB + lo.k[ks], b);
    mma16816(s0, qa[ks], b[0], b[1]);
    mma16816(s1, qa[ks], b[2], b[3]);
  }
}
__device__ __forceinline__ void pv16(uint32_t vbuf, int key0, const LaneOff& lo, const float (&p0)[4],
                                     const float (&p1)[4], float (&o)[8][4]) {
  uint32_t a[4] = {pack_bf16(p0[0], p0[1]), pack_bf16(p0[2], p0[3]), pack_bf16(p1[0], p1[1]),
                   pack_bf16(p1[2], p1[3])};
#pragma unroll
  for (int np = 0; np < 4; ++np) {
    uint32_t b[4];
    ldsm_x4_t(vbuf + key0 * ROWB + lo.v[np], b);
    mma16816(o[2 * np], a, b[0], b[1]);
    mma16816(o[2 * np + 1], a, b[2], b[3]);
  }
}

// Single n8 block variants for the last 8 band keys of a row block (w <= 4:
// 16 rows + 2w keys fit 24 columns): S = Q . K[key0 .. key0+7]^T, and
// O += P . V[key0 .. key0+7] with m16n8k8 (key0 a multiple of 8).
__device__ __forceinline__ void mma1688(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(b0));
}
__device__ __forceinline__ void qk8(uint32_t kbuf, int key0, int lane, const uint32_t (&qa)[4][4], float (&s0)[4]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) s0[e] = 0.f;
#pragma unroll
  for (int k2 = 0; k2 < 2; ++k2) {
    uint32_t b[4];
    ldsm_x4(swz(kbuf, key0 + (lane & 7), 4 * k2 + (lane >> 3)), b);
    mma16816(s0, qa[2 * k2], b[0], b[1]);
    mma16816(s0, qa[2 * k2 + 1], b[2], b[3]);
  }
}
__device__ __forceinline__ void pv8(uint32_t vbuf, int key0, int lane, const float (&p0)[4], float (&o)[8][4]) {
  const uint32_t a0 = pack_bf16(p0[0], p0[1]), a1 = pack_bf16(p0[2], p0[3]);
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    uint32_t b[4];
    ldsm_x4_t(swz(vbuf, key0 + (lane & 7), 4 * half + (lane >> 3)), b);
#pragma unroll
    for (int i = 0; i < 4; ++i) mma1688(o[4 * half + i], a0, a1, b[i]);
  }
}

// Head-pair mode (head_dim 32, two heads per 64-dim smem row): the same contractions restricted
// to one head's 32 dims, hh = 0 (dims 0-31: k-steps / n-tiles of the first head) or 1.
__device__ __forceinline__ void qk16_hh(uint32_t kbuf, int key0, const LaneOff& lo, const uint32_t (&qa)[4][4],
                                        float (&s0)[4], float (&s1)[4], int hh) {
#pragma unroll
  for (int e = 0; e < 4; ++e) s0[e] = s1[e] = 0.f;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int ks = 2 * hh + k;
    uint32_t b[4];
    ldsm_x4(kbuf + key0 * ROWB + lo.k[ks], b);
    mma16816(s0, qa[ks], b[0], b[1]);
    mma16816(s1, qa[ks], b[2], b[3]);
  }
}
__device__ __forceinline__ void pv16_hh(uint32_t vbuf, int key0, const LaneOff& lo, const float (&p0)[4],
                                        const float (&p1)[4], float (&o)[8][4], int hh) {
  uint32_t a[4] = {pack_bf16(p0[0], p0[1]), pack_bf16(p0[2], p0[3]), pack_bf16(p1[0], p1[1]),
                   pack_bf16(p1[2], p1[3])};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int np = 2 * hh + k;
    uint32_t b[4];
    ldsm_x4_t(vbuf + key0 * ROWB + lo.v[np], b);
    mma16816(o[2 * np], a, b[0], b[1]);
    mma16816(o[2 * np + 1], a, b[2], b[3]);
  }
}
__device__ __forceinline__ void qk8_hh(uint32_t kbuf, int key0, int lane, const uint32_t (&qa)[4][4], float (&s0)[4],
                                       int hh) {
#pragma unroll
  for (int e = 0; e < 4; ++e) s0[e] = 0.f;
  uint32_t b[4];
  ldsm_x4(swz(kbuf, key0 + (lane & 7), 4 * hh + (lane >> 3)), b);
  mma16816(s0, qa[2 * hh], b[0], b[1]);
  mma16816(s0, qa[2 * hh + 1], b[2], b[3]);
}
__device__ __forceinline__ void pv8_hh(uint32_t vbuf, int key0, int lane, const float (&p0)[4], float (&o)[8][4],
                                       int hh) {
  const uint32_t a0 = pack_bf16(p0[0], p0[1]), a1 = pack_bf16(p0[2], p0[3]);
  uint32_t b[4];
  ldsm_x4_t(swz(vbuf, key0 + (lane & 7), 4 * hh + (lane >> 3)), b);
#pragma unroll
  for (int i = 0; i < 4; ++i) mma1688(o[4 * hh + i], a0, a1, b[i]);
}
// unaligned-key (lane-addressed) variants for the full-row records (key0 = w + 16 np)
__device__ __forceinline__ void qk16l_hh(uint32_t kbuf, int key0, int lane, const uint32_t (&qa)[4][4],
                                         float (&s0)[4], float (&s1)[4], int hh) {
  const int krow = key0 + (lane & 7) + ((lane >> 4) << 3);
#pragma unroll
  for (int e = 0; e < 4; ++e) s0[e] = s1[e] = 0.f;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int ks = 2 * hh + k;
    uint32_t b[4];
    ldsm_x4(swz(kbuf, krow, ks * 2 + ((lane >> 3) & 1)), b);
    mma16816(s0, qa[ks], b[0], b[1]);
    mma16816(s1, qa[ks], b[2], b[3]);
  }
}
__device__ __forceinline__ void pv16l_hh(uint32_t vbuf, int key0, int lane, const float (&p0)[4],
                                         const float (&p1)[4], float (&o)[8][4], int hh) {
  uint32_t a[4] = {pack_bf16(p0[0], p0[1]), pack_bf16(p0[2], p0[3]), pack_bf16(p1[0], p1[1]),
                   pack_bf16(p1[2], p1[3])};
  const int vrow = key0 + (lane & 7) + (((lane >> 3) & 1) << 3);
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int np = 2 * hh + k;
    uint32_t b[4];
    ldsm_x4_t(swz(vbuf, vrow, np * 2 + (lane >> 4)), b);
    mma16816(o[2 * np], a, b[0], b[1]);
    mma16816(o[2 * np + 1], a, b[2], b[3]);
  }
}

// Online-softmax update over NB n8 blocks of RAW logits (masked to -inf) for
// rows (g, g+8).  m is kept in raw-logit units; c2 = log2(e)/scale.  Overwrites s with P.
// kFresh: o is still zero (first update of a row block) -> skip the O rescale.
template <int NB, bool kFresh = false>
__device__ __forceinline__ void softmax_update(float (&s)[NB][4], float c2, float& m0, float& m1,
                                               float& l0, float& l1, float (&o)[8][4]) {
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

__device__ __forceinline__ void zero_o(float (&o)[8][4]) {
#pragma unroll
  for (int nb = 0; nb < 8; ++nb) o[nb][0] = o[nb][1] = o[nb][2] = o[nb][3] = 0.f;
}
// movmatrix: 8x8 b16 transpose across the warp (C-fragment rows <-> B-fragment columns)
__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t r;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}

// Full-row split-softmax records of one item (the producer warp, all 32 lanes): the "full rows"
// (CLS; query rows under longformer) against the tile's own 64 doc keys, Kb/Vb rows w .. w + 63.
// Keys are the M dimension (S^T = K Qf^T, O^T = V^T P^T), so 8 full rows cost one n8 column
// block: 16 + 16 mma.sync for a tile instead of 64 with the rows as a 16-row M fragment of which
// the sparse pattern uses one.  P^T moves from the C layout of S^T to the B layout of the PV
// product by movmatrix.  Record f: (m, l, -, -, acc[64]) -- m in natural logit units, l the sum of
// exp(s - m) over the tile's keys, acc = sum exp(s - m) v (R/attention.py:416-473 split form).
// A bf16 pair (row, col..col+1) of one head's q for the QFG variants: zero past the token range and
// past head_dim (32-dim heads ride in the zero-padded 64-dim layout of the staged rows).
__device__ __forceinline__ uint32_t ldg_pair(const Params& p, int h, int64_t row, int col) {
  return (row < p.T && col < p.dout)
             ? __ldg(reinterpret_cast<const uint32_t*>(p.q + row * p.ld_q + (int64_t)h * p.dout + col))
             : 0u;
}

template <int PAIR, int QFG = 0>
__device__ __forceinline__ void full_row_records(const Params& p, uint32_t qf, uint32_t kb, uint32_t vb, int lane,
                                                 int tile, int h, int rows_here, int qrow0) {
  const int g8 = lane >> 2, t = lane & 3;
  const float c2 = p.c2;
  const float to_nat = c2 * 0.69314718055994530942f;  // raw logit -> natural units (1/scale)
  const int w = p.w;
#pragma unroll 1
  for (int hh = 0; hh < (PAIR ? 2 : 1); ++hh) {
    const int ks0 = PAIR ? 2 * hh : 0, nks = PAIR ? 2 : 4;  // this head's k-steps (dims) / m-tiles
    const int ht = PAIR ? 2 * h + hh : h;
#pragma unroll 1
    for (int fb = 0; fb * 8 < p.fneed; ++fb) {
      // B fragments of full rows fb*8 .. fb*8+7 (Qf rows = B columns): k-steps 2i, 2i+1 per x4
      uint32_t qb[4][2];
      if constexpr (QFG) {  // B fragments straight from the rows' q (L2): rows qrow0 + fb*8 + g8
        const int64_t row = qrow0 + fb * 8 + g8;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          qb[ks][0] = ldg_pair(p, h, row, ks * 16 + 2 * t);
          qb[ks][1] = ldg_pair(p, h, row, ks * 16 + 8 + 2 * t);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          uint32_t r[4];
          ldsm_x4(swz(qf, fb * 8 + (lane & 7), 4 * i + (lane >> 3)), r);
          qb[2 * i][0] = r[0]; qb[2 * i][1] = r[1]; qb[2 * i + 1][0] = r[2]; qb[2 * i + 1][1] = r[3];
        }
      }
      float s[4][4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        s[mt][0] = s[mt][1] = s[mt][2] = s[mt][3] = 0.f;
#pragma unroll
        for (int k = 0; k < nks; ++k) {
          const int ks = ks0 + k;
          uint32_t a[4];
          ldsm_x4(swz(kb, w + mt * 16 + (lane & 15), ks * 2 + (lane >> 4)), a);
          mma16816(s[mt], a, qb[ks][0], qb[ks][1]);
        }
      }
      // keys past the document end: -inf; column (full row) max over the 64 keys
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (mt * 16 + g8 + ((e >> 1) << 3) >= rows_here) s[mt][e] = -INFINITY;
          if (e & 1) mx1 = fmaxf(mx1, s[mt][e]);
          else mx0 = fmaxf(mx0, s[mt][e]);
        }
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
      }
      const float b0 = mx0 == -INFINITY ? 0.f : mx0 * c2, b1 = mx1 == -INFINITY ? 0.f : mx1 * c2;
      float l0 = 0.f, l1 = 0.f;
      uint32_t pb[4][2];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        s[mt][0] = ex2(fmaf(s[mt][0], c2, -b0));
        s[mt][1] = ex2(fmaf(s[mt][1], c2, -b1));
        s[mt][2] = ex2(fmaf(s[mt][2], c2, -b0));
        s[mt][3] = ex2(fmaf(s[mt][3], c2, -b1));
        l0 += s[mt][0] + s[mt][2];
        l1 += s[mt][1] + s[mt][3];
        pb[mt][0] = movm_t(pack_bf16(s[mt][0], s[mt][1]));  // keys 2t, 2t+1 of column g8
        pb[mt][1] = movm_t(pack_bf16(s[mt][2], s[mt][3]));  // keys 2t+8, 2t+9
      }
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
      }
      // O^T (dims x full rows) = V^T P^T: A = V^T through ldmatrix.trans of the key-major V rows
      float ot[4][4];
#pragma unroll
      for (int k = 0; k < nks; ++k) {
        const int dm = ks0 + k;
        ot[k][0] = ot[k][1] = ot[k][2] = ot[k][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          uint32_t a[4];
          ldsm_x4_t(swz(vb, w + kk * 16 + (lane & 7) + ((lane >> 4) << 3), dm * 2 + ((lane >> 3) & 1)), a);
          mma16816(ot[k], a, pb[kk][0], pb[kk][1]);
        }
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int f = fb * 8 + 2 * t + c;
        if (f >= p.fneed) continue;
        float* rec = p.partials + (((int64_t)tile * p.Ht + ht) * p.fmax + f) * REC;
        if (g8 == 0) {
          rec[0] = (c ? mx1 : mx0) * to_nat;
          rec[1] = c ? l1 : l0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const bool live = k < nks;  // PAIR: the head's 32 dims, then zeros
          rec[4 + k * 16 + g8] = live ? ot[k][c] : 0.f;
          rec[4 + k * 16 + g8 + 8] = live ? ot[k][2 + c] : 0.f;
        }
      }
    }
  }
}

// NBC: band chunks of 32 keys per 16-row warp block (ceil((16+2w)/32)).
// GR: global rows staged per head (16 or 32).  NS: pipeline stages.
// NBB: band n8 blocks of the single-shot path (NBC = 1): 3 when 16 + 2w <= 24.
// PAIR (head_dim 32, NBC = 1): items are head pairs (2h, 2h + 1) sharing the 64-dim smem rows.
// QFG (NBC = 2, 8 < w <= 16): no Qf box in the stage (the producer's records and the first tile's head
// rows read those q rows from L2), the band's second chunk is 16 keys (16 + 2w <= 48), Kb/Vb rows = the
// 96-row box: a 36 KB stage, so three CTAs per SM fit two stages each.
template <int NBC, int GR, int NS, int NBB = 4, int PAIR = 0, int QFG = 0>
__global__ void __launch_bounds__(NTHREADS, min_ctas(NBC, QFG)) band_attn_kernel(
    const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmQf,
    const __grid_constant__ CUtensorMap tmKg, const __grid_constant__ CUtensorMap tmVg,
    const __grid_constant__ CUtensorMap tmKb, const __grid_constant__ CUtensorMap tmVb,
    const __grid_constant__ CUtensorMap tmO, Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  // Persistent: CTA b processes tiles b, b + gridDim.x, ...; the TMA ring runs
  // continuously across tile boundaries (global head iteration counter `it`).
  // the record merge (a programmatic dependent) may be scheduled now; it waits for this grid
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int ntiles = __ldg(p.tile_base + p.nseq);
  if ((int)blockIdx.x >= ntiles) return;
  const int w = p.w;
  constexpr int kb_rows = QFG ? 96 : 48 + 32 * NBC;
  constexpr int NF = QFG ? 2 : 3;  // cls + query row boxes per stage: K, V (, Q)
  constexpr int q_bytes = BM * ROWB, f_bytes = GR * ROWB, kb_bytes = kb_rows * ROWB;
  constexpr int stage_bytes = q_bytes + NF * f_bytes + 2 * kb_bytes;
  constexpr int g_off = q_bytes + (QFG ? 0 : f_bytes);  // Kg, then Vg
  const int kb_box = BM + 2 * w;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * stage_bytes);
  const uint32_t sm0 = smem_u32(smem);
  auto q_buf = [&](int s) { return sm0 + s * stage_bytes; };
  auto qf_buf = [&](int s) { return sm0 + s * stage_bytes + q_bytes; };
  auto kg_buf = [&](int s) { return sm0 + s * stage_bytes + g_off; };
  auto vg_buf = [&](int s) { return sm0 + s * stage_bytes + g_off + f_bytes; };
  auto kb_buf = [&](int s) { return sm0 + s * stage_bytes + q_bytes + NF * f_bytes; };
  auto vb_buf = [&](int s) { return sm0 + s * stage_bytes + q_bytes + NF * f_bytes + kb_bytes; };
  const uint32_t full_bar = smem_u32(bars), empty_bar = smem_u32(bars + NS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // Zero the Kb/Vb rows the TMA box never writes (band chunks read up to kb_rows).
  for (int s = 0; s < NS; ++s) {
    uint8_t* kb = smem + s * stage_bytes + q_bytes + NF * f_bytes;
    for (int o = kb_box * ROWB + threadIdx.x * 16; o < kb_bytes; o += NTHREADS * 16) {
      *reinterpret_cast<uint4*>(kb + o) = make_uint4(0, 0, 0, 0);
      *reinterpret_cast<uint4*>(kb + kb_bytes + o) = make_uint4(0, 0, 0, 0);
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      mbar_init(empty_bar + 8 * s, NDOCW + 1);  // doc warps + the producer's records
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  if (warp == PRODW) {
    // The whole warp walks the items (converged); one elect.sync lane issues each item's loads, so
    // the TMA operands stay warp-uniform (no per-lane waterfall loop around UTMALDG).  One item
    // behind the loads, the warp computes the item's full-row records (full_row_records) and
    // releases the stage with the doc warps (empty barrier: NDOCW + 1 arrivals).
    {
      if (elect_one()) {
        prefetch_map(&tmQ); prefetch_map(&tmKb); prefetch_map(&tmVb);
        prefetch_map(&tmKg); prefetch_map(&tmVg); prefetch_map(&tmQf);
      }
      __syncwarp();
      const uint32_t bytes = (uint32_t)((p.doc_rows ? q_bytes : 0) + NF * f_bytes + 2 * kb_box * ROWB);
      const bool recs = p.fneed > 0 && !p.cls_skip;
      int it = 0, prev_tile = -1, prev_h = 0, prev_rows = 0, prev_start = 0;
      auto records = [&](int pit) {  // full-row records of item pit, then release its stage
        const int sp = pit % NS;
        mbar_wait(full_bar + 8 * sp, (pit / NS) & 1);
        if (recs)
          full_row_records<PAIR, QFG>(p, qf_buf(sp), kb_buf(sp), vb_buf(sp), lane, prev_tile, prev_h, prev_rows,
                                      prev_start);
        __syncwarp();
        if (elect_one()) mbar_arrive(empty_bar + 8 * sp);
        __syncwarp();
      };
      for (int tix = blockIdx.x; tix < ntiles; tix += gridDim.x) {
        const int tile = p.reverse ? ntiles - 1 - tix : tix;
        const int j = find_seq(p.tile_base, p.nseq, tile);
        const SeqGroups g = seq_groups(p.cu, p.qlen, j);
        const int r0 = (tile - __ldg(p.tile_base + j)) * BM;
        const int doc_row0 = g.start + g.off[2] + r0;
        const int rows_here = min(BM, g.len[2] - r0);
        for (int h = 0; h < p.H; ++h, ++it) {
          const int s = it % NS;
          if (it >= NS) mbar_wait(empty_bar + 8 * s, ((it / NS) & 1) ^ 1);
          const uint32_t fb = full_bar + 8 * s;
          if (elect_one()) {
            if (SC_BAND_PF > 0 && h + SC_BAND_PF * NS < p.H) {  // L2 prefetch of the boxes of a later item of this tile
              if (p.doc_rows) tma_prefetch_3d(&tmQ, h + SC_BAND_PF * NS, doc_row0);
              tma_prefetch_3d(&tmKb, h + SC_BAND_PF * NS, doc_row0 - w);
              tma_prefetch_3d(&tmVb, h + SC_BAND_PF * NS, doc_row0 - w);
            }
            mbar_expect_tx(fb, bytes);
            if (p.doc_rows) tma_load_3d(q_buf(s), &tmQ, h, doc_row0, fb);
            tma_load_3d(kb_buf(s), &tmKb, h, doc_row0 - w, fb);
            tma_load_3d(vb_buf(s), &tmVb, h, doc_row0 - w, fb);
            tma_load_3d(kg_buf(s), &tmKg, h, g.start, fb);
            tma_load_3d(vg_buf(s), &tmVg, h, g.start, fb);
            if (!QFG) tma_load_3d(qf_buf(s), &tmQf, h, g.start, fb);
          }
          __syncwarp();
          if (it > 0) records(it - 1);
          prev_tile = tile; prev_h = h; prev_rows = rows_here; prev_start = g.start;
        }
      }
      if (it > 0) records(it - 1);
    }
    return;
  }

  // ------------------------------------------------------------ doc warps
  const int gq = lane >> 2, tq = lane & 3;
  const int wr0 = warp * 16;
  const LaneOff LO = lane_offsets(lane);
  const float c2 = p.c2;
  const int hl_bits = p.hl[0][0] | (p.hl[0][1] << 1) | (p.hl[1][0] << 2) | (p.hl[1][1] << 3);
  const int hdoc_bits = p.hdoc[0] | (p.hdoc[1] << 1);
  // Band mask of an interior tile (no sequence edge in reach): bit (nb*4 + e) of
  // chunk bc set when that score element is inside the +-w band.  Tile-independent.
  uint32_t bmask_int[NBC];
#pragma unroll
  for (int bc = 0; bc < NBC; ++bc) {
    uint32_t m = 0;
#pragma unroll
    for (int nb = 0; nb < 4; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int diff = 32 * bc + nb * 8 + 2 * tq + (e & 1) - (gq + ((e >> 1) << 3));  // t - r + w
        m |= (diff >= 0 && diff <= 2 * w ? 1u : 0u) << (nb * 4 + e);
      }
    bmask_int[bc] = m;
  }
  int it = 0, last_j = -1;
  uint32_t gmask[GR / 16];
  for (int tix = blockIdx.x; tix < ntiles; tix += gridDim.x) {
    const int tile = p.reverse ? ntiles - 1 - tix : tix;
    const int j = find_seq(p.tile_base, p.nseq, tile);
    const SeqGroups g = seq_groups(p.cu, p.qlen, j);
    const int n_doc = g.len[2];
    const int r0 = (tile - __ldg(p.tile_base + j)) * BM;
    const int rows_here = min(BM, n_doc - r0);
    const int doc_row0 = g.start + g.off[2] + r0;
    const int G = 1 + g.len[1];
    const bool active = p.doc_rows && wr0 < rows_here;
    const int ra = r0 + wr0 + gq, rb = ra + 8;  // doc-relative rows of this thread

    // Static masks (tile independent except at sequence edges): bit (nb*4 + e)
    // set when that score element is a valid key.
    uint32_t bmask[NBC];
    const bool edge = (r0 - w + wr0 < 0) || (r0 - w + wr0 + 32 * NBC > n_doc);
  #pragma unroll
    for (int bc = 0; bc < NBC; ++bc) {
      uint32_t m = bmask_int[bc];
      if (edge) {  // sequence start / end in reach: drop keys outside [0, n_doc)
  #pragma unroll
        for (int nb = 0; nb < 4; ++nb)
  #pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int t = r0 - w + wr0 + 32 * bc + nb * 8 + 2 * tq + (e & 1);
            if (t < 0 || t >= n_doc) m &= ~(1u << (nb * 4 + e));
          }
      }
      bmask[bc] = m;
    }
    if (j != last_j) {  // global-key mask: per sequence (query-group length, links)
      last_j = j;
  #pragma unroll
      for (int gc = 0; gc < GR / 16; ++gc) {
        uint32_t m = 0;
  #pragma unroll
        for (int nb = 0; nb < 2; ++nb)
  #pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int kg = gc * 16 + nb * 8 + 2 * tq + (e & 1);
            const bool ok = kg < G && (kg == 0 ? p.link_cls : p.link_query);
            m |= (ok ? 1u : 0u) << (nb * 4 + e);
          }
        gmask[gc] = m;
      }
    }
    float ninv_a = 0.f, ninv_b = 0.f;
    if (p.padding == SC_PAD_ZERO_LOGIT) {
      ninv_a = (float)(2 * w + 1 - max(0, min(n_doc, ra + w + 1) - max(0, ra - w)));
      ninv_b = (float)(2 * w + 1 - max(0, min(n_doc, rb + w + 1) - max(0, rb - w)));
    }

    for (int h = 0; h < p.H; ++h, ++it) {
      const int s = it % NS;
      mbar_wait(full_bar + 8 * s, (it / NS) & 1);
      if (active) {
        uint32_t qa[4][4];
        load_q(q_buf(s), wr0, LO, qa);
        float o[8][4];
        zero_o(o);
        float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
        if (ninv_a > 0.f) { m0 = 0.f; l0 = tq == 0 ? ninv_a : 0.f; }
        if (ninv_b > 0.f) { m1 = 0.f; l1 = tq == 0 ? ninv_b : 0.f; }
        float pinv0 = 0.f, pinv1 = 0.f;  // PAIR: 1 / l of head 2h + 1 (its half of O: n-tiles 4-7)
        if constexpr (NBC == 1 && PAIR) {
          // Head pair, single shot per head: heads 2h (dims 0-31) and 2h + 1 (dims 32-63) share the
          // staged rows; two score sets and softmaxes, one O fragment (n-tiles 0-3 / 4-7).
          constexpr int NG = GR / 8;
          float ma0 = m0, ma1 = m1, la0 = l0, la1 = l1;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            float sc[NG + NBB][4];
  #pragma unroll
            for (int gc = 0; gc < GR / 16; ++gc) qk16_hh(kg_buf(s), gc * 16, LO, qa, sc[2 * gc], sc[2 * gc + 1], hh);
            qk16_hh(kb_buf(s), wr0, LO, qa, sc[NG], sc[NG + 1], hh);
            if constexpr (NBB == 4) qk16_hh(kb_buf(s), wr0 + 16, LO, qa, sc[NG + 2], sc[NG + 3], hh);
            else qk8_hh(kb_buf(s), wr0 + 16, lane, qa, sc[NG + 2], hh);
  #pragma unroll
            for (int nb = 0; nb < NG; ++nb)
  #pragma unroll
              for (int e = 0; e < 4; ++e)
                if (!((gmask[nb >> 1] >> ((nb & 1) * 4 + e)) & 1)) sc[nb][e] = -INFINITY;
  #pragma unroll
            for (int nb = 0; nb < NBB; ++nb)
  #pragma unroll
              for (int e = 0; e < 4; ++e)
                if (!((bmask[0] >> (nb * 4 + e)) & 1)) sc[NG + nb][e] = -INFINITY;
            float hm0 = ma0, hm1 = ma1, hl0 = la0, hl1 = la1;
            softmax_update<NG + NBB, true>(sc, c2, hm0, hm1, hl0, hl1, o);
  #pragma unroll
            for (int gc = 0; gc < GR / 16; ++gc) pv16_hh(vg_buf(s), gc * 16, LO, sc[2 * gc], sc[2 * gc + 1], o, hh);
            pv16_hh(vb_buf(s), wr0, LO, sc[NG], sc[NG + 1], o, hh);
            if constexpr (NBB == 4) pv16_hh(vb_buf(s), wr0 + 16, LO, sc[NG + 2], sc[NG + 3], o, hh);
            else pv8_hh(vb_buf(s), wr0 + 16, lane, sc[NG + 2], o, hh);
            if (hh == 0) { m0 = hm0; m1 = hm1; l0 = hl0; l1 = hl1; }  // head 2h
            else { ma0 = hm0; ma1 = hm1; la0 = hl0; la1 = hl1; }      // head 2h + 1
          }
          // head 2h + 1's row sums ride in (la0, la1); normalise its half of O here
          la0 += __shfl_xor_sync(0xffffffffu, la0, 1);
          la0 += __shfl_xor_sync(0xffffffffu, la0, 2);
          la1 += __shfl_xor_sync(0xffffffffu, la1, 1);
          la1 += __shfl_xor_sync(0xffffffffu, la1, 2);
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(pinv0) : "f"(la0));
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(pinv1) : "f"(la1));
        } else if constexpr (NBC == 1) {
          // Single shot: all keys of the row block (globals + band) in one softmax.
          constexpr int NG = GR / 8;
          float sc[NG + NBB][4];
  #pragma unroll
          for (int gc = 0; gc < GR / 16; ++gc) qk16(kg_buf(s), gc * 16, LO, qa, sc[2 * gc], sc[2 * gc + 1]);
          qk16(kb_buf(s), wr0, LO, qa, sc[NG], sc[NG + 1]);
          if constexpr (NBB == 4) qk16(kb_buf(s), wr0 + 16, LO, qa, sc[NG + 2], sc[NG + 3]);
          else qk8(kb_buf(s), wr0 + 16, lane, qa, sc[NG + 2]);
  #pragma unroll
          for (int nb = 0; nb < NG; ++nb)
  #pragma unroll
            for (int e = 0; e < 4; ++e)
              if (!((gmask[nb >> 1] >> ((nb & 1) * 4 + e)) & 1)) sc[nb][e] = -INFINITY;
  #pragma unroll
          for (int nb = 0; nb < NBB; ++nb)
  #pragma unroll
            for (int e = 0; e < 4; ++e)
              if (!((bmask[0] >> (nb * 4 + e)) & 1)) sc[NG + nb][e] = -INFINITY;
          softmax_update<NG + NBB, true>(sc, c2, m0, m1, l0, l1, o);
  #pragma unroll
          for (int gc = 0; gc < GR / 16; ++gc) pv16(vg_buf(s), gc * 16, LO, sc[2 * gc], sc[2 * gc + 1], o);
          pv16(vb_buf(s), wr0, LO, sc[NG], sc[NG + 1], o);
          if constexpr (NBB == 4) pv16(vb_buf(s), wr0 + 16, LO, sc[NG + 2], sc[NG + 3], o);
          else pv8(vb_buf(s), wr0 + 16, lane, sc[NG + 2], o);
        } else {
          // global keys: cls (key 0) and the query group (keys 1..G-1)
  #pragma unroll
          for (int gc = 0; gc < GR / 16; ++gc) {
            float sc[2][4];
            qk16(kg_buf(s), gc * 16, LO, qa, sc[0], sc[1]);
  #pragma unroll
            for (int nb = 0; nb < 2; ++nb)
  #pragma unroll
              for (int e = 0; e < 4; ++e)
                if (!((gmask[gc] >> (nb * 4 + e)) & 1)) sc[nb][e] = -INFINITY;
            softmax_update<2>(sc, c2, m0, m1, l0, l1, o);
            pv16(vg_buf(s), gc * 16, LO, sc[0], sc[1], o);
          }
          // band keys: Kb row 0 = doc row r0 - w; this warp reads rows wr0 + [0, 32*NBC)
  #pragma unroll
          for (int bc = 0; bc < NBC; ++bc) {
            const int kb0 = wr0 + 32 * bc;
            if (QFG && bc == NBC - 1) {  // the band's last 16 keys (16 + 2w <= 48)
              float sc[2][4];
              qk16(kb_buf(s), kb0, LO, qa, sc[0], sc[1]);
  #pragma unroll
              for (int nb = 0; nb < 2; ++nb)
  #pragma unroll
                for (int e = 0; e < 4; ++e)
                  if (!((bmask[bc] >> (nb * 4 + e)) & 1)) sc[nb][e] = -INFINITY;
              softmax_update<2>(sc, c2, m0, m1, l0, l1, o);
              pv16(vb_buf(s), kb0, LO, sc[0], sc[1], o);
              continue;
            }
            float sc[4][4];
            qk16(kb_buf(s), kb0, LO, qa, sc[0], sc[1]);
            qk16(kb_buf(s), kb0 + 16, LO, qa, sc[2], sc[3]);
  #pragma unroll
            for (int nb = 0; nb < 4; ++nb)
  #pragma unroll
              for (int e = 0; e < 4; ++e)
                if (!((bmask[bc] >> (nb * 4 + e)) & 1)) sc[nb][e] = -INFINITY;
            softmax_update<4>(sc, c2, m0, m1, l0, l1, o);
            pv16(vb_buf(s), kb0, LO, sc[0], sc[1], o);
            pv16(vb_buf(s), kb0 + 16, LO, sc[2], sc[3], o);
          }
        }
        l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
        l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
        float i0, i1;  // approximate reciprocal: O leaves as bf16
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(i0) : "f"(l0));
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(i1) : "f"(l1));
        if (wr0 + 16 <= rows_here) {
          // Full 16-row block: stmatrix the bf16 O fragments into this warp's
          // (now dead) Q rows -- same 128B swizzle as the TMA box -- and TMA-store
          // them: 16 rows x 128 B leave in whole lines instead of 16 scattered
          // 4-byte stores per row.
          const uint32_t ob = q_buf(s);
  #pragma unroll
          for (int np = 0; np < 4; ++np) {
            const float a0 = (PAIR && np >= 2) ? pinv0 : i0, a1 = (PAIR && np >= 2) ? pinv1 : i1;
            stsm_x4(ob + wr0 * ROWB + LO.v[np],
                    pack_bf16(o[2 * np][0] * a0, o[2 * np][1] * a0), pack_bf16(o[2 * np][2] * a1, o[2 * np][3] * a1),
                    pack_bf16(o[2 * np + 1][0] * a0, o[2 * np + 1][1] * a0),
                    pack_bf16(o[2 * np + 1][2] * a1, o[2 * np + 1][3] * a1));
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (elect_one()) tma_store_3d(&tmO, ob + wr0 * ROWB, h, doc_row0 + wr0);
          __syncwarp();
        } else {
        __nv_bfloat16* out_h = p.out + h * p.dout + 2 * tq;
        if (ra < n_doc) {
          uint32_t* dst = reinterpret_cast<uint32_t*>(out_h + (int64_t)(doc_row0 + wr0 + gq) * p.ld_out);
  #pragma unroll
          for (int nb = 0; nb < 8; ++nb) {
            const float a0 = (PAIR && nb >= 4) ? pinv0 : i0;
            if (nb * 8 < p.dout) dst[nb * 4] = pack_bf16(o[nb][0] * a0, o[nb][1] * a0);
          }
        }
        if (rb < n_doc) {
          uint32_t* dst = reinterpret_cast<uint32_t*>(out_h + (int64_t)(doc_row0 + wr0 + gq + 8) * p.ld_out);
  #pragma unroll
          for (int nb = 0; nb < 8; ++nb) {
            const float a1 = (PAIR && nb >= 4) ? pinv1 : i1;
            if (nb * 8 < p.dout) dst[nb * 4] = pack_bf16(o[nb][2] * a1, o[nb][3] * a1);
          }
        }
        }
      }

      // Head rows over the global keys (first tile of the sequence only): rows
      // f < G (cls, query group) attend cls / query keys per their links.  Rows
      // with a FULL doc link leave a split-softmax record (merged below); the
      // others (sparse: query rows) are final and stored here.
      if (r0 == 0 && warp == ((h + 2) & (NDOCW - 1))) {
  #pragma unroll
        for (int hh = 0; hh < (PAIR ? 2 : 1); ++hh) {
  #pragma unroll
        for (int fc = 0; fc < GR / 16; ++fc) {
          if (fc * 16 < G) {
            uint32_t qa[4][4];
            if constexpr (QFG) {  // A fragments of rows fc*16 + (gq, gq + 8) straight from their q (L2)
              const int64_t ra0 = g.start + fc * 16 + gq;
  #pragma unroll
              for (int ks = 0; ks < 4; ++ks) {
                qa[ks][0] = ldg_pair(p, h, ra0, ks * 16 + 2 * tq);
                qa[ks][1] = ldg_pair(p, h, ra0 + 8, ks * 16 + 2 * tq);
                qa[ks][2] = ldg_pair(p, h, ra0, ks * 16 + 8 + 2 * tq);
                qa[ks][3] = ldg_pair(p, h, ra0 + 8, ks * 16 + 8 + 2 * tq);
              }
            } else {
              load_q(qf_buf(s), fc * 16, LO, qa);
            }
            float sc[GR / 8][4];
  #pragma unroll
            for (int gc = 0; gc < GR / 16; ++gc) {
              if constexpr (PAIR) qk16_hh(kg_buf(s), gc * 16, LO, qa, sc[2 * gc], sc[2 * gc + 1], hh);
              else qk16(kg_buf(s), gc * 16, LO, qa, sc[2 * gc], sc[2 * gc + 1]);
            }
  #pragma unroll
            for (int nb = 0; nb < GR / 8; ++nb)
  #pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int f = fc * 16 + gq + ((e >> 1) << 3);
                const int kg = nb * 8 + 2 * tq + (e & 1);
                const int grp = f == 0 ? 0 : 1;
                const bool ok = f < G && kg < G && ((hl_bits >> (grp * 2 + (kg == 0 ? 0 : 1))) & 1);
                if (!ok) sc[nb][e] = -INFINITY;
              }
            float o[8][4];
            zero_o(o);
            float hm0 = -INFINITY, hm1 = -INFINITY, hl0 = 0.f, hl1 = 0.f;
            softmax_update<GR / 8, true>(sc, c2, hm0, hm1, hl0, hl1, o);
  #pragma unroll
            for (int gc = 0; gc < GR / 16; ++gc) {
              if constexpr (PAIR) pv16_hh(vg_buf(s), gc * 16, LO, sc[2 * gc], sc[2 * gc + 1], o, hh);
              else pv16(vg_buf(s), gc * 16, LO, sc[2 * gc], sc[2 * gc + 1], o);
            }
            hl0 += __shfl_xor_sync(0xffffffffu, hl0, 1);
            hl0 += __shfl_xor_sync(0xffffffffu, hl0, 2);
            hl1 += __shfl_xor_sync(0xffffffffu, hl1, 1);
            hl1 += __shfl_xor_sync(0xffffffffu, hl1, 2);
            const float to_nat = c2 * 0.69314718055994530942f;
            const int ht = PAIR ? 2 * h + hh : h;  // head of the layout
  #pragma unroll
            for (int half = 0; half < 2; ++half) {
              const int f = fc * 16 + gq + 8 * half;
              if (f >= G) continue;
              const int grp = f == 0 ? 0 : 1;
              const float mm = half ? hm1 : hm0, ll = half ? hl1 : hl0;
              if ((hdoc_bits >> grp) & 1) {
                float* rec = p.partials + (((int64_t)(p.ntiles_max + j) * p.Ht + ht) * p.fmax + f) * REC;
                if (tq == 0) {
                  rec[0] = ll > 0.f ? mm * to_nat : -INFINITY;
                  rec[1] = ll;
                }
  #pragma unroll
                for (int nb = 0; nb < 8; ++nb) {
                  const int src = PAIR ? (nb & 3) + 4 * hh : nb;
                  const bool live = !PAIR || nb < 4;
                  *reinterpret_cast<float2*>(rec + 4 + nb * 8 + 2 * tq) =
                      live ? make_float2(o[src][2 * half], o[src][2 * half + 1]) : make_float2(0.f, 0.f);
                }
              } else {
                const float inv = ll > 0.f ? 1.f / ll : 0.f;
                const int hdim = PAIR ? 32 : p.dout;  // this head's dims
                uint32_t* dst = reinterpret_cast<uint32_t*>(p.out + (int64_t)(g.start + f) * p.ld_out + ht * hdim + 2 * tq);
  #pragma unroll
                for (int nb = 0; nb < 8; ++nb) {
                  const int src = PAIR ? nb + 4 * hh : nb;
                  if (nb * 8 < hdim) dst[nb * 4] = pack_bf16(o[src & 7][2 * half] * inv, o[src & 7][2 * half + 1] * inv);
                }
              }
            }
          }
        }
        }
      }
      __syncwarp();
      if (elect_one()) {  // the same lane that issued this warp's O store
        if (active) tma_store_wait_read();  // the stage's Q rows are about to be refilled
        mbar_arrive(empty_bar + 8 * s);
      }
      __syncwarp();
    }

  }
}

// Merge of the split-softmax records into the head rows with a FULL doc link
// (CLS; query rows under longformer): one CTA of MERGE_WARPS warps per (sequence,
// head, row).  Records: one per doc tile of the sequence + the first tile's
// global-key record.  Warp w folds records w, w + MERGE_WARPS, ... with a running
// max (lane = 2 dims, loads of several records in flight), then warp 0 folds the
// warps' (max, l, acc) through shared memory.  Launched as a programmatic dependent
// of the band kernel (griddepcontrol): its CTAs are resident before the band
// kernel's last CTAs finish, and wait for the grid's records here.
constexpr int MERGE_WARPS = 8;

// WPI warps per (sequence, head, row) item, MERGE_WARPS / WPI items per CTA: 8 for long sequences
// (65 records at 4k tokens), 1 for short ones (passages: 4 records -- one warp folds them all).
template <int WPI>
__global__ void __launch_bounds__(MERGE_WARPS * 32) merge_full_rows_kernel(Params p) {
  constexpr int ITEMS = MERGE_WARPS / WPI;
  __shared__ float sacc[MERGE_WARPS][D];
  __shared__ float sml[MERGE_WARPS][2];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, sub = warp % WPI;
  const int64_t item = (int64_t)blockIdx.x * ITEMS + warp / WPI;
  const int f = (int)(item % p.fmax);
  const int h = (int)((item / p.fmax) % p.H);
  const int j = (int)(item / ((int64_t)p.fmax * p.H));
  bool valid = j < p.nseq;
  SeqGroups g{};
  int nrec = 0;
  const float *trec = nullptr, *grec = nullptr;
  const int64_t rstride = (int64_t)p.H * p.fmax * REC;
  if (valid) {
    g = seq_groups(p.cu, p.qlen, j);
    valid = f < 1 + g.len[1] && p.hdoc[f == 0 ? 0 : 1];
    const int tb = __ldg(p.tile_base + j), te = __ldg(p.tile_base + j + 1);
    nrec = valid ? te - tb + 1 : 0;
    trec = p.partials + (((int64_t)tb * p.H + h) * p.fmax + f) * REC;
    grec = p.partials + (((int64_t)(p.ntiles_max + j) * p.H + h) * p.fmax + f) * REC;
  }
  auto rec_of = [&](int r) { return r < nrec - 1 ? trec + r * rstride : grec; };

  float M = -INFINITY, l = 0.f, a0 = 0.f, a1 = 0.f;
  constexpr int U = 4;  // records in flight per warp
  for (int base = sub; base < nrec; base += U * WPI) {
    float2 ml[U], v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = base + u * WPI;
      if (r < nrec) {
        const float* rc = rec_of(r);
        ml[u] = __ldg(reinterpret_cast<const float2*>(rc));
        v[u] = __ldg(reinterpret_cast<const float2*>(rc + 4 + 2 * lane));
      } else {
        ml[u] = make_float2(-INFINITY, 0.f);
        v[u] = make_float2(0.f, 0.f);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!(ml[u].y > 0.f)) continue;  // warp-uniform (every lane reads the same (m, l))
      if (ml[u].x > M) {
        const float sc = __expf(M - ml[u].x);  // M = -inf: 0
        l *= sc; a0 *= sc; a1 *= sc;
        M = ml[u].x;
      }
      const float b = __expf(ml[u].x - M);
      l = fmaf(b, ml[u].y, l);
      a0 = fmaf(b, v[u].x, a0);
      a1 = fmaf(b, v[u].y, a1);
    }
  }
  if constexpr (WPI > 1) {  // fold the item's warps through shared memory (one item per CTA)
    sacc[warp][2 * lane] = a0;
    sacc[warp][2 * lane + 1] = a1;
    if (lane == 0) { sml[warp][0] = M; sml[warp][1] = l; }
    __syncthreads();
    if (sub != 0) return;
    float Mt = -INFINITY;
#pragma unroll
    for (int w = 0; w < WPI; ++w) Mt = fmaxf(Mt, sml[warp + w][0]);
    float lt = 0.f, o0 = 0.f, o1 = 0.f;
#pragma unroll
    for (int w = 0; w < WPI; ++w) {
      if (!(sml[warp + w][1] > 0.f)) continue;
      const float sc = __expf(sml[warp + w][0] - Mt);
      lt = fmaf(sc, sml[warp + w][1], lt);
      o0 = fmaf(sc, sacc[warp + w][2 * lane], o0);
      o1 = fmaf(sc, sacc[warp + w][2 * lane + 1], o1);
    }
    l = lt; a0 = o0; a1 = o1;
  }
  if (!valid) return;
  const float inv = l > 0.f ? 1.f / l : 0.f;
  if (2 * lane < p.dout) {
    __nv_bfloat16* dst = p.out + (int64_t)(g.start + f) * p.ld_out + h * p.dout + 2 * lane;
    *reinterpret_cast<uint32_t*>(dst) = pack_bf16(a0 * inv, a1 * inv);
  }
}

// Programmatic-dependent launch of the merge: 8 warps per item for long sequences, 1 for short ones
// (average doc tiles per sequence <= 16: at most ~17 records).
static int launch_merge(const Params& p, int64_t items, int64_t total_tokens, cudaStream_t st) {
  const bool short_seqs = total_tokens <= (int64_t)p.nseq * 16 * BM;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(short_seqs ? (items + MERGE_WARPS - 1) / MERGE_WARPS : items));
  cfg.blockDim = dim3(MERGE_WARPS * 32);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (short_seqs) cudaLaunchKernelEx(&cfg, merge_full_rows_kernel<1>, p);
  else cudaLaunchKernelEx(&cfg, merge_full_rows_kernel<MERGE_WARPS>, p);
  SC_CHECK_LAUNCH("merge_full_rows_kernel");
  return SC_OK;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(ptr);
  }
  return fn;
}

// [rows][heads][d] bf16 (row stride ld elements) as a 3-D map with 64 x 1 x box_rows boxes
static bool make_map(CUtensorMap* m, const void* base, int d, int heads, int64_t rows, int64_t ld_elems,
                     int box_rows) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)heads, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)(d * 2), (cuuint64_t)(ld_elems * 2)};
  cuuint32_t box[3] = {(cuuint32_t)D, 1u, (cuuint32_t)box_rows};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             SC_BAND_L2PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

using KernelFn = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, Params);

// Stage count: as many as fit two CTAs per SM (<= ~113 KB each), at least 2.
template <int NBC, int GR, int QFG = 0>
constexpr int stage_bytes_of() {
  return (BM + (QFG ? 2 : 3) * GR + 2 * (QFG ? 96 : 48 + 32 * NBC)) * ROWB;
}
template <int NBC, int GR, int QFG = 0>
constexpr int stages_for() {
  constexpr int budget = 227 * 1024 / min_ctas(NBC, QFG) - 2048;
  return (3 * stage_bytes_of<NBC, GR, QFG>() <= budget) ? 3 : 2;
}

template <int NBC, int GR, int NBB = 4, int PAIR = 0, int QFG = 0>
static int launch_one(const CUtensorMap* maps, const Params& p, unsigned grid, cudaStream_t st) {
  constexpr int NS = stages_for<NBC, GR, QFG>();
  constexpr int stage_bytes = stage_bytes_of<NBC, GR, QFG>();
  constexpr size_t smem = (size_t)NS * stage_bytes + 2 * NS * 8 + 64 + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(band_attn_kernel<NBC, GR, NS, NBB, PAIR, QFG>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (cudaFuncSetAttribute(band_attn_kernel<NBC, GR, NS, NBB, PAIR, QFG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess) {
      set_error("band kernel: shared memory request of %zu bytes failed", smem);
      return SC_ERR_UNSUPPORTED;
    }
    attr = true;
  }
  // Persistent grid: every resident CTA slot (SMs x CTAs/SM) loops over tiles.
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (num_sms <= 0) num_sms = 148;
  }
  static int grid_cap = -1;  // measurement only (SC_BAND_GRID=N): persistent grid of N CTAs
  if (grid_cap < 0) grid_cap = getenv("SC_BAND_GRID") ? atoi(getenv("SC_BAND_GRID")) : 0;
  const unsigned slots = grid_cap > 0 ? (unsigned)grid_cap : (unsigned)(num_sms * min_ctas(NBC, QFG));
  band_attn_kernel<NBC, GR, NS, NBB, PAIR, QFG><<<grid < slots ? grid : slots, NTHREADS, smem, st>>>(
      maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], maps[6], p);
  SC_CHECK_LAUNCH("band_attn_kernel");
  return SC_OK;
}

// SC_BAND_QFG=0 keeps the 2-CTA, Qf-staged form for 8 < w <= 16 (measurement A/B)
static bool qfg_enabled() {
  static int v = -1;
  if (v < 0) v = getenv("SC_BAND_QFG") ? atoi(getenv("SC_BAND_QFG")) : 1;
  return v != 0;
}

template <int GR>
static int launch_gr(int nbc, bool pair, const CUtensorMap* maps, const Params& p, unsigned grid, cudaStream_t st) {
  if (pair && nbc == 1)
    return p.w <= 4 ? launch_one<1, GR, 3, 1>(maps, p, grid, st) : launch_one<1, GR, 4, 1>(maps, p, grid, st);
  switch (nbc) {
    case 1: return p.w <= 4 ? launch_one<1, GR, 3>(maps, p, grid, st) : launch_one<1, GR>(maps, p, grid, st);
    case 2:
      if (GR == 16 && p.w <= 16 && qfg_enabled()) return launch_one<2, 16, 4, 0, 1>(maps, p, grid, st);
      return launch_one<2, GR>(maps, p, grid, st);
    case 3: return launch_one<3, GR>(maps, p, grid, st);
    case 4: return launch_one<4, GR>(maps, p, grid, st);
    case 5: return launch_one<5, GR>(maps, p, grid, st);
    case 6: return launch_one<6, GR>(maps, p, grid, st);
    case 7: return launch_one<7, GR>(maps, p, grid, st);
  }
  set_error("band kernel: window too large");
  return SC_ERR_UNSUPPORTED;
}

}  // namespace bandk

size_t band_workspace_bytes(int nseq, int T, int H, int d, int tile_rows, int max_qgroup_len,
                            const Links& L) {
  int f = full_rows_needed(L, max_qgroup_len);
  if (f == 0 || tile_rows <= 0) return 0;
  // records: one per doc tile (<= ceil(T/64) + nseq) + one global-key record per
  // sequence, each H x f x (m, l, pad, pad, acc[d]).
  int64_t recs = (T + tile_rows - 1) / tile_rows + 2 * (int64_t)nseq;
  return (size_t)recs * H * f * ((d < 64 ? 64 : d) + 4) * sizeof(float);  // records keep 64 dims (d = 32 zero-padded)
}

int launch_attn_band(const AttnArgs& a, int dtype, const int32_t* seq_tile_base,
                     const int32_t* seq_head_base, int tile_rows, int max_qgroup_len, void* ws,
                     size_t ws_bytes, cudaStream_t st, bool doc_rows) {
  using namespace bandk;
  const Links& L = a.links;
  // Head-rows-only mode stages just the tile's own 64 doc keys (no halo).
  const int w = doc_rows ? L.w[2][2] : 0;
  auto unsupported = [](const char* why) {
    set_error("band kernel: %s", why);
    return SC_ERR_UNSUPPORTED;
  };
  if (dtype != SC_DTYPE_BF16) return unsupported("needs bf16");
  if (a.d != D && a.d != 32) return unsupported("needs head_dim 32 or 64");
  // QDS head rows attend every key (like longformer), so head-rows-only mode
  // ignores the globals; QDS doc rows need the tcgen05 kernel's dense segment.
  if (a.glob_cu && doc_rows) return unsupported("QDS global tokens");
  if (w < 0 || w > MAX_W) return unsupported("doc->doc link must be a window <= 96");
  for (int x : {L.w[2][0], L.w[2][1], L.w[0][2], L.w[1][2], L.w[0][0], L.w[0][1], L.w[1][0], L.w[1][1]})
    if (x != SC_LINK_FULL && x != SC_LINK_NONE) return unsupported("windowed link outside doc->doc");
  if (max_qgroup_len + 1 > 64) return unsupported("query group longer than 63 rows");
  if (tile_rows != BM || !seq_tile_base || !seq_head_base) return unsupported("layout tiles must be 64 rows");
  if (((uintptr_t)a.q | (uintptr_t)a.k | (uintptr_t)a.v | (uintptr_t)a.out) & 15)
    return unsupported("16-byte alignment");
  if ((a.ld * 2) % 16 || (a.ld_out * 2) % 16) return unsupported("row strides");
  const int fneed = full_rows_needed(L, max_qgroup_len);
  const size_t need = band_workspace_bytes(a.nseq, a.T, a.H, a.d, tile_rows, max_qgroup_len, L);
  if (need > ws_bytes || (need && !ws)) return unsupported("workspace too small");
  const int GR = (max_qgroup_len + 1 <= 16) ? 16 : (max_qgroup_len + 1 <= 32 ? 32 : 64);

  // head_dim 32, single-chunk windows: items are head pairs (64-dim rows of two adjacent heads);
  // SC_BAND_NOPAIR=1 keeps one zero-padded head per item (measurement A/B)
  const int nbc0 = (16 + 2 * w + 31) / 32;
  static int nopair = -1;
  if (nopair < 0) nopair = getenv("SC_BAND_NOPAIR") ? atoi(getenv("SC_BAND_NOPAIR")) : 0;
  const bool pair = doc_rows && a.d == 32 && a.H % 2 == 0 && nbc0 == 1 && !nopair;
  CUtensorMap maps[7];
  const int dd = pair ? 64 : a.d, H = pair ? a.H / 2 : a.H;
  if (!make_map(&maps[0], a.q, dd, H, a.T, a.ld, BM) || !make_map(&maps[1], a.q, dd, H, a.T, a.ld, GR) ||
      !make_map(&maps[2], a.k, dd, H, a.T, a.ld, GR) || !make_map(&maps[3], a.v, dd, H, a.T, a.ld, GR) ||
      !make_map(&maps[4], a.k, dd, H, a.T, a.ld, BM + 2 * w) ||
      !make_map(&maps[5], a.v, dd, H, a.T, a.ld, BM + 2 * w) ||
      !make_map(&maps[6], a.out, dd, H, a.T, a.ld_out, 16))
    return unsupported("cuTensorMapEncodeTiled failed");

  Params p;
  p.nseq = a.nseq; p.H = H; p.Ht = a.H; p.w = w; p.doc_rows = doc_rows ? 1 : 0; p.dout = pair ? 64 : a.d;
  const int nbc = (16 + 2 * w + 31) / 32;
  p.kb_rows = 48 + 32 * nbc;
  p.fneed = fneed; p.fmax = fneed; p.padding = a.padding;
  p.link_cls = L.w[2][0] == SC_LINK_FULL; p.link_query = L.w[2][1] == SC_LINK_FULL;
  p.c2 = 1.4426950408889634f / a.scale;
  p.cu = a.cu; p.qlen = a.qlen; p.tile_base = seq_tile_base;
  p.q = static_cast<const __nv_bfloat16*>(a.q); p.ld_q = a.ld; p.T = a.T;
  p.out = static_cast<__nv_bfloat16*>(a.out); p.ld_out = a.ld_out;
  p.partials = static_cast<float*>(ws);
  for (int gsrc = 0; gsrc < 2; ++gsrc) {
    p.hl[gsrc][0] = L.w[gsrc][0] == SC_LINK_FULL;
    p.hl[gsrc][1] = L.w[gsrc][1] == SC_LINK_FULL;
    p.hdoc[gsrc] = L.w[gsrc][2] == SC_LINK_FULL;
  }
  const unsigned grid = (unsigned)((a.T + BM - 1) / BM + a.nseq);  // upper bound on tiles (record indexing)
  p.ntiles_max = (int)grid;
  static int rev = -1;
  if (rev < 0) {
    const char* e = getenv("SC_BAND_REVERSE");
    rev = e ? (atoi(e) != 0) : 1;
  }
  p.reverse = rev;
  static int cls_skip = -1;
  if (cls_skip < 0) cls_skip = getenv("SC_BAND_CLS_SKIP") ? atoi(getenv("SC_BAND_CLS_SKIP")) : 0;
  p.cls_skip = cls_skip;
  // Doc rows + head rows over the global keys (first tile of each sequence).
  // (seq_head_base is unused: head rows are addressed through cu_seqlens.)
  (void)seq_head_base;
  int rc = GR == 16 ? launch_gr<16>(nbc, pair, maps, p, grid, st)
         : GR == 32 ? launch_gr<32>(nbc, pair, maps, p, grid, st)
                    : launch_gr<64>(nbc, pair, maps, p, grid, st);
  if (rc || fneed == 0) return rc;
  Params pm = p;  // the merge walks the layout's heads
  pm.H = a.H;
  pm.dout = a.d;
  return launch_merge(pm, (int64_t)a.nseq * a.H * fneed, a.T, st);
}

int launch_head_merge(const AttnArgs& a, const int32_t* seq_tile_base, int tile_rows, int max_qgroup_len, void* ws,
                      cudaStream_t st) {
  using namespace bandk;
  const Links& L = a.links;
  const int fneed = full_rows_needed(L, max_qgroup_len);
  if (fneed == 0) return SC_OK;
  Params p{};
  p.nseq = a.nseq; p.H = a.H; p.Ht = a.H; p.fneed = fneed; p.fmax = fneed; p.dout = a.d;
  p.cu = a.cu; p.qlen = a.qlen; p.tile_base = seq_tile_base;
  p.out = static_cast<__nv_bfloat16*>(a.out); p.ld_out = a.ld_out;
  p.partials = static_cast<float*>(ws);
  p.ntiles_max = (int)((a.T + tile_rows - 1) / tile_rows + a.nseq);
  for (int gsrc = 0; gsrc < 2; ++gsrc) p.hdoc[gsrc] = L.w[gsrc][2] == SC_LINK_FULL;
  return launch_merge(p, (int64_t)a.nseq * a.H * fneed, a.T, st);
}

}  // namespace sc
