// fp32 doc-band attention for the parity path (precision "f32" / "f64").
//
// The generic kernel (attn_generic.cu) gives every (row, head) one warp and
// one serial online-softmax chain: latency-bound (3.5 ms per layer at
// 8 x 4099 tokens).  Here a CTA takes 64 doc rows of one sequence x one head,
// stages the band keys / values (64 + 2w rows) and the cls / query-group keys
// in shared memory, and gives each row four threads that each own 16 of the
// 64 dims: per key, 16 FMAs per thread, a two-step shuffle to complete the
// dot product, the online softmax update (replicated in the four threads) and
// 16 FMAs of P V.  fp32 math throughout, the reference's key set and padding
// semantics (R/band.py:48-52, R/attention.py:228-257): band keys
// |t - r| <= w inside the doc, the cls / query keys when linked, zero-logit
// padding slots entering with logit 0.  Head rows go to the generic kernel.
#include <cuda_fp16.h>
#include <stdlib.h>

#include "attn.cuh"
#include "mma_tile.cuh"

namespace sc {
namespace bandf {

constexpr int BM = 64;       // doc rows per CTA
constexpr int D = 64;
constexpr int MAXW = 32;     // band window supported
constexpr int KB = BM + 2 * MAXW;
constexpr int MAXH = 32;     // cls + query-group keys
constexpr int NT = 4 * BM;   // four threads per row

struct Params {
  const float *q, *k, *v;
  int64_t ld;
  float* out;
  int64_t ld_out;
  const int32_t *cu, *qlen, *tile_base;
  int nseq, H, w, padding, link_cls, link_query;
  float scale;
  int32_t* status;
  // split-softmax records of the full rows (cls; query rows under longformer) over each tile's own
  // doc keys: rec[((tile * H + h) * fmax + f) * (D + 2)] = (m, l, acc[D]), merged by the generic
  // kernel's head-row pass
  float* partials;
  int fneed, fmax;
};

constexpr int DP = D + 4;  // padded smem row (floats): neighbouring rows land 4 banks apart

__global__ void __launch_bounds__(NT) band_f32_kernel(Params p) {
  extern __shared__ float4 smem_f4[];
  float* smem = reinterpret_cast<float*>(smem_f4);
  const int tile = blockIdx.x, h = blockIdx.y;
  if (tile >= __ldg(p.tile_base + p.nseq)) return;  // grid is an upper bound
  const int j = find_seq(p.tile_base, p.nseq, tile);
  const SeqGroups g = seq_groups(p.cu, p.qlen, j);
  const int dlen = g.len[2], dstart = g.start + g.off[2];
  const int r0 = (tile - __ldg(p.tile_base + j)) * BM;
  const int w = p.w, hoff = h * D;
  const int nhead = 1 + g.len[1];
  const int kb_rows = BM + 2 * w;
  float* sK = smem;                      // [kb_rows][DP]
  float* sV = sK + kb_rows * DP;         // [kb_rows][DP]
  float* sKh = sV + kb_rows * DP;        // [MAXH][DP]
  float* sVh = sKh + MAXH * DP;          // [MAXH][DP]

  // stage band K/V rows (doc positions r0 - w ..) and the head keys, float4 per thread
  for (int idx = threadIdx.x; idx < kb_rows * (D / 4); idx += NT) {
    const int r = idx / (D / 4), c = (idx % (D / 4)) * 4;
    const int pos = r0 - w + r;
    float4 kv = make_float4(0.f, 0.f, 0.f, 0.f), vv = kv;
    if (pos >= 0 && pos < dlen) {
      kv = *reinterpret_cast<const float4*>(p.k + (int64_t)(dstart + pos) * p.ld + hoff + c);
      vv = *reinterpret_cast<const float4*>(p.v + (int64_t)(dstart + pos) * p.ld + hoff + c);
    }
    *reinterpret_cast<float4*>(sK + r * DP + c) = kv;
    *reinterpret_cast<float4*>(sV + r * DP + c) = vv;
  }
  for (int idx = threadIdx.x; idx < nhead * (D / 4); idx += NT) {
    const int r = idx / (D / 4), c = (idx % (D / 4)) * 4;
    *reinterpret_cast<float4*>(sKh + r * DP + c) =
        *reinterpret_cast<const float4*>(p.k + (int64_t)(g.start + r) * p.ld + hoff + c);
    *reinterpret_cast<float4*>(sVh + r * DP + c) =
        *reinterpret_cast<const float4*>(p.v + (int64_t)(g.start + r) * p.ld + hoff + c);
  }

  const int rl = threadIdx.x >> 2, part = threadIdx.x & 3;  // row in tile, dim quarter
  const int rs = r0 + rl;                                    // doc-relative row
  const int c0 = part * 16;
  __syncthreads();

  // full-row records: head row f against this tile's 64 doc keys (smem band rows w .. w + 63)
  if (p.partials) {
    float* qf = sKh + MAXH * DP * 2;  // [D] (after sVh)
    float* ps = qf + D;               // [BM]
    float* red = ps + BM;             // [4][D] + [4]
    for (int f = 0; f < p.fneed && f < nhead; ++f) {
      if (threadIdx.x < D) qf[threadIdx.x] = p.q[(int64_t)(g.start + f) * p.ld + hoff + threadIdx.x];
      __syncthreads();
      float sdot = 0.f;
      const float* kr = sK + (w + rl) * DP + c0;
#pragma unroll
      for (int e = 0; e < 16; ++e) sdot = fmaf(qf[c0 + e], kr[e], sdot);
      sdot += __shfl_xor_sync(0xffffffffu, sdot, 1);
      sdot += __shfl_xor_sync(0xffffffffu, sdot, 2);
      if (part == 0) ps[rl] = rs < dlen ? sdot / p.scale : -INFINITY;
      __syncthreads();
      if (threadIdx.x < 32) {  // max and sum over the 64 keys by one warp
        float mx = fmaxf(ps[threadIdx.x], ps[threadIdx.x + 32]);
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float e0 = mx == -INFINITY ? 0.f : expf(ps[threadIdx.x] - mx);
        const float e1 = mx == -INFINITY ? 0.f : expf(ps[threadIdx.x + 32] - mx);
        ps[threadIdx.x] = e0;
        ps[threadIdx.x + 32] = e1;
        float sm = e0 + e1;
        for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
        if (threadIdx.x == 0) { red[4 * D] = mx; red[4 * D + 1] = sm; }
      }
      __syncthreads();
      {  // acc[c] = sum_k p_k v_k[c]: thread (c, quarter of the keys)
        const int c = threadIdx.x & (D - 1), sub = threadIdx.x >> 6;
        float a2 = 0.f;
        for (int kk = sub * 16; kk < sub * 16 + 16; ++kk) a2 = fmaf(ps[kk], sV[(w + kk) * DP + c], a2);
        red[sub * D + c] = a2;
      }
      __syncthreads();
      if (threadIdx.x < D) {
        float* rec = p.partials + (((int64_t)tile * p.H + h) * p.fmax + f) * (D + 2);
        rec[2 + threadIdx.x] = red[threadIdx.x] + red[D + threadIdx.x] + red[2 * D + threadIdx.x] +
                               red[3 * D + threadIdx.x];
        if (threadIdx.x == 0) { rec[0] = red[4 * D]; rec[1] = red[4 * D + 1]; }
      }
      __syncthreads();
    }
  }
  float q[16];
  if (rs < dlen) {
    const float* qr = p.q + (int64_t)(dstart + rs) * p.ld + hoff + c0;
#pragma unroll
    for (int e = 0; e < 16; e += 4) {
      const float4 t = *reinterpret_cast<const float4*>(qr + e);
      q[e] = t.x; q[e + 1] = t.y; q[e + 2] = t.z; q[e + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int e = 0; e < 16; ++e) q[e] = 0.f;
  }
  __syncthreads();

  float m = -INFINITY, l = 0.f, acc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) acc[e] = 0.f;
  if (p.padding == SC_PAD_ZERO_LOGIT && rs < dlen) {
    const int lo = max(0, rs - w), hi = min(dlen, rs + w + 1);
    const int n_inv = (2 * w + 1) - max(0, hi - lo);
    if (n_inv > 0) { m = 0.f; l = (float)n_inv; }
  }
  // one key: dot over this thread's 16 dims, completed across the row's four threads
  auto key = [&](const float* kr, const float* vr, bool valid) {
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < 16; e += 4) {
      const float4 t = *reinterpret_cast<const float4*>(kr + c0 + e);
      s = fmaf(q[e], t.x, fmaf(q[e + 1], t.y, fmaf(q[e + 2], t.z, fmaf(q[e + 3], t.w, s))));
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (!valid) return;
    s = s / p.scale;
    if (s > m) {
      const float alpha = m == -INFINITY ? 0.f : expf(m - s);
      l *= alpha;
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[e] *= alpha;
      m = s;
    }
    const float pk = expf(s - m);
    l += pk;
#pragma unroll
    for (int e = 0; e < 16; e += 4) {
      const float4 t = *reinterpret_cast<const float4*>(vr + c0 + e);
      acc[e] = fmaf(pk, t.x, acc[e]);
      acc[e + 1] = fmaf(pk, t.y, acc[e + 1]);
      acc[e + 2] = fmaf(pk, t.z, acc[e + 2]);
      acc[e + 3] = fmaf(pk, t.w, acc[e + 3]);
    }
  };
  // pattern order: cls, query group, doc band (R/attention.py segment order; the softmax is joint)
  if (p.link_cls) key(sKh, sVh, rs < dlen);
  if (p.link_query)
    for (int t = 1; t < nhead; ++t) key(sKh + t * DP, sVh + t * DP, rs < dlen);
  // band: smem row rl + b addresses doc position rs - w + b
  for (int b = 0; b <= 2 * w; ++b) {
    const int pos = rs - w + b;
    key(sK + (rl + b) * DP, sV + (rl + b) * DP, rs < dlen && pos >= 0 && pos < dlen);
  }
  if (rs >= dlen) return;
  float* o = p.out + (int64_t)(dstart + rs) * p.ld_out + hoff + c0;
  if (!(l > 0.f)) {
    if (part == 0 && p.status) atomicOr(p.status, 1);
#pragma unroll
    for (int e = 0; e < 16; e += 4) *reinterpret_cast<float4*>(o + e) = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const float inv = 1.f / l;
#pragma unroll
  for (int e = 0; e < 16; e += 4)
    *reinterpret_cast<float4*>(o + e) = make_float4(acc[e] * inv, acc[e + 1] * inv, acc[e + 2] * inv, acc[e + 3] * inv);
}

}  // namespace bandf


// ---------------------------------------------------------------------------
// The same doc-band attention on the tensor cores: fp32 operands as fp16 pairs
// (x = hi + lo, hi = fp16_rn(x), lo = fp16_rn(x - hi): 22 significant bits) and
// three mma.sync m16n8k16 products per contraction, hi.hi + hi.lo + lo.hi
// (dropped lo.lo <= 2^-22 relative), fp32 accumulation -- for S = Q K^T and for
// O = P V alike.  CTA = 64 doc rows x 1 head, 4 warps x 16 rows; K / V of the
// band (64 + 2w rows) and of the cls / query keys staged once per CTA as hi / lo
// planes in 128B-swizzled shared memory (ldmatrix-able), Q straight from global
// into A fragments.  One softmax over the row's whole key set (globals + band:
// at most 32 + 80 keys).  The rotating warp (h % 4) also writes the full rows'
// split-softmax records over the tile's own 64 keys (cls; query rows under
// longformer / full) in the band_f32_kernel format.  The old SIMT kernel re-read
// 2w + 1 K/V rows from shared memory per row and was bound by shared-memory
// bandwidth (1.3 ms per layer at 32 x 4099); this one reads each staged row once
// per 16-row block through ldmatrix.
namespace bandx3 {

constexpr int BM = 64, D = 64, MAXW = 32, GRM = 32, NT = 128;
constexpr int MAXCH = (16 + 2 * MAXW + 15) / 16;  // band chunks of 16 keys per 16-row block
constexpr int ROWB = 128;                          // one plane row: 64 fp16

__device__ __forceinline__ void mma_h(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// (x, y) -> packed fp16 hi pair and the packed fp16 residual pair
__device__ __forceinline__ void split_h2(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x, y);
  const float2 f = __half22float2(h);
  const __half2 l = __floats2half2_rn(x - f.x, y - f.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
// C(16 x 16 keys, two n8 tiles) += A(16 x 64) . B[row0 .. row0+15]^T
__device__ __forceinline__ void qk16h(uint32_t bbuf, int row0, int lane, const uint32_t (&a)[4][4], float (&c0)[4],
                                      float (&c1)[4]) {
  const int brow = row0 + (lane & 7) + ((lane >> 4) << 3);
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    uint32_t b[4];
    mmat::ldsm_x4(mmat::swz(bbuf, brow, ks * 2 + ((lane >> 3) & 1)), b);
    mma_h(c0, a[ks], b[0], b[1]);
    mma_h(c1, a[ks], b[2], b[3]);
  }
}
// O(16 x 64) += A(16 x 16 keys) . B[row0 .. row0+15]  (B rows = keys)
__device__ __forceinline__ void pv16h(uint32_t bbuf, int row0, int lane, const uint32_t (&a)[4], float (&o)[8][4]) {
  const int brow = row0 + (lane & 7) + (((lane >> 3) & 1) << 3);
#pragma unroll
  for (int np = 0; np < 4; ++np) {
    uint32_t b[4];
    mmat::ldsm_x4_t(mmat::swz(bbuf, brow, np * 2 + (lane >> 4)), b);
    mma_h(o[2 * np], a, b[0], b[1]);
    mma_h(o[2 * np + 1], a, b[2], b[3]);
  }
}
// S += Q K^T over one 16-key block in three products (small terms first)
__device__ __forceinline__ void qk16x3(uint32_t kh, uint32_t kl, int row0, int lane, const uint32_t (&qh)[4][4],
                                       const uint32_t (&ql)[4][4], float (&c0)[4], float (&c1)[4]) {
  qk16h(kl, row0, lane, qh, c0, c1);
  qk16h(kh, row0, lane, ql, c0, c1);
  qk16h(kh, row0, lane, qh, c0, c1);
}
// O += P V over one 16-key block (P as two C-layout n8 tiles of fp32 probabilities)
__device__ __forceinline__ void pv16x3(uint32_t vh, uint32_t vl, int row0, int lane, const float (&p0)[4],
                                       const float (&p1)[4], float (&o)[8][4]) {
  uint32_t ah[4], al[4];
  split_h2(p0[0], p0[1], ah[0], al[0]);
  split_h2(p0[2], p0[3], ah[1], al[1]);
  split_h2(p1[0], p1[1], ah[2], al[2]);
  split_h2(p1[2], p1[3], ah[3], al[3]);
  pv16h(vl, row0, lane, ah, o);
  pv16h(vh, row0, lane, al, o);
  pv16h(vh, row0, lane, ah, o);
}
// A fragments (hi, lo) of 16 fp32 rows x 64 dims straight from global; row(i) == nullptr -> zeros
template <typename F>
__device__ __forceinline__ void load_q_x3(int lane, F&& row, uint32_t (&qh)[4][4], uint32_t (&ql)[4][4]) {
  const int gq = lane >> 2, tq = lane & 3;
  const float* r0 = row(gq);
  const float* r1 = row(gq + 8);
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int c = ks * 16 + half * 8 + 2 * tq;
      const float2 a = r0 ? *reinterpret_cast<const float2*>(r0 + c) : make_float2(0.f, 0.f);
      const float2 b = r1 ? *reinterpret_cast<const float2*>(r1 + c) : make_float2(0.f, 0.f);
      split_h2(a.x, a.y, qh[ks][2 * half], ql[ks][2 * half]);
      split_h2(b.x, b.y, qh[ks][2 * half + 1], ql[ks][2 * half + 1]);
    }
  }
}
// The fp32 values behind load_q_x3's fragments (raw[ks][2 * half + row8]), and their split.
template <typename F>
__device__ __forceinline__ void load_q_raw(int lane, F&& row, float2 (&raw)[4][4]) {
  const int gq = lane >> 2, tq = lane & 3;
  const float* r0 = row(gq);
  const float* r1 = row(gq + 8);
#pragma unroll
  for (int ks = 0; ks < 4; ++ks)
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int c = ks * 16 + half * 8 + 2 * tq;
      raw[ks][2 * half] = r0 ? __ldg(reinterpret_cast<const float2*>(r0 + c)) : make_float2(0.f, 0.f);
      raw[ks][2 * half + 1] = r1 ? __ldg(reinterpret_cast<const float2*>(r1 + c)) : make_float2(0.f, 0.f);
    }
}
__device__ __forceinline__ void split_q(const float2 (&raw)[4][4], uint32_t (&qh)[4][4], uint32_t (&ql)[4][4]) {
#pragma unroll
  for (int ks = 0; ks < 4; ++ks)
#pragma unroll
    for (int i = 0; i < 4; ++i) split_h2(raw[ks][i].x, raw[ks][i].y, qh[ks][i], ql[ks][i]);
}
// hi / lo planes of `nrows` fp32 rows (64 dims) into swizzled smem; row(i) == nullptr -> zeros.
// Loads are issued in batches of UNR float4 per thread before any is split and stored, so a
// thread keeps UNR global loads in flight (one-at-a-time staging was load-latency bound).
constexpr int UNR = 8;
template <typename F>
__device__ __forceinline__ void stage_x3(uint32_t hbuf, uint32_t lbuf, int nrows, F&& row) {
  const int n = nrows * 16;
  for (int base = 0; base < n; base += NT * UNR) {
    float4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int idx = base + u * NT + threadIdx.x;
      const float* src = idx < n ? row(idx >> 4) : nullptr;
      v[u] = src ? __ldg(reinterpret_cast<const float4*>(src + 4 * (idx & 15))) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int idx = base + u * NT + threadIdx.x;
      if (idx >= n) break;
      const int r = idx >> 4, c4 = idx & 15;
      uint32_t h0, l0, h1, l1;
      split_h2(v[u].x, v[u].y, h0, l0);
      split_h2(v[u].z, v[u].w, h1, l1);
      const uint32_t off = (c4 & 1) * 8;
      asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(mmat::swz(hbuf, r, c4 >> 1) + off), "r"(h0), "r"(h1));
      asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(mmat::swz(lbuf, r, c4 >> 1) + off), "r"(l0), "r"(l1));
    }
  }
}

__global__ void __launch_bounds__(NT, 4) band_f32x3_kernel(bandf::Params p) {
  extern __shared__ __align__(1024) uint8_t smem_x3[];
  const int tile = blockIdx.x, h = blockIdx.y;
  if (tile >= __ldg(p.tile_base + p.nseq)) return;  // grid is an upper bound
  const int j = find_seq(p.tile_base, p.nseq, tile);
  const SeqGroups g = seq_groups(p.cu, p.qlen, j);
  const int dlen = g.len[2], dstart = g.start + g.off[2];
  const int r0 = (tile - __ldg(p.tile_base + j)) * BM;
  const int rows_here = min(BM, dlen - r0);
  const int w = p.w, hoff = h * D;
  const int nhead = 1 + g.len[1];
  const int kb_rows = (BM + 2 * w + 15) & ~15;
  const uint32_t sm = mmat::smem_u32(smem_x3);
  const uint32_t KH = sm, KL = KH + kb_rows * ROWB, VH = KL + kb_rows * ROWB, VL = VH + kb_rows * ROWB;
  const uint32_t GKH = VL + kb_rows * ROWB, GKL = GKH + GRM * ROWB, GVH = GKL + GRM * ROWB, GVL = GVH + GRM * ROWB;

  // stage the band rows (doc positions r0 - w ..) and the cls / query keys as hi / lo planes
  auto band_k = [&](int r) -> const float* {
    const int pos = r0 - w + r;
    return (pos >= 0 && pos < dlen) ? p.k + (int64_t)(dstart + pos) * p.ld + hoff : nullptr;
  };
  auto band_v = [&](int r) -> const float* {
    const int pos = r0 - w + r;
    return (pos >= 0 && pos < dlen) ? p.v + (int64_t)(dstart + pos) * p.ld + hoff : nullptr;
  };
  // this thread's Q fragment values (rows gq, gq + 8 of its warp's block), loaded before the staging
  // so their latency overlaps it
  float2 qraw[4][4];
  {
    const int wq = (threadIdx.x >> 5) * 16, lq = threadIdx.x & 31;
    load_q_raw(lq, [&](int i) -> const float* {
      return wq + i < rows_here ? p.q + (int64_t)(dstart + r0 + wq + i) * p.ld + hoff : nullptr;
    }, qraw);
  }
  stage_x3(KH, KL, kb_rows, band_k);
  stage_x3(VH, VL, kb_rows, band_v);
  const int g_rows = (p.link_cls || p.link_query || p.partials) ? (nhead + 15) & ~15 : 0;  // 16-key blocks used
  stage_x3(GKH, GKL, g_rows, [&](int r) -> const float* { return r < nhead ? p.k + (int64_t)(g.start + r) * p.ld + hoff : nullptr; });
  stage_x3(GVH, GVL, g_rows, [&](int r) -> const float* { return r < nhead ? p.v + (int64_t)(g.start + r) * p.ld + hoff : nullptr; });
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const float c2 = 1.4426950408889634f / p.scale;
  const int wr0 = warp * 16;
  const bool glob = p.link_cls || p.link_query;
  const int nch = (16 + 2 * w + 15) / 16;

  if (wr0 < rows_here) {
    uint32_t qh[4][4], ql[4][4];
    split_q(qraw, qh, ql);
    float sg[4][4], sb[2 * MAXCH][4];
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) sg[nb][0] = sg[nb][1] = sg[nb][2] = sg[nb][3] = 0.f;
#pragma unroll
    for (int nb = 0; nb < 2 * MAXCH; ++nb) sb[nb][0] = sb[nb][1] = sb[nb][2] = sb[nb][3] = 0.f;
    if (glob) {
#pragma unroll
      for (int gb = 0; gb < 2; ++gb)
        if (gb * 16 < nhead) qk16x3(GKH, GKL, gb * 16, lane, qh, ql, sg[2 * gb], sg[2 * gb + 1]);
    }
#pragma unroll
    for (int ch = 0; ch < MAXCH; ++ch)
      if (ch < nch) qk16x3(KH, KL, wr0 + 16 * ch, lane, qh, ql, sb[2 * ch], sb[2 * ch + 1]);
    // masks: global key kg valid when linked; band smem row kr = doc position r0 - w + kr
    const int ra = r0 + wr0 + gq;  // doc-relative rows of this thread: ra, ra + 8
#pragma unroll
    for (int nb = 0; nb < 4; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kg = nb * 8 + 2 * tq + (e & 1);
        if (!(glob && kg < nhead && (kg == 0 ? p.link_cls : p.link_query))) sg[nb][e] = -INFINITY;
      }
#pragma unroll
    for (int nb = 0; nb < 2 * MAXCH; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int pos = r0 - w + wr0 + nb * 8 + 2 * tq + (e & 1);
        const int rr = ra + ((e >> 1) << 3);
        if (!(nb < 2 * nch && pos >= 0 && pos < dlen && pos - rr <= w && rr - pos <= w)) sb[nb][e] = -INFINITY;
      }
    // one softmax over the row's key set (zero-logit padding: the missing band slots enter with logit 0)
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    if (p.padding == SC_PAD_ZERO_LOGIT) {
      const int rb = ra + 8;
      const float na = (float)(2 * w + 1 - max(0, min(dlen, ra + w + 1) - max(0, ra - w)));
      const float nbv = (float)(2 * w + 1 - max(0, min(dlen, rb + w + 1) - max(0, rb - w)));
      if (na > 0.f) { m0 = 0.f; l0 = tq == 0 ? na : 0.f; }
      if (nbv > 0.f) { m1 = 0.f; l1 = tq == 0 ? nbv : 0.f; }
    }
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
      m0 = fmaxf(m0, fmaxf(sg[nb][0], sg[nb][1]));
      m1 = fmaxf(m1, fmaxf(sg[nb][2], sg[nb][3]));
    }
#pragma unroll
    for (int nb = 0; nb < 2 * MAXCH; ++nb) {
      m0 = fmaxf(m0, fmaxf(sb[nb][0], sb[nb][1]));
      m1 = fmaxf(m1, fmaxf(sb[nb][2], sb[nb][3]));
    }
    m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 1));
    m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 2));
    m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 1));
    m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 2));
    if (p.padding == SC_PAD_ZERO_LOGIT) {  // the padding's exp(0 - m) share of l
      l0 = l0 > 0.f && m0 != -INFINITY ? l0 * exp2f(-m0 * c2) : l0;
      l1 = l1 > 0.f && m1 != -INFINITY ? l1 * exp2f(-m1 * c2) : l1;
    }
    const float b0 = m0 == -INFINITY ? 0.f : m0 * c2, b1 = m1 == -INFINITY ? 0.f : m1 * c2;
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
      sg[nb][0] = exp2f(fmaf(sg[nb][0], c2, -b0)); sg[nb][1] = exp2f(fmaf(sg[nb][1], c2, -b0));
      sg[nb][2] = exp2f(fmaf(sg[nb][2], c2, -b1)); sg[nb][3] = exp2f(fmaf(sg[nb][3], c2, -b1));
      l0 += sg[nb][0] + sg[nb][1];
      l1 += sg[nb][2] + sg[nb][3];
    }
#pragma unroll
    for (int nb = 0; nb < 2 * MAXCH; ++nb) {
      sb[nb][0] = exp2f(fmaf(sb[nb][0], c2, -b0)); sb[nb][1] = exp2f(fmaf(sb[nb][1], c2, -b0));
      sb[nb][2] = exp2f(fmaf(sb[nb][2], c2, -b1)); sb[nb][3] = exp2f(fmaf(sb[nb][3], c2, -b1));
      l0 += sb[nb][0] + sb[nb][1];
      l1 += sb[nb][2] + sb[nb][3];
    }
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    float o[8][4];
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) o[nb][0] = o[nb][1] = o[nb][2] = o[nb][3] = 0.f;
    if (glob) {
#pragma unroll
      for (int gb = 0; gb < 2; ++gb)
        if (gb * 16 < nhead) pv16x3(GVH, GVL, gb * 16, lane, sg[2 * gb], sg[2 * gb + 1], o);
    }
#pragma unroll
    for (int ch = 0; ch < MAXCH; ++ch)
      if (ch < nch) pv16x3(VH, VL, wr0 + 16 * ch, lane, sb[2 * ch], sb[2 * ch + 1], o);
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int rr = ra + 8 * half;
      if (rr >= dlen) continue;
      const float l = half ? l1 : l0;
      float* dst = p.out + (int64_t)(dstart + rr) * p.ld_out + hoff + 2 * tq;
      if (!(l > 0.f)) {
        if (tq == 0 && p.status) atomicOr(p.status, 1);
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) *reinterpret_cast<float2*>(dst + nb * 8) = make_float2(0.f, 0.f);
        continue;
      }
      const float inv = 1.f / l;
#pragma unroll
      for (int nb = 0; nb < 8; ++nb)
        *reinterpret_cast<float2*>(dst + nb * 8) = make_float2(o[nb][2 * half] * inv, o[nb][2 * half + 1] * inv);
    }
  }

  // full-row records: head rows f < fneed against this tile's own doc keys (band rows w .. w + 63)
  if (p.partials && warp == (h & 3)) {
    for (int fc = 0; fc * 16 < p.fneed && fc * 16 < nhead; ++fc) {
      uint32_t qh[4][4], ql[4][4];
      load_q_x3(lane, [&](int i) -> const float* {
        const int f = fc * 16 + i;
        return f < p.fneed && f < nhead ? p.q + (int64_t)(g.start + f) * p.ld + hoff : nullptr;
      }, qh, ql);
      float sc[8][4];
#pragma unroll
      for (int nb = 0; nb < 8; ++nb) sc[nb][0] = sc[nb][1] = sc[nb][2] = sc[nb][3] = 0.f;
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) qk16x3(KH, KL, w + 16 * kc, lane, qh, ql, sc[2 * kc], sc[2 * kc + 1]);
      float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
      for (int nb = 0; nb < 8; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (nb * 8 + 2 * tq + (e & 1) >= rows_here) sc[nb][e] = -INFINITY;
          if (e < 2) m0 = fmaxf(m0, sc[nb][e]);
          else m1 = fmaxf(m1, sc[nb][e]);
        }
      m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 1));
      m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 2));
      m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 1));
      m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 2));
      float l0 = 0.f, l1 = 0.f;
#pragma unroll
      for (int nb = 0; nb < 8; ++nb) {
        sc[nb][0] = exp2f((sc[nb][0] - m0) * c2); sc[nb][1] = exp2f((sc[nb][1] - m0) * c2);
        sc[nb][2] = exp2f((sc[nb][2] - m1) * c2); sc[nb][3] = exp2f((sc[nb][3] - m1) * c2);
        l0 += sc[nb][0] + sc[nb][1];
        l1 += sc[nb][2] + sc[nb][3];
      }
      l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
      l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
      l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
      l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
      float o[8][4];
#pragma unroll
      for (int nb = 0; nb < 8; ++nb) o[nb][0] = o[nb][1] = o[nb][2] = o[nb][3] = 0.f;
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) pv16x3(VH, VL, w + 16 * kc, lane, sc[2 * kc], sc[2 * kc + 1], o);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int f = fc * 16 + gq + 8 * half;
        if (f >= p.fneed || f >= nhead) continue;
        float* rec = p.partials + (((int64_t)tile * p.H + h) * p.fmax + f) * (D + 2);
        if (tq == 0) {
          rec[0] = (half ? m1 : m0) / p.scale;  // raw logit -> the record's natural units
          rec[1] = half ? l1 : l0;
        }
#pragma unroll
        for (int nb = 0; nb < 8; ++nb)
          *reinterpret_cast<float2*>(rec + 2 + nb * 8 + 2 * tq) = make_float2(o[nb][2 * half], o[nb][2 * half + 1]);
      }
    }
  }
}

}  // namespace bandx3

// fp32 doc rows by band_f32_kernel; the caller handles the head rows.  SC_ERR_UNSUPPORTED outside
// the envelope (fp32, d = 64, window <= 32, doc -> cls / query links FULL or NONE, no QDS).
int launch_attn_band_f32(const AttnArgs& a, int dtype, const int32_t* seq_tile_base, int tile_rows,
                         int max_qgroup_len, float* records, int fneed, cudaStream_t st) {
  using namespace bandf;
  const Links& L = a.links;
  const int w = L.w[2][2];
  auto unsupported = [](const char* why) {
    set_error("fp32 band kernel: %s", why);
    return SC_ERR_UNSUPPORTED;
  };
  if (dtype != SC_DTYPE_F32 || a.d != D) return unsupported("needs fp32 and head_dim 64");
  if (a.glob_cu) return unsupported("QDS");
  if (w < 0 || w > MAXW) return unsupported("doc window");
  for (int x : {L.w[2][0], L.w[2][1]})
    if (x != SC_LINK_FULL && x != SC_LINK_NONE) return unsupported("windowed doc->head link");
  if (max_qgroup_len + 1 > MAXH) return unsupported("query group too long");
  if (tile_rows != BM || !seq_tile_base) return unsupported("layout tiles must be 64 rows");
  if ((((uintptr_t)a.q | (uintptr_t)a.k | (uintptr_t)a.v | (uintptr_t)a.out) & 15) || (a.ld % 4) || (a.ld_out % 4))
    return unsupported("alignment");
  Params p;
  p.q = static_cast<const float*>(a.q); p.k = static_cast<const float*>(a.k); p.v = static_cast<const float*>(a.v);
  p.ld = a.ld; p.out = static_cast<float*>(a.out); p.ld_out = a.ld_out;
  p.cu = a.cu; p.qlen = a.qlen; p.tile_base = seq_tile_base; p.nseq = a.nseq; p.H = a.H; p.w = w;
  p.padding = a.padding; p.link_cls = L.w[2][0] == SC_LINK_FULL; p.link_query = L.w[2][1] == SC_LINK_FULL;
  p.scale = a.scale; p.status = a.status;
  p.partials = fneed > 0 ? records : nullptr; p.fneed = fneed; p.fmax = fneed;
  const unsigned grid = (unsigned)((a.T + BM - 1) / BM + a.nseq);
  // + the full-row scratch: q row, 64 probabilities, 4 x 64 partial sums, (m, l)
  constexpr int kExtra = D + BM + 4 * D + 2;
  const size_t smem = ((size_t)(2 * (BM + 2 * w) + 2 * MAXH) * DP + kExtra) * sizeof(float);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(band_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(((2 * KB + 2 * MAXH) * DP + kExtra) * sizeof(float)));
    attr = true;
  }
  static int simt = -1;  // SC_F32_SIMT=1: the CUDA-core kernel (measurement A/B)
  if (simt < 0) simt = getenv("SC_F32_SIMT") ? atoi(getenv("SC_F32_SIMT")) : 0;
  if (!simt) {
    const int kb_rows = (bandx3::BM + 2 * w + 15) & ~15;
    const size_t smem3 = (size_t)(4 * kb_rows + 4 * bandx3::GRM) * bandx3::ROWB;
    static bool attr3 = false;
    if (!attr3) {
      cudaFuncSetAttribute(bandx3::band_f32x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (4 * ((bandx3::BM + 2 * bandx3::MAXW + 15) & ~15) + 4 * bandx3::GRM) * bandx3::ROWB);
      attr3 = true;
    }
    bandx3::band_f32x3_kernel<<<dim3(grid, (unsigned)a.H), bandx3::NT, smem3, st>>>(p);
    SC_CHECK_LAUNCH("band_f32x3_kernel");
    return SC_OK;
  }
  band_f32_kernel<<<dim3(grid, (unsigned)a.H), NT, smem, st>>>(p);
  SC_CHECK_LAUNCH("band_f32_kernel");
  return SC_OK;
}

}  // namespace sc
