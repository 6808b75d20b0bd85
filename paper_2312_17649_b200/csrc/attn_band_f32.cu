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
#include "attn.cuh"

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
  band_f32_kernel<<<dim3(grid, (unsigned)a.H), NT, smem, st>>>(p);
  SC_CHECK_LAUNCH("band_f32_kernel");
  return SC_OK;
}

}  // namespace sc
