// Attention backward for GPU fine-tuning: the adjoint of
// sc_attn_fwd for every pattern / window / padding / QDS, fp32 math.
// Replaces the reference's chain group_attention_backward ->
// attend_segments_backward -> masked_segment_softmax_backward ->
// band_scores/band_apply_backward (R/attention.py:260-269, :348-378,
// :476-507; R/band.py:239-274).
//
// Per source row i with key slots K(i) (the forward's segments; zero-logit
// padding slots join the normaliser only):
//   P_ij = exp(s_ij - lse_i),  dP_ij = dO_i . V_j,  D_i = dO_i . O_i,
//   dS_ij = P_ij (dP_ij - D_i) / scale,
//   dQ_i = sum_j dS_ij K_j,  dK_j = sum_i dS_ij Q_i,  dV_j = sum_i P_ij dO_i.
// Two gather-form kernels, no atomics, so results are bit-reproducible:
//   1. query-major, one warp per (row, head): lse_i and D_i (kept in the
//      caller's workspace), then dQ_i;
//   2. key-major, one warp per (key row, head): enumerates the source rows
//      whose slots address the key (the transposed pattern, QDS included)
//      and reduces dK_j, dV_j in registers.
// Global QDS rows attend every key densely (their windowed result is
// discarded by the reference, R/attention.py:461-470, :488-493).
#include <stdlib.h>

#include <algorithm>

#include "attn.cuh"

namespace sc {

constexpr int kBwdWarps = 4;
constexpr int kBwdMaxD = 128;
constexpr int kLongRange = 32;  // ranges of >= this many rows go lane-parallel (coop_dots)

// A head row lives in registers: lane holds dims lane + 32e, e < E (E = ceil(d/32)).
template <typename T, int E>
__device__ __forceinline__ void load_vec(float (&x)[E], const T* __restrict__ r, int lane, int d) {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int c = lane + 32 * e;
    x[e] = c < d ? to_f32(r[c]) : 0.f;
  }
}

template <typename T, int E>
__device__ __forceinline__ float dot_part(const float (&x)[E], const T* __restrict__ r, float (&y)[E], int lane,
                                          int d) {
  float acc = 0.f;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int c = lane + 32 * e;
    y[e] = c < d ? to_f32(r[c]) : 0.f;
    acc = fmaf(x[e], y[e], acc);
  }
  return acc;
}

struct BwdArgs {
  AttnArgs a;
  const void* dout;
  int64_t ld_dout;
  void* dq;
  void* dk;
  void* dv;
  int grad_bf16;
  int64_t ld_grad;
  float2* stats;  // [T*H]: (lse, D); lse = +inf for rows without keys
  int mode;       // 0: every row; 1: only the head rows (cls + query group) of every sequence
  int maxh;       // mode 1: 1 + max qgroup_len (items per sequence)
};

// Item -> (row, head).  Mode 1 enumerates nseq x maxh slots, skipping slots past a sequence's head rows.
__device__ __forceinline__ bool map_item(const BwdArgs& b, int64_t item, int& row, int& h) {
  const AttnArgs& a = b.a;
  h = (int)(item % a.H);
  const int64_t r = item / a.H;
  if (b.mode == 0) {
    row = (int)r;
    return row < a.T;
  }
  const int j = (int)(r / b.maxh), i = (int)(r % b.maxh);
  if (j >= a.nseq || i >= 1 + a.qlen[j]) return false;
  row = a.cu[j] + i;
  return true;
}

__device__ __forceinline__ bool is_global(const AttnArgs& a, int row) {
  return a.glob_cu != nullptr && a.flags && (a.flags[row] & 1);
}

// A run of candidate rows: rows base + t for t in [lo, hi) (or glob_pos[lo..hi) when pos != null),
// minus rows rejected by `skip`.
struct Range {
  int base, lo, hi;
  const int32_t* pos;
  int skip;  // 0 none, 1 drop QDS-global rows, 2 keep only non-global rows (same test)
};

__device__ __forceinline__ int range_row(const Range& R, int t) { return R.base + (R.pos ? R.pos[t] : t); }

// Key ranges of source row (gs, rs) of sequence j, forward slot order.  Returns the count.
__device__ __forceinline__ int key_ranges(const AttnArgs& a, const SeqGroups& g, int j, int gs, int rs,
                                          bool src_global, Range (&out)[4]) {
  const bool qds = a.glob_cu != nullptr;
  int n = 0;
  for (int t = 0; t < 3; ++t) {
    const int w = src_global ? SC_LINK_FULL : a.links.w[gs][t];
    if (w == SC_LINK_NONE) continue;
    int lo = 0, hi = g.len[t];
    if (w >= 0) { lo = max(0, rs - w); hi = min(g.len[t], rs + w + 1); }
    out[n++] = Range{g.start + g.off[t], lo, hi, nullptr, (qds && gs == 2 && t == 2 && w >= 0) ? 1 : 0};
  }
  if (qds && gs == 2 && !src_global)
    out[n++] = Range{g.start + g.off[2], a.glob_cu[j], a.glob_cu[j + 1], a.glob_pos, 0};
  return n;
}

// Source ranges whose slots address key (tg, r) of sequence j (the transposed pattern).
__device__ __forceinline__ int source_ranges(const AttnArgs& a, const SeqGroups& g, int j, int tg, int r,
                                             bool key_global, Range (&out)[5]) {
  const bool qds = a.glob_cu != nullptr;
  int n = 0;
  for (int gs = 0; gs < 3; ++gs) {
    const int w = a.links.w[gs][tg];
    const bool qds_doc = qds && gs == 2;
    if (w == SC_LINK_NONE || (qds_doc && tg == 2 && w >= 0 && key_global)) continue;
    int lo = 0, hi = g.len[gs];
    if (w >= 0) { lo = max(0, r - w); hi = min(g.len[gs], r + w + 1); }
    out[n++] = Range{g.start + g.off[gs], lo, hi, nullptr, qds_doc ? 1 : 0};
  }
  if (qds) {
    if (key_global) out[n++] = Range{g.start + g.off[2], 0, g.len[2], nullptr, 1};  // dense globals segment
    out[n++] = Range{g.start + g.off[2], a.glob_cu[j], a.glob_cu[j + 1], a.glob_pos, 0};  // global rows
  }
  return n;
}

// Visit the rows of a range: full 32-row chunks lane-parallel (chunk(valid, row)), the rest in
// groups of kGroup rows processed together by the whole warp (group(rows, ok)) so their loads and
// reductions overlap.  Work units (chunks / groups, counted across ranges by `unit`) are dealt
// round-robin to the nsplit warps cooperating on one item.
constexpr int kGroup = 4;

template <typename Group, typename Chunk>
__device__ __forceinline__ void visit(const AttnArgs& a, const Range& R, int lane, int split, int nsplit, int& unit,
                                      Group&& group, Chunk&& chunk) {
  int t = R.lo;
  if (R.hi - R.lo >= kLongRange) {
    for (; t + 32 <= R.hi; t += 32) {
      if (unit++ % nsplit != split) continue;
      const int row = range_row(R, t + lane);
      const bool valid = !(R.skip && is_global(a, row));
      chunk(valid, row);
    }
  }
  for (; t < R.hi; t += kGroup) {
    if (unit++ % nsplit != split) continue;
    int rows[kGroup];
    bool ok[kGroup];
#pragma unroll
    for (int u = 0; u < kGroup; ++u) {
      ok[u] = t + u < R.hi;
      rows[u] = range_row(R, ok[u] ? t + u : t);
      if (ok[u] && R.skip && is_global(a, rows[u])) ok[u] = false;
    }
    group(rows, ok);
  }
}

// N independent warp reductions, interleaved.
template <int N>
__device__ __forceinline__ void warp_sum_n(float (&v)[N]) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int u = 0; u < N; ++u) v[u] += __shfl_xor_sync(0xffffffffu, v[u], off);
  }
}

// Lane-private dot product of a shared-memory row x with one global row (16-byte loads when aligned).
template <typename T>
__device__ __forceinline__ float lane_dot(const float* __restrict__ x, const T* __restrict__ r, int d) {
  float acc = 0.f;
  constexpr int V = 16 / sizeof(T);
  if ((d % V) == 0 && (reinterpret_cast<uintptr_t>(r) & 15) == 0) {
    const uint4* rv = reinterpret_cast<const uint4*>(r);
    for (int c = 0; c < d / V; ++c) {
      const uint4 u = __ldg(rv + c);
      if constexpr (sizeof(T) == 2) {
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(b2[e]);
          acc = fmaf(x[V * c + 2 * e], f.x, fmaf(x[V * c + 2 * e + 1], f.y, acc));
        }
      } else {
        const float* f = reinterpret_cast<const float*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) acc = fmaf(x[V * c + e], f[e], acc);
      }
    }
    return acc;
  }
  for (int c = 0; c < d; ++c) acc = fmaf(x[c], to_f32(r[c]), acc);
  return acc;
}

// Per-warp staging of register rows (lane holds dims lane + 32e) into shared memory.
template <int E>
__device__ __forceinline__ void stash(float* dst, const float (&x)[E], int lane, int d) {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int c = lane + 32 * e;
    if (c < d) dst[c] = x[e];
  }
}

// Item geometry.  NS == 1: one warp per item, kBwdWarps items per CTA.  NS > 1: one CTA of NS warps
// per item, the warps splitting the item's key (or source) ranges; partials reduced in shared memory
// in warp order (deterministic).
template <int NS>
struct ItemSlot {
  static constexpr int kWarpsPerCta = NS > 1 ? NS : kBwdWarps;
  __device__ static int64_t item(int warp) { return NS > 1 ? (int64_t)blockIdx.x : (int64_t)blockIdx.x * kBwdWarps + warp; }
  __device__ static int split(int warp) { return NS > 1 ? warp : 0; }
};

// Kernel 1: lse_i, D_i and dQ_i per (row, head).
template <typename T, int E, int NS>
__global__ void __launch_bounds__(ItemSlot<NS>::kWarpsPerCta * 32) attn_bwd_dq_kernel(BwdArgs b) {
  constexpr int WPC = ItemSlot<NS>::kWarpsPerCta;
  __shared__ float xs_all[WPC][2][kBwdMaxD];
  __shared__ float red_ml[NS][2];
  __shared__ float red_v[NS > 1 ? NS : 1][kBwdMaxD];
  const AttnArgs& a = b.a;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int split = ItemSlot<NS>::split(warp);
  int row, h;
  if (!map_item(b, ItemSlot<NS>::item(warp), row, h)) return;  // uniform per CTA when NS > 1
  const int j = find_seq(a.cu, a.nseq, row);
  const T* Q = static_cast<const T*>(a.q);
  const T* K = static_cast<const T*>(a.k);
  const T* V = static_cast<const T*>(a.v);
  const T* O = static_cast<const T*>(a.out);
  const T* dO = static_cast<const T*>(b.dout);
  const int d = a.d, hoff = h * d;
  const float inv_scale = 1.f / a.scale;
  const SeqGroups g = seq_groups(a.cu, a.qlen, j);
  const int i = row - g.start;
  const int gs = i == 0 ? 0 : (i < 1 + g.len[1] ? 1 : 2);
  const int rs = i - g.off[gs];
  const bool src_global = gs == 2 && is_global(a, row);

  float qr[E], dr[E], o[E];
  load_vec<T, E>(qr, Q + (int64_t)row * a.ld + hoff, lane, d);
  load_vec<T, E>(dr, dO + (int64_t)row * b.ld_dout + hoff, lane, d);
  load_vec<T, E>(o, O + (int64_t)row * a.ld_out + hoff, lane, d);
  float* qs = xs_all[warp][0];
  float* ds_ = xs_all[warp][1];
  stash<E>(qs, qr, lane, d);
  stash<E>(ds_, dr, lane, d);
  __syncwarp();
  float dpart = 0.f;
#pragma unroll
  for (int e = 0; e < E; ++e) dpart = fmaf(dr[e], o[e], dpart);
  const float D = warp_sum(dpart);

  Range R[4];
  const int nr = key_ranges(a, g, j, gs, rs, src_global, R);

  // pass 1: row max and normaliser (uniform per warp); zero-logit padding slots enter with logit 0
  float m = -INFINITY, l = 0.f;
  if (split == 0 && a.padding == SC_PAD_ZERO_LOGIT && !src_global) {
    int n_inv = 0;
    for (int t = 0; t < 3; ++t) {
      const int w = a.links.w[gs][t];
      if (w < 0) continue;
      const int lo = max(0, rs - w), hi = min(g.len[t], rs + w + 1);
      n_inv += (2 * w + 1) - max(0, hi - lo);
    }
    if (n_inv > 0) { m = 0.f; l = (float)n_inv; }
  }
  auto fold = [&](float s) {  // uniform logit
    if (s > m) { l = l * expf(m - s) + 1.f; m = s; }
    else l += expf(s - m);
  };
  int unit = 0;
  for (int ri = 0; ri < nr; ++ri) {
    visit(a, R[ri], lane, split, NS, unit,
          [&](const int (&kr)[kGroup], const bool (&ok)[kGroup]) {
            float sp[kGroup];
#pragma unroll
            for (int u = 0; u < kGroup; ++u) {
              float y[E];
              sp[u] = ok[u] ? dot_part<T, E>(qr, K + (int64_t)kr[u] * a.ld + hoff, y, lane, d) : 0.f;
            }
            warp_sum_n<kGroup>(sp);
#pragma unroll
            for (int u = 0; u < kGroup; ++u)
              if (ok[u]) fold(sp[u] * inv_scale);
          },
          [&](bool valid, int kr) {
            const float s = valid ? lane_dot<T>(qs, K + (int64_t)kr * a.ld + hoff, d) * inv_scale : -INFINITY;
            const float cmax = warp_max(s);
            if (cmax == -INFINITY) return;
            const float mnew = fmaxf(m, cmax);
            const float csum = warp_sum(valid ? expf(s - mnew) : 0.f);
            l = l * (m == -INFINITY ? 0.f : expf(m - mnew)) + csum;
            m = mnew;
          });
  }
  if constexpr (NS > 1) {  // combine the warps' (m, l) in warp order
    if (lane == 0) { red_ml[split][0] = m; red_ml[split][1] = l; }
    __syncthreads();
    m = -INFINITY;
    for (int u = 0; u < NS; ++u) m = fmaxf(m, red_ml[u][0]);
    l = 0.f;
    for (int u = 0; u < NS; ++u)
      if (red_ml[u][0] != -INFINITY) l += red_ml[u][1] * expf(red_ml[u][0] - m);
  }
  const float lse = l > 0.f ? m + logf(l) : INFINITY;
  if (lane == 0 && split == 0) b.stats[(int64_t)row * a.H + h] = make_float2(lse, D);

  // pass 2: dQ_i = sum_j dS_ij K_j
  float dq[E];
#pragma unroll
  for (int e = 0; e < E; ++e) dq[e] = 0.f;
  if (l > 0.f) {
    unit = 0;
    for (int ri = 0; ri < nr; ++ri) {
      visit(a, R[ri], lane, split, NS, unit,
            [&](const int (&kr)[kGroup], const bool (&ok)[kGroup]) {
              float kv[kGroup][E], sp[2 * kGroup];
#pragma unroll
              for (int u = 0; u < kGroup; ++u) {
                float vv[E];
                sp[u] = ok[u] ? dot_part<T, E>(qr, K + (int64_t)kr[u] * a.ld + hoff, kv[u], lane, d) : 0.f;
                sp[kGroup + u] = ok[u] ? dot_part<T, E>(dr, V + (int64_t)kr[u] * a.ld + hoff, vv, lane, d) : 0.f;
              }
              warp_sum_n<2 * kGroup>(sp);
#pragma unroll
              for (int u = 0; u < kGroup; ++u) {
                if (!ok[u]) continue;
                const float dsv = expf(sp[u] * inv_scale - lse) * (sp[kGroup + u] - D) * inv_scale;
#pragma unroll
                for (int e = 0; e < E; ++e) dq[e] = fmaf(dsv, kv[u][e], dq[e]);
              }
            },
            [&](bool valid, int kr) {
              float dsv = 0.f;
              if (valid) {
                const float sd = lane_dot<T>(qs, K + (int64_t)kr * a.ld + hoff, d);
                const float dp = lane_dot<T>(ds_, V + (int64_t)kr * a.ld + hoff, d);
                dsv = expf(sd * inv_scale - lse) * (dp - D) * inv_scale;
              }
              const unsigned vm = __ballot_sync(0xffffffffu, valid && dsv != 0.f);
#pragma unroll
              for (int kk = 0; kk < 32; ++kk) {
                const float dsk = __shfl_sync(0xffffffffu, dsv, kk);
                const T* krp = K + (int64_t)__shfl_sync(0xffffffffu, kr, kk) * a.ld + hoff;
                if ((vm >> kk) & 1u) {
#pragma unroll
                  for (int e = 0; e < E; ++e) {
                    const int c = lane + 32 * e;
                    if (c < d) dq[e] = fmaf(dsk, to_f32(krp[c]), dq[e]);
                  }
                }
              }
            });
    }
  }
  if constexpr (NS > 1) {
    stash<E>(red_v[split], dq, lane, d);
    __syncthreads();
    if (split != 0) return;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int c = lane + 32 * e;
      float acc = 0.f;
      if (c < d)
        for (int u = 0; u < NS; ++u) acc += red_v[u][c];
      dq[e] = acc;
    }
  }
  const int64_t dqo = (int64_t)row * b.ld_grad + hoff;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int c = lane + 32 * e;
    if (c < d) store_grad(b.dq, dqo + c, dq[e], b.grad_bf16);
  }
}

// Kernel 2: dK_j, dV_j per (key row, head), over the transposed pattern.
template <typename T, int E, int NS>
__global__ void __launch_bounds__(ItemSlot<NS>::kWarpsPerCta * 32) attn_bwd_dkv_kernel(BwdArgs b) {
  constexpr int WPC = ItemSlot<NS>::kWarpsPerCta;
  __shared__ float xs_all[WPC][2][kBwdMaxD];
  __shared__ float red_k[NS > 1 ? NS : 1][kBwdMaxD];
  __shared__ float red_vv[NS > 1 ? NS : 1][kBwdMaxD];
  const AttnArgs& a = b.a;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int split = ItemSlot<NS>::split(warp);
  int krow, h;
  if (!map_item(b, ItemSlot<NS>::item(warp), krow, h)) return;
  const int j = find_seq(a.cu, a.nseq, krow);
  const T* Q = static_cast<const T*>(a.q);
  const T* K = static_cast<const T*>(a.k);
  const T* V = static_cast<const T*>(a.v);
  const T* dO = static_cast<const T*>(b.dout);
  const int d = a.d, hoff = h * d;
  const float inv_scale = 1.f / a.scale;
  const SeqGroups g = seq_groups(a.cu, a.qlen, j);
  const int i = krow - g.start;
  const int tg = i == 0 ? 0 : (i < 1 + g.len[1] ? 1 : 2);
  const int r = i - g.off[tg];
  const bool key_global = tg == 2 && is_global(a, krow);

  float kr[E], vr[E];
  load_vec<T, E>(kr, K + (int64_t)krow * a.ld + hoff, lane, d);
  load_vec<T, E>(vr, V + (int64_t)krow * a.ld + hoff, lane, d);
  float* ks = xs_all[warp][0];
  float* vs = xs_all[warp][1];
  stash<E>(ks, kr, lane, d);
  stash<E>(vs, vr, lane, d);
  __syncwarp();
  float dk[E], dv[E];
#pragma unroll
  for (int e = 0; e < E; ++e) { dk[e] = 0.f; dv[e] = 0.f; }

  Range R[5];
  const int nr = source_ranges(a, g, j, tg, r, key_global, R);
  int unit = 0;
  for (int ri = 0; ri < nr; ++ri) {
    visit(a, R[ri], lane, split, NS, unit,
          [&](const int (&src)[kGroup], const bool (&ok)[kGroup]) {
            float qv[kGroup][E], gv[kGroup][E], sp[2 * kGroup];
            float2 st[kGroup];
#pragma unroll
            for (int u = 0; u < kGroup; ++u) {
              sp[u] = ok[u] ? dot_part<T, E>(kr, Q + (int64_t)src[u] * a.ld + hoff, qv[u], lane, d) : 0.f;
              sp[kGroup + u] =
                  ok[u] ? dot_part<T, E>(vr, dO + (int64_t)src[u] * b.ld_dout + hoff, gv[u], lane, d) : 0.f;
              st[u] = ok[u] ? b.stats[(int64_t)src[u] * a.H + h] : make_float2(INFINITY, 0.f);
            }
            warp_sum_n<2 * kGroup>(sp);
#pragma unroll
            for (int u = 0; u < kGroup; ++u) {
              if (!ok[u]) continue;
              const float p = expf(sp[u] * inv_scale - st[u].x);
              const float dsv = p * (sp[kGroup + u] - st[u].y) * inv_scale;
#pragma unroll
              for (int e = 0; e < E; ++e) {
                dk[e] = fmaf(dsv, qv[u][e], dk[e]);
                dv[e] = fmaf(p, gv[u][e], dv[e]);
              }
            }
          },
          [&](bool valid, int src) {
            float p = 0.f, dsv = 0.f;
            if (valid) {
              const float2 st = b.stats[(int64_t)src * a.H + h];
              const float sd = lane_dot<T>(ks, Q + (int64_t)src * a.ld + hoff, d);
              const float dp = lane_dot<T>(vs, dO + (int64_t)src * b.ld_dout + hoff, d);
              p = expf(sd * inv_scale - st.x);
              dsv = p * (dp - st.y) * inv_scale;
            }
            const unsigned live = __ballot_sync(0xffffffffu, valid && p != 0.f);
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) {
              const float pk = __shfl_sync(0xffffffffu, p, kk), dsk = __shfl_sync(0xffffffffu, dsv, kk);
              const int sr = __shfl_sync(0xffffffffu, src, kk);
              if ((live >> kk) & 1u) {
                const T* qp = Q + (int64_t)sr * a.ld + hoff;
                const T* gp = dO + (int64_t)sr * b.ld_dout + hoff;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                  const int c = lane + 32 * e;
                  if (c < d) {
                    dk[e] = fmaf(dsk, to_f32(qp[c]), dk[e]);
                    dv[e] = fmaf(pk, to_f32(gp[c]), dv[e]);
                  }
                }
              }
            }
          });
  }
  if constexpr (NS > 1) {
    stash<E>(red_k[split], dk, lane, d);
    stash<E>(red_vv[split], dv, lane, d);
    __syncthreads();
    if (split != 0) return;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int c = lane + 32 * e;
      float ak = 0.f, av = 0.f;
      if (c < d)
        for (int u = 0; u < NS; ++u) { ak += red_k[u][c]; av += red_vv[u][c]; }
      dk[e] = ak;
      dv[e] = av;
    }
  }
  const int64_t ko = (int64_t)krow * b.ld_grad + hoff;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int c = lane + 32 * e;
    if (c < d) {
      store_grad(b.dk, ko + c, dk[e], b.grad_bf16);
      store_grad(b.dv, ko + c, dv[e], b.grad_bf16);
    }
  }
}

// Mode 0: one warp per (row, head).  Mode 1 (head rows / keys): a CTA of kHeadSplit warps per
// (row, head) when sequences are long (dense ranges of thousands of keys), else one warp each.
constexpr int kHeadSplit = 16;
constexpr int kSplitMinAvgLen = 768;

template <typename T, int E>
int launch_generic(const BwdArgs& b, int which, cudaStream_t st) {
  const bool split = b.mode == 1 && (int64_t)b.a.T >= (int64_t)kSplitMinAvgLen * b.a.nseq;
  if (!split) {
    const int64_t items = b.mode == 0 ? (int64_t)b.a.T * b.a.H : (int64_t)b.a.nseq * b.maxh * b.a.H;
    const unsigned blocks = (unsigned)((items + kBwdWarps - 1) / kBwdWarps);
    if (which == 0) attn_bwd_dq_kernel<T, E, 1><<<blocks, kBwdWarps * 32, 0, st>>>(b);
    else attn_bwd_dkv_kernel<T, E, 1><<<blocks, kBwdWarps * 32, 0, st>>>(b);
  } else {
    const unsigned blocks = (unsigned)((int64_t)b.a.nseq * b.maxh * b.a.H);
    if (which == 0) attn_bwd_dq_kernel<T, E, kHeadSplit><<<blocks, kHeadSplit * 32, 0, st>>>(b);
    else attn_bwd_dkv_kernel<T, E, kHeadSplit><<<blocks, kHeadSplit * 32, 0, st>>>(b);
  }
  SC_CHECK_LAUNCH(which == 0 ? "attn_bwd_dq_kernel" : "attn_bwd_dkv_kernel");
  return SC_OK;
}

template <typename T>
int launch_generic_d(const BwdArgs& b, int which, cudaStream_t st) {
  const int d = b.a.d;
  if (d <= 32) return launch_generic<T, 1>(b, which, st);
  if (d <= 64) return launch_generic<T, 2>(b, which, st);
  return launch_generic<T, 4>(b, which, st);
}

int launch_generic_any(const BwdArgs& b, int dtype, int which, cudaStream_t st) {
  return dtype == SC_DTYPE_F32 ? launch_generic_d<float>(b, which, st) : launch_generic_d<__nv_bfloat16>(b, which, st);
}

}  // namespace sc

using namespace sc;

// SC_BWD_GENERIC=1 forces the generic kernels (A/B experiments, parity cross-checks).
static bool force_generic() {
  static const bool v = [] {
    const char* e = getenv("SC_BWD_GENERIC");
    return e && atoi(e) != 0;
  }();
  return v;
}

static size_t stats_bytes(int32_t total_tokens, int32_t heads) {
  return (size_t)(total_tokens > 0 ? total_tokens : 0) * (size_t)(heads > 0 ? heads : 0) * sizeof(float2);
}

// Head-key partials of the tiled path: <= T/64 + nseq tiles x H x 2 x NH x 64 fp32.
static size_t part_bytes(int32_t total_tokens, int32_t heads, int32_t nseq, int32_t max_qgroup_len) {
  const int nh = 1 + max_qgroup_len <= 16 ? 16 : 32;
  const size_t tiles = (size_t)(total_tokens / 64 + 1) + (size_t)(nseq > 0 ? nseq : 0);
  return tiles * (size_t)(heads > 0 ? heads : 0) * 2 * nh * 64 * sizeof(float);
}

// Head-row pass split over key ranges: nseq x H x kMaxHeadSplit x 32 rows x (m, l, dq[64]).
constexpr int kMaxHeadSplit = 8;
static size_t split_bytes(int32_t heads, int32_t nseq) {
  return (size_t)(nseq > 0 ? nseq : 0) * (heads > 0 ? heads : 0) * kMaxHeadSplit * 32 * 66 * sizeof(float);
}

extern "C" size_t sc_attn_bwd_workspace_bytes(int32_t total_tokens, int32_t heads, int32_t nseq,
                                              int32_t max_qgroup_len) {
  return ((stats_bytes(total_tokens, heads) + 255) & ~(size_t)255) +
         ((part_bytes(total_tokens, heads, nseq, max_qgroup_len) + 255) & ~(size_t)255) + split_bytes(heads, nseq);
}

extern "C" int sc_attn_bwd(const void* q, const void* k, const void* v, int64_t row_stride, const void* out,
                           int64_t out_row_stride, const void* dout, int64_t dout_row_stride, void* dq, void* dk,
                           void* dv, int64_t grad_row_stride, int32_t grad_dtype, const int32_t* cu_seqlens,
                           const int32_t* qgroup_len,
                           int32_t nseq, int32_t total_tokens, int32_t heads, int32_t head_dim, const int32_t* links,
                           int32_t padding, float scale, int32_t dtype, const uint8_t* tok_flags,
                           const int32_t* glob_cu, const int32_t* glob_pos, const int32_t* seq_tile_base,
                           int32_t tile_rows, int32_t max_qgroup_len, int32_t n_tiles, void* workspace,
                           size_t workspace_bytes, void* stream) {
  BwdArgs b = {};
  AttnArgs& a = b.a;
  SC_CHECK_ARG(load_links(links, &a.links), "sc_attn_bwd: bad links");
  SC_CHECK_ARG(q && k && v && out && dout && dq && dk && dv && cu_seqlens && qgroup_len, "sc_attn_bwd: null pointer");
  SC_CHECK_ARG(nseq >= 1 && total_tokens >= 3 * nseq, "sc_attn_bwd: bad nseq/total_tokens");
  SC_CHECK_ARG(heads >= 1 && head_dim >= 1 && head_dim <= kBwdMaxD, "sc_attn_bwd: head_dim must be in [1,128]");
  SC_CHECK_ARG(grad_row_stride >= (int64_t)heads * head_dim, "sc_attn_bwd: gradient row stride too small");
  SC_CHECK_ARG(padding == SC_PAD_EXCLUDE || padding == SC_PAD_ZERO_LOGIT, "unknown padding mode %d", padding);
  SC_CHECK_ARG(scale > 0.f, "scale must be positive");
  SC_CHECK_ARG(dtype == SC_DTYPE_F32 || dtype == SC_DTYPE_BF16, "sc_attn_bwd: bad dtype %d", dtype);
  SC_CHECK_ARG((glob_cu == nullptr) == (glob_pos == nullptr) && (glob_cu == nullptr || tok_flags != nullptr),
               "sc_attn_bwd: QDS globals need tok_flags, glob_cu and glob_pos");
  SC_CHECK_ARG(max_qgroup_len >= 1, "sc_attn_bwd: max_qgroup_len must be >= 1");
  SC_CHECK_ARG(grad_dtype == SC_DTYPE_F32 || grad_dtype == SC_DTYPE_BF16, "sc_attn_bwd: bad grad_dtype %d",
               grad_dtype);
  SC_CHECK_ARG(workspace && workspace_bytes >= stats_bytes(total_tokens, heads),
               "sc_attn_bwd: workspace must hold sc_attn_bwd_workspace_bytes(T, H, nseq, max_qgroup_len) bytes");
  a.q = q; a.k = k; a.v = v; a.ld = row_stride; a.out = const_cast<void*>(out); a.ld_out = out_row_stride;
  a.cu = cu_seqlens; a.qlen = qgroup_len; a.nseq = nseq; a.T = total_tokens; a.H = heads; a.d = head_dim;
  a.padding = padding; a.scale = scale; a.flags = tok_flags; a.glob_cu = glob_cu; a.glob_pos = glob_pos;
  b.dout = dout; b.ld_dout = dout_row_stride; b.dq = dq; b.dk = dk; b.dv = dv; b.ld_grad = grad_row_stride;
  b.grad_bf16 = grad_dtype == SC_DTYPE_BF16;
  b.stats = static_cast<float2*>(workspace);
  b.maxh = 1 + max_qgroup_len;
  cudaStream_t st = (cudaStream_t)stream;

  // Fast path: bf16, d = 64, no QDS, a finite doc->doc window <= 24, head groups <= 32 rows, 64-row
  // tiles from sc_index_build: doc rows / keys on the tiled tensor-core kernels, head rows / keys generic.
  const int wdd = a.links.w[2][2];
  const bool aligned = ((row_stride | out_row_stride | dout_row_stride) % 8) == 0 &&
                       (((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)out | (uintptr_t)dout) % 16) == 0 &&
                       grad_row_stride % 2 == 0 && ((uintptr_t)dq | (uintptr_t)dk | (uintptr_t)dv) % 8 == 0;
  // (bf16 gradients: 4-byte aligned pairs suffice, implied by the above)
  const bool fast = dtype == SC_DTYPE_BF16 && head_dim == 64 && glob_cu == nullptr && seq_tile_base &&
                    tile_rows == 64 && wdd >= 0 && wdd <= 24 && b.maxh <= 32 && aligned &&
                    !force_generic();
  if (!fast) {
    b.mode = 0;
    int rc = launch_generic_any(b, dtype, 0, st);
    return rc ? rc : launch_generic_any(b, dtype, 1, st);
  }
  BandBwdArgs p = {};
  p.q = (const __nv_bfloat16*)q; p.k = (const __nv_bfloat16*)k; p.v = (const __nv_bfloat16*)v;
  p.out = (const __nv_bfloat16*)out; p.dout = (const __nv_bfloat16*)dout;
  p.ld = row_stride; p.ld_out = out_row_stride; p.ld_dout = dout_row_stride;
  p.dq = dq; p.dk = dk; p.dv = dv; p.ld_grad = grad_row_stride; p.stats = b.stats; p.grad_bf16 = b.grad_bf16;
  p.cu = cu_seqlens; p.qlen = qgroup_len; p.tile_base = seq_tile_base; p.nseq = nseq; p.H = heads; p.w = wdd;
  p.links = a.links; p.padding = padding; p.inv_scale = 1.f / scale;
  // head-key partials when the workspace has room (else the generic head-key pass sums doc sources)
  const size_t soff = (stats_bytes(total_tokens, heads) + 255) & ~(size_t)255;
  const size_t pbytes = (part_bytes(total_tokens, heads, nseq, max_qgroup_len) + 255) & ~(size_t)255;
  if (workspace_bytes >= soff + pbytes)
    p.head_part = reinterpret_cast<float*>(static_cast<char*>(workspace) + soff);
  // head-row pass: 1 warp per (sequence, head) CTA for short sequences (<= 4 key chunks of 64: every
  // CTA resident in one wave), else 2 (measured best of 1 / 2 / 8 at 8 x 4099), keys split over CTAs
  // when there are too few (sequence, head) pairs
  p.head_warps = (int64_t)total_tokens <= (int64_t)256 * nseq ? 1 : 2;
  static const int hw_env = [] { const char* e = getenv("SC_BWD_HEAD_WARPS"); return e ? atoi(e) : 0; }();
  if (hw_env == 1 || hw_env == 2 || hw_env == 8) p.head_warps = hw_env;  // measurement override
  p.head_ks = 1;
  if (workspace_bytes >= soff + pbytes + split_bytes(heads, nseq)) {
    p.head_split = reinterpret_cast<float*>(static_cast<char*>(workspace) + soff + pbytes);
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int items = nseq * heads;
    const int want = (2 * sms + items - 1) / items;
    const int by_len = (int)((int64_t)total_tokens / nseq / 64 / p.head_warps);  // >= one 64-key chunk per warp
    p.head_ks = std::max(1, std::min({kMaxHeadSplit, want, by_len}));
    static const int ks_env = [] { const char* e = getenv("SC_BWD_HEAD_KS"); return e ? atoi(e) : 0; }();
    if (ks_env >= 1 && ks_env <= kMaxHeadSplit) p.head_ks = ks_env;  // measurement override
  }
  int ntiles = n_tiles;
  if (ntiles < 0 && (cudaMemcpyAsync(&ntiles, seq_tile_base + nseq, sizeof(int), cudaMemcpyDeviceToHost, st) !=
                         cudaSuccess ||
                     cudaStreamSynchronize(st) != cudaSuccess)) {
    set_error("sc_attn_bwd: reading the tile count failed");
    return SC_ERR_CUDA;
  }
  b.mode = 1;
  int rc = launch_attn_bwd_band(p, ntiles, b.maxh, 3, st);   // head rows: stats + dQ (tensor cores)
  if (!rc && ntiles) rc = launch_attn_bwd_band(p, ntiles, b.maxh, 0, st);  // doc rows: stats + dQ
  if (!rc && ntiles) rc = launch_attn_bwd_band(p, ntiles, b.maxh, 1, st);  // doc keys: dK, dV
  // head keys: the head-row pass wrote their dK/dV from the head sources (chunk 0) when the
  // doc-source partials exist; add those.  Otherwise the generic pass sums every source.
  if (p.head_part != nullptr && ntiles > 0) {
    if (!rc) rc = launch_attn_bwd_band(p, ntiles, b.maxh, 2, st);
  } else if (!rc) {
    rc = launch_generic_any(b, dtype, 1, st);
  }
  return rc;
}
